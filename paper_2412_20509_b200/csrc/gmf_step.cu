// K3 (tracked objective), K2 (tracker + EMA/adaptive update + NB shape) and
// the small helper kernels of the fit engine.
#include "gmf_engine.cuh"

namespace gmf {

// value of Y at (local row i, column j): dense or CSR (binary search in row)
GMF_D double y_at(const Params& P, int64_t i, int64_t j) {
  if (P.yfmt == GMF_Y_DENSE_I32) return (double)P.y[i * P.m + j];
  int64_t lo = P.rp[i], hi = P.rp[i + 1];
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    const int cm = P.ci[mid];
    if (cm == j) return (double)P.cv[mid];
    if (cm < j) lo = mid + 1; else hi = mid;
  }
  return 0.0;
}

// eta at (i, j) in fp64 from the current parameters (optim.py:274-280)
template <typename T>
GMF_D double eta_at(const Params& P, int64_t i, int64_t j) {
  const T* tr = tptr<T>(P.th_row) + i * P.Kr;
  const T* tc = tptr<T>(P.th_col) + j * P.Kc;
  double eta = 0.0;
  for (int k = 0; k < P.d; ++k) eta += (double)tr[P.q + k] * (double)tc[P.p + k];
  const T* x = tptr<T>(P.x) + i * P.p;
  for (int k = 0; k < P.p; ++k) eta += (double)x[k] * (double)tc[k];
  const T* z = tptr<T>(P.z) + j * P.q;
  for (int k = 0; k < P.q; ++k) eta += (double)tr[k] * (double)z[k];
  if (P.has_off) eta += (double)tptr<T>(P.off)[i];
  return eta;
}

// ---------------------------------------------------------------------------
// K3: tracked objective partials of the current state (optim.py:283-290).
// Runs at epoch boundaries (t % S == 0); the last CTA folds the deviance
// partials, the per-block row norms and the column norms into the record.
// ---------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(kThreads) k_obj(Params P) {
  __shared__ double scr[kThreads / 32];
  const Ctrl* C = P.ctrl;
  if (C->stopped || (C->t % P.S) != 0) return;
  const double alpha = C->nb_shape;
  const T* wg = tptr<T>(P.w);
  double s = 0.0;
  for (int64_t e = blockIdx.x * (int64_t)kThreads + threadIdx.x; e < P.E;
       e += (int64_t)gridDim.x * kThreads) {
    const int64_t i = P.erow[e];
    const int64_t j = P.ecol[e];
    const double mu = exp(eta_at<T>(P, i, j));
    const double w = P.has_w ? (double)wg[i * P.m + j] : 1.0;
    s += w * unit_deviance(P.fam, y_at(P, i, j), mu, alpha);
  }
  s = block_sum<kThreads>(s, scr);
  if (threadIdx.x == 0) P.objpart[blockIdx.x] = s;
  unsigned int* tk = P.tickets + 2 * P.CT + 1;
  if (!last_block_ticket(tk, gridDim.x)) return;
  // column norms ||B||^2, ||V||^2 (model.py:259-265)
  const T* tc = tptr<T>(P.th_col);
  double nb = 0.0, nv = 0.0;
  for (int64_t e = threadIdx.x; e < P.m * P.Kc; e += kThreads) {
    const double v = (double)tc[e];
    if ((int)(e % P.Kc) < P.p) nb += v * v; else nv += v * v;
  }
  nb = block_sum<kThreads>(nb, scr);
  nv = block_sum<kThreads>(nv, scr);
  if (threadIdx.x == 0) {
    double dev = 0.0;
    for (unsigned int b = 0; b < gridDim.x; ++b) dev += __ldcg(P.objpart + b);
    double ng = 0.0, nu = 0.0;
    for (int64_t r = 0; r < P.R; ++r) {
      ng += __ldcg(P.blocksum + 2 * r);
      nu += __ldcg(P.blocksum + 2 * r + 1);
    }
    P.rec[R_DEV] = dev;
    P.rec[R_NGAM] = ng;
    P.rec[R_NU] = nu;
    P.rec[R_NB] = nb;
    P.rec[R_NV] = nv;
    *tk = 0u;
  }
}

// ---------------------------------------------------------------------------
// K2: tracker decision (optim.py:301-338), snapshot refresh, EMA + adaptive
// update of rows I and columns J (optim.py:450-462), NB shape update
// (optim.py:205-229, 469-473).  Every CTA computes the tracker decision from
// the immutable Ctrl + gathered records; the last CTA commits Ctrl.
// Grid: [row CTAs | column CTAs | snapshot CTAs].
// ---------------------------------------------------------------------------
struct Decision {
  double obj;
  int boundary, snap, stop, conv, div, div_init, streak;
};

GMF_D const double* rec_of(const Params& P, const unsigned char* gathered, int r) {
  return reinterpret_cast<const double*>(gathered + (int64_t)r * P.rec_stride);
}

GMF_D Decision decide(const Params& P, const Ctrl& C, const unsigned char* gathered) {
  Decision D;
  D.obj = 0.0;
  D.boundary = (C.t % P.S) == 0;
  D.snap = 0; D.stop = 0; D.conv = C.converged; D.div = 0; D.div_init = 0; D.streak = C.streak;
  if (D.boundary) {
    double dev = 0, ng = 0, nu = 0, nb = 0, nv = 0;
    for (int r = 0; r < P.world; ++r) {
      const double* rc = rec_of(P, gathered, r);
      dev += __ldcg(rc + R_DEV); ng += __ldcg(rc + R_NGAM); nu += __ldcg(rc + R_NU);
      nb = __ldcg(rc + R_NB); nv = __ldcg(rc + R_NV);   // replicated column state
    }
    D.obj = P.escale * dev / (2.0 * P.phi) +
            0.5 * (P.lam_b * nb + P.lam_g * ng + P.lam_u * nu + P.lam_v * nv);
    if (C.t == 0) {
      if (!isfinite(D.obj)) { D.div_init = 1; D.stop = 1; }
      else D.snap = 1;
    } else if (!isfinite(D.obj)) {
      D.div = 1; D.stop = 1;
    } else {
      if ((C.trace_len + 1) % P.snap_stride == 0) D.snap = 1;
      const double rel = fabs(D.obj - C.last_obj) / (fabs(C.last_obj) + 1e-12);
      D.streak = rel < P.tol ? D.streak + 1 : 0;
      if (D.streak >= 2) { D.conv = 1; D.stop = 1; }
    }
  }
  if (C.t >= P.max_steps) D.stop = 1;
  return D;
}

template <typename T>
__global__ void __launch_bounds__(kThreads) k_apply(Params P, const unsigned char* gathered) {
  __shared__ double scr[kThreads / 32];
  const Ctrl C = *P.ctrl;
  if (C.stopped) return;
  if (!gathered) gathered = reinterpret_cast<const unsigned char*>(P.rec);
  const Decision D = decide(P, C, gathered);
  const bool upd = !D.stop;
  const long long t = C.t;
  const int64_t blk = upd ? P.bseq[t] : -1;
  const int64_t sidx = t % P.S;
  const double rho = upd ? P.rho_tab[t] : 0.0;
  const double at = upd ? P.alpt_tab[t] : 0.0;
  const int Kr = P.Kr, Kc = P.Kc;
  const int bx = blockIdx.x;
  double ng = 0.0, nu = 0.0;

  if (bx < P.n_row_ctas) {
    // ---------------- rows of block I ----------------
    if (blk >= 0) {
      const int64_t r0 = P.rbp[blk], nI = P.rbp[blk + 1] - r0;
      const int64_t e = (int64_t)bx * kThreads + threadIdx.x;
      if (e < nI * Kr) {
        const int64_t il = e / Kr;
        const int k = (int)(e % Kr);
        const int64_t i = r0 + il;
        T* th = tptr<T>(P.th_row) + i * Kr + k;
        const T old = *th;
        if (D.snap) tptr<T>(P.sn_row)[i * Kr + k] = old;
        const int64_t nJ = P.cbp[sidx + 1] - P.cbp[sidx];
        const double s_row = (double)P.m / (double)nJ;
        const T* rp = tptr<T>(P.rowpart);
        T gs = T(0), hs = T(0);
        for (int ct = 0; ct < P.CT; ++ct) {
          const T* src = rp + ((int64_t)ct * P.nstar_max + il) * (2 * Kr);
          gs += src[k];
          hs += src[Kr + k];
        }
        const T lam = T(k < P.q ? P.lam_g : P.lam_u);
        const T G = T(s_row) * gs + lam * old;
        const T H = T(s_row) * hs + lam;
        T* gb = tptr<T>(P.gb_row) + i * Kr + k;
        T* hb = tptr<T>(P.hb_row) + i * Kr + k;
        const T gn = (T(1) - T(P.a1)) * *gb + T(P.a1) * G;
        const T hn = (T(1) - T(P.a2)) * *hb + T(P.a2) * H;
        *gb = gn;
        *hb = hn;
        const T delta = -T(at) * gn / (hn + T(P.damp));
        const T nv = old + T(rho) * delta;
        *th = nv;
        const double sq = (double)nv * (double)nv;
        if (k < P.q) ng = sq; else nu = sq;
      }
    } else if (D.snap) {
      // no update this step; dirty rows are copied by the snapshot CTAs
    }
    ng = block_sum<kThreads>(ng, scr);
    nu = block_sum<kThreads>(nu, scr);
    if (threadIdx.x == 0) { P.rnpart[2 * bx] = ng; P.rnpart[2 * bx + 1] = nu; }
  } else if (bx < P.n_row_ctas + P.n_col_ctas) {
    // ---------------- columns (all m; update only J) ----------------
    const int64_t e = (int64_t)(bx - P.n_row_ctas) * kThreads + threadIdx.x;
    if (e < P.m * Kc) {
      const int64_t j = e / Kc;
      const int k = (int)(e % Kc);
      T* th = tptr<T>(P.th_col) + j * Kc + k;
      const T old = *th;
      if (D.snap) tptr<T>(P.sn_col)[j * Kc + k] = old;
      int64_t pos = -1;
      if (blk >= 0) {
        if (P.col_identity) pos = j;
        else if (P.cbof[j] == sidx) pos = P.cpos[j];
      }
      if (pos >= 0) {
        const double s_col = P.rbscale[blk];
        T gs = T(0), hs = T(0);
        for (int r = 0; r < P.world; ++r) {
          const T* cp = reinterpret_cast<const T*>(rec_of(P, gathered, r) + REC_HDR) + pos * (2 * Kc);
          gs += cp[k];
          hs += cp[Kc + k];
        }
        const T lam = T(k < P.p ? P.lam_b : P.lam_v);
        const T G = T(s_col) * gs + lam * old;
        const T H = T(s_col) * hs + lam;
        T* gb = tptr<T>(P.gb_col) + j * Kc + k;
        T* hb = tptr<T>(P.hb_col) + j * Kc + k;
        const T gn = (T(1) - T(P.a1)) * *gb + T(P.a1) * G;
        const T hn = (T(1) - T(P.a2)) * *hb + T(P.a2) * H;
        *gb = gn;
        *hb = hn;
        const T delta = -T(at) * gn / (hn + T(P.damp));
        *th = old + T(rho) * delta;
      }
    }
  } else if (D.snap) {
    // ---------------- snapshot of dirty row blocks other than I ----------------
    const int sc = bx - P.n_row_ctas - P.n_col_ctas;
    const int nsc = gridDim.x - P.n_row_ctas - P.n_col_ctas;
    const T* src = tptr<T>(P.th_row);
    T* dst = tptr<T>(P.sn_row);
    for (int64_t r = 0; r < P.R; ++r) {
      if (r == blk || P.last_mod[r] < C.last_snap_t) continue;
      const int64_t a = P.rbp[r] * Kr, b = P.rbp[r + 1] * Kr;
      for (int64_t e = a + (int64_t)sc * kThreads + threadIdx.x; e < b;
           e += (int64_t)nsc * kThreads)
        dst[e] = src[e];
    }
  }

  // ---------------- commit (last CTA) ----------------
  unsigned int* tk = P.tickets + 2 * P.CT + 2;
  if (!last_block_ticket(tk, gridDim.x)) return;
  if (threadIdx.x != 0) return;
  Ctrl N = C;
  if (D.boundary) {
    P.trace_obj[C.trace_len] = D.obj;
    P.trace_nb[C.trace_len] = C.nb_shape;
    N.trace_len = C.trace_len + 1;
    N.last_obj = D.obj;
    N.streak = D.streak;
    N.converged = D.conv;
    N.diverged = D.div;
    N.diverged_init = D.div_init;
  }
  if (D.snap) {
    N.last_snap_t = t;
    N.snapshot_trace_len = N.trace_len;
  }
  if (upd) {
    if (P.est_alpha) {
      double num = 0.0, den = 0.0;
      for (int r = 0; r < P.world; ++r) {
        const double* rc = rec_of(P, gathered, r);
        num += __ldcg(rc + R_NBNUM);
        den += __ldcg(rc + R_NBDEN);
      }
      double ah = den > 0.0 ? num / den : P.nbceil;
      ah = fmin(fmax(P.nbfloor, ah), P.nbceil);
      N.nb_shape = (1.0 - rho) * C.nb_shape + rho * ah;
    }
    double g2 = 0.0, u2 = 0.0;
    for (int b = 0; b < P.n_row_ctas; ++b) {
      g2 += __ldcg(P.rnpart + 2 * b);
      u2 += __ldcg(P.rnpart + 2 * b + 1);
    }
    P.blocksum[2 * blk] = g2;
    P.blocksum[2 * blk + 1] = u2;
    P.last_mod[blk] = t;
    N.t = t + 1;
  }
  N.stopped = D.stop;
  *P.ctrl = N;
  *tk = 0u;
}

// per-block squared row norms (gamma part, u part), one CTA per block
template <typename T>
__global__ void __launch_bounds__(kThreads) k_blocknorm(Params P) {
  __shared__ double scr[kThreads / 32];
  const int64_t r = blockIdx.x;
  const T* th = tptr<T>(P.th_row);
  const int64_t a = P.rbp[r] * P.Kr, b = P.rbp[r + 1] * P.Kr;
  double ng = 0.0, nu = 0.0;
  for (int64_t e = a + threadIdx.x; e < b; e += kThreads) {
    const double v = (double)th[e];
    if ((int)(e % P.Kr) < P.q) ng += v * v; else nu += v * v;
  }
  ng = block_sum<kThreads>(ng, scr);
  nu = block_sum<kThreads>(nu, scr);
  if (threadIdx.x == 0) { P.blocksum[2 * r] = ng; P.blocksum[2 * r + 1] = nu; }
}

// standalone gradient outputs (gradients.py:109-112) from the K1 partials
template <typename T>
__global__ void __launch_bounds__(kThreads) k_gradout(Params P, long long blk, long long sidx,
                                                     T* g_row, T* h_row, T* g_col, T* h_col,
                                                     double* nb_sums) {
  const int Kr = P.Kr, Kc = P.Kc;
  const int64_t r0 = P.rbp[blk], nI = P.rbp[blk + 1] - r0;
  const int64_t j0 = P.cbp[sidx], nJ = P.cbp[sidx + 1] - j0;
  const double s_row = (double)P.m / (double)nJ;
  const double s_col = P.rbscale[blk];
  const int64_t e = blockIdx.x * (int64_t)kThreads + threadIdx.x;
  const int64_t nr = nI * Kr;
  if (e < nr) {
    const int64_t il = e / Kr;
    const int k = (int)(e % Kr);
    const T* rp = tptr<T>(P.rowpart);
    T gs = T(0), hs = T(0);
    for (int ct = 0; ct < P.CT; ++ct) {
      const T* src = rp + ((int64_t)ct * P.nstar_max + il) * (2 * Kr);
      gs += src[k];
      hs += src[Kr + k];
    }
    const T lam = T(k < P.q ? P.lam_g : P.lam_u);
    g_row[e] = T(s_row) * gs + lam * tptr<T>(P.th_row)[(r0 + il) * Kr + k];
    h_row[e] = T(s_row) * hs + lam;
  } else if (e < nr + nJ * Kc) {
    const int64_t f = e - nr;
    const int64_t pos = f / Kc;
    const int k = (int)(f % Kc);
    const int64_t j = P.col_identity ? pos : (int64_t)P.cidx[j0 + pos];
    const T* cp = reinterpret_cast<const T*>(P.rec + REC_HDR) + pos * (2 * Kc);
    const T lam = T(k < P.p ? P.lam_b : P.lam_v);
    g_col[f] = T(s_col) * cp[k] + lam * tptr<T>(P.th_col)[j * Kc + k];
    h_col[f] = T(s_col) * cp[Kc + k] + lam;
  }
  if (e == 0 && nb_sums) {
    nb_sums[0] = P.rec[R_NBNUM];
    nb_sums[1] = P.rec[R_NBDEN];
  }
}

// full deviance over all local entries (model.py:268-276): warp per row
template <typename T>
__global__ void __launch_bounds__(kThreads) k_objfull(Params P, double alpha, double* part,
                                                      unsigned int* ticket, double* out) {
  __shared__ double scr[kThreads / 32];
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * (int64_t)kThreads + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * kThreads) >> 5;
  const T* wg = tptr<T>(P.w);
  double s = 0.0;
  for (int64_t i = gw; i < P.n; i += nw) {
    if (P.yfmt == GMF_Y_DENSE_I32) {
      for (int64_t j = lane; j < P.m; j += 32) {
        const double mu = exp(eta_at<T>(P, i, j));
        const double w = P.has_w ? (double)wg[i * P.m + j] : 1.0;
        s += w * unit_deviance(P.fam, (double)P.y[i * P.m + j], mu, alpha);
      }
    } else {
      // zeros everywhere, corrected at the stored nonzeros
      for (int64_t j = lane; j < P.m; j += 32)
        s += unit_deviance(P.fam, 0.0, exp(eta_at<T>(P, i, j)), alpha);
      for (int64_t k = P.rp[i] + lane; k < P.rp[i + 1]; k += 32) {
        const int64_t j = P.ci[k];
        const double mu = exp(eta_at<T>(P, i, j));
        s += unit_deviance(P.fam, (double)P.cv[k], mu, alpha) - unit_deviance(P.fam, 0.0, mu, alpha);
      }
    }
  }
  s = block_sum<kThreads>(s, scr);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
  if (last_block_ticket(ticket, gridDim.x)) {
    if (threadIdx.x == 0) {
      double tot = 0.0;
      for (unsigned int b = 0; b < gridDim.x; ++b) tot += __ldcg(part + b);
      *out = tot;
      *ticket = 0u;
    }
  }
}

// ---------------------------------------------------------------------------
// host launchers
// ---------------------------------------------------------------------------
int launch_obj(const Params& P, int dtype, cudaStream_t st) {
  if (dtype == GMF_F64) k_obj<double><<<P.n_obj_ctas, kThreads, 0, st>>>(P);
  else k_obj<float><<<P.n_obj_ctas, kThreads, 0, st>>>(P);
  GMF_LAUNCH_CHECK("k_obj");
  return GMF_OK;
}

int launch_apply(const Params& P, int dtype, const void* gathered, cudaStream_t st) {
  const int grid = P.n_row_ctas + P.n_col_ctas + kSnapCtas;
  const unsigned char* g = reinterpret_cast<const unsigned char*>(gathered);
  if (dtype == GMF_F64) k_apply<double><<<grid, kThreads, 0, st>>>(P, g);
  else k_apply<float><<<grid, kThreads, 0, st>>>(P, g);
  GMF_LAUNCH_CHECK("k_apply");
  return GMF_OK;
}

int launch_blocknorm(const Params& P, int dtype, cudaStream_t st) {
  if (P.R <= 0) return GMF_OK;
  if (dtype == GMF_F64) k_blocknorm<double><<<(unsigned)P.R, kThreads, 0, st>>>(P);
  else k_blocknorm<float><<<(unsigned)P.R, kThreads, 0, st>>>(P);
  GMF_LAUNCH_CHECK("k_blocknorm");
  return GMF_OK;
}

int launch_gradout(const Params& P, int dtype, long long blk, long long sidx, int64_t nI,
                   int64_t nJ, void* g_row, void* h_row, void* g_col, void* h_col,
                   double* nb_sums, cudaStream_t st) {
  const int64_t tot = nI * P.Kr + nJ * P.Kc;
  const int grid = (int)((tot + kThreads - 1) / kThreads) > 0 ? (int)((tot + kThreads - 1) / kThreads) : 1;
  if (dtype == GMF_F64)
    k_gradout<double><<<grid, kThreads, 0, st>>>(P, blk, sidx, (double*)g_row, (double*)h_row,
                                                 (double*)g_col, (double*)h_col, nb_sums);
  else
    k_gradout<float><<<grid, kThreads, 0, st>>>(P, blk, sidx, (float*)g_row, (float*)h_row,
                                                (float*)g_col, (float*)h_col, nb_sums);
  GMF_LAUNCH_CHECK("k_gradout");
  return GMF_OK;
}

int launch_objfull(const Params& P, int dtype, double alpha, double* part, unsigned int* ticket,
                   double* out, cudaStream_t st) {
  const int grid = 2 * kSMs;
  if (dtype == GMF_F64) k_objfull<double><<<grid, kThreads, 0, st>>>(P, alpha, part, ticket, out);
  else k_objfull<float><<<grid, kThreads, 0, st>>>(P, alpha, part, ticket, out);
  GMF_LAUNCH_CHECK("k_objfull");
  return GMF_OK;
}

}  // namespace gmf
