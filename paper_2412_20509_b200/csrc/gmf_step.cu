// Per-step kernels of the multi-rank path -- K3 (tracked objective) and K2
// (tracker + EMA/adaptive update + NB shape) -- plus helper kernels.  The
// single-rank path runs the same bodies inside the persistent k_fit.
#include "gmf_kern.cuh"

namespace gmf {

// ---------------------------------------------------------------------------
// K3: tracked objective of the current state at epoch boundaries
// (optim.py:283-290).  The last CTA folds the partials, the per-block row
// norms and the column norms into the rank record.  It also folds the row
// norms of the block updated by the previous k_apply (rnpart) into blocksum.
// ---------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(kThreads) k_obj(Params P) {
  __shared__ double scr[kThreads / 32];
  const Ctrl* C = P.ctrl;
  if (C->stopped || (C->t % P.S) != 0) return;
  obj_partial<T>(P, C->nb_shape, blockIdx.x, gridDim.x, P.objpart + OBJ_W * blockIdx.x);
  unsigned int* tk = P.tickets + 2 * P.CT + 1;
  if (!last_block_ticket(tk, gridDim.x)) return;
  const double dev = sum_parts<kThreads>(P.objpart + 0, gridDim.x, OBJ_W, scr);
  const double nb = sum_parts<kThreads>(P.objpart + 1, gridDim.x, OBJ_W, scr);
  const double nv = sum_parts<kThreads>(P.objpart + 2, gridDim.x, OBJ_W, scr);
  const double ng = sum_parts<kThreads>(P.blocksum + 0, P.R, 2, scr);
  const double nu = sum_parts<kThreads>(P.blocksum + 1, P.R, 2, scr);
  if (threadIdx.x == 0) {
    P.rec[R_DEV] = dev;
    P.rec[R_NGAM] = ng;
    P.rec[R_NU] = nu;
    P.rec[R_NB] = nb;
    P.rec[R_NV] = nv;
    *tk = 0u;
  }
}

GMF_D const double* rec_of(const Params& P, const unsigned char* gathered, int r) {
  return reinterpret_cast<const double*>(gathered + (int64_t)r * P.rec_stride);
}

// ---------------------------------------------------------------------------
// K2: every CTA computes the tracker decision from the gathered records of
// all ranks (immutable during the kernel); the last CTA commits Ctrl.
// Grid: [row CTAs | column CTAs | snapshot CTAs].
// ---------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(kThreads) k_apply(Params P, const unsigned char* gathered) {
  __shared__ double scr[kThreads / 32];
  const Ctrl C = *P.ctrl;
  if (C.stopped) return;
  if (!gathered) gathered = reinterpret_cast<const unsigned char*>(P.rec);
  double dev = 0, ng = 0, nu = 0, nb = 0, nv = 0, nbn = 0, nbd = 0;
  for (int r = 0; r < P.world; ++r) {
    const double* rc = rec_of(P, gathered, r);
    dev += __ldcg(rc + R_DEV); ng += __ldcg(rc + R_NGAM); nu += __ldcg(rc + R_NU);
    nb = __ldcg(rc + R_NB); nv = __ldcg(rc + R_NV);   // replicated column state
    nbn += __ldcg(rc + R_NBNUM); nbd += __ldcg(rc + R_NBDEN);
  }
  const Decision D = decide_from(P, C, dev, ng, nu, nb, nv);
  const bool upd = !D.stop;
  const long long t = C.t;
  const int64_t blk = upd ? P.bseq[t] : -1;
  const int64_t sidx = t % P.S;
  const double rho = upd ? P.rho_tab[t] : 0.0;
  const double at = upd ? P.alpt_tab[t] : 0.0;
  const int Kr = P.Kr, Kc = P.Kc;
  const int bx = blockIdx.x;
  // copy-on-write snapshot: save block I's rows on its first update after a
  // snapshot point (snap_ver is written only by the committing last CTA)
  const long long per_now = C.snap_period + (D.snap ? 1 : 0);
  const bool cow = upd && P.snap_ver[blk >= 0 ? blk : 0] != per_now;

  if (bx < P.n_row_ctas) {
    double rg = 0.0, ru = 0.0;
    if (blk >= 0) {
      const int64_t r0 = P.rbp[blk], nI = P.rbp[blk + 1] - r0;
      const int64_t e = (int64_t)bx * kThreads + threadIdx.x;
      if (e < nI * Kr) {
        const int64_t il = e / Kr;
        const int k = (int)(e % Kr);
        const int64_t i = r0 + il;
        T* th = tptr<T>(P.th_row) + i * Kr + k;
        if (cow) tptr<T>(P.sn_row)[i * Kr + k] = *th;
        const int64_t nJ = P.cbp[sidx + 1] - P.cbp[sidx];
        T gs, hs;
        rowpart_sum<T>(P, il, k, gs, hs);
        const T nvv = ema_update<T>(P, th, tptr<T>(P.gb_row) + i * Kr + k,
                                    tptr<T>(P.hb_row) + i * Kr + k, gs, hs,
                                    (double)P.m / (double)nJ, k < P.q ? P.lam_g : P.lam_u, rho, at);
        const double sq = (double)nvv * (double)nvv;
        if (k < P.q) rg = sq; else ru = sq;
      }
    }
    rg = block_sum<kThreads>(rg, scr);
    ru = block_sum<kThreads>(ru, scr);
    if (threadIdx.x == 0) { P.rnpart[2 * bx] = rg; P.rnpart[2 * bx + 1] = ru; }
  } else if (bx < P.n_row_ctas + P.n_col_ctas) {
    const int64_t e = (int64_t)(bx - P.n_row_ctas) * kThreads + threadIdx.x;
    if (e < P.m * Kc) {
      const int64_t j = e / Kc;
      const int k = (int)(e % Kc);
      T* th = tptr<T>(P.th_col) + j * Kc + k;
      if (D.snap) tptr<T>(P.sn_col)[j * Kc + k] = *th;
      int64_t pos = -1;
      if (blk >= 0) {
        if (P.col_identity) pos = j;
        else if (P.cbof[j] == sidx) pos = P.cpos[j];
      }
      if (pos >= 0) {
        T gs = T(0), hs = T(0);
        for (int r = 0; r < P.world; ++r) {
          const T* cp = reinterpret_cast<const T*>(rec_of(P, gathered, r) + REC_HDR) + pos * (2 * Kc);
          gs += ldcg_t<T>(cp + k);
          hs += ldcg_t<T>(cp + Kc + k);
        }
        ema_update<T>(P, th, tptr<T>(P.gb_col) + j * Kc + k, tptr<T>(P.hb_col) + j * Kc + k, gs, hs,
                      P.rbscale[blk], k < P.p ? P.lam_b : P.lam_v, rho, at);
      }
    }
  }

  // ---------------- commit (last CTA) ----------------
  unsigned int* tk = P.tickets + 2 * P.CT + 2;
  if (!last_block_ticket(tk, gridDim.x)) return;
  double g2 = 0.0, u2 = 0.0;
  if (upd) {
    g2 = sum_parts<kThreads>(P.rnpart, P.n_row_ctas, 2, scr);
    u2 = sum_parts<kThreads>(P.rnpart + 1, P.n_row_ctas, 2, scr);
  }
  if (threadIdx.x != 0) return;
  if (D.boundary) {
    P.trace_obj[C.trace_len] = D.obj;
    P.trace_nb[C.trace_len] = C.nb_shape;
  }
  if (upd) {
    P.blocksum[2 * blk] = g2;
    P.blocksum[2 * blk + 1] = u2;
    if (cow) P.snap_ver[blk] = per_now;
  }
  *P.ctrl = advance(P, C, D, nbn, nbd);
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

// tracked entries packed (row, col, Y, 0), built once per fit (the sample is fixed)
__global__ void __launch_bounds__(kThreads) k_eval_pack(Params P, int4* out) {
  for (int64_t e = blockIdx.x * (int64_t)kThreads + threadIdx.x; e < P.E;
       e += (int64_t)gridDim.x * kThreads) {
    const int64_t i = P.erow[e], j = P.ecol[e];
    out[e] = make_int4((int)i, (int)j, (int)y_lookup(P, i, j), P.eslot ? P.eslot[e] : 0);
  }
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
    T gs, hs;
    rowpart_sum<T>(P, il, k, gs, hs);
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
        const int64_t j = csr_col_at(P, k);
        const double mu = exp(eta_at<T>(P, i, j));
        s += unit_deviance(P.fam, (double)csr_val_at(P, k), mu, alpha) - unit_deviance(P.fam, 0.0, mu, alpha);
      }
    }
  }
  s = block_sum<kThreads>(s, scr);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
  if (last_block_ticket(ticket, gridDim.x)) {
    const double tot = sum_parts<kThreads>(part, gridDim.x, 1, scr);
    if (threadIdx.x == 0) {
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
  const int grid = P.n_row_ctas + P.n_col_ctas;
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

int launch_eval_pack(const Params& P, int4* out, cudaStream_t st) {
  if (P.E <= 0) return GMF_OK;
  int64_t b = (P.E + kThreads - 1) / kThreads;
  if (b > 4 * kSMs) b = 4 * kSMs;
  k_eval_pack<<<(unsigned)b, kThreads, 0, st>>>(P, out);
  GMF_LAUNCH_CHECK("k_eval_pack");
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
