// Per-step kernels of the multi-rank path -- K3 (tracked objective) and K2
// (tracker + EMA/adaptive update + NB shape) -- plus helper kernels.  The
// single-rank path runs the same bodies inside the persistent k_fit.
#include <type_traits>

#include <vector>

#include "gmf_kern.cuh"

namespace gmf {

// ---------------------------------------------------------------------------
// K3: tracked objective of the current state at epoch boundaries
// (optim.py:283-290).  The last CTA folds the partials, the per-block row
// norms and the column norms into the rank record.  It also folds the row
// norms of the block updated by the previous k_apply (rnpart) into blocksum.
// ---------------------------------------------------------------------------
// ---- tracked-objective caches for the per-step path (bucket NK known at
// run time; the persistent kernel's compile-time versions are in gmf_grad.cu)
template <typename T>
GMF_D void ecache_fill_rt(const Params& P, int64_t slot, int64_t i) {
  const int NKr = P.nkb;
  T* row = tptr<T>(P.ecache) + slot * (NKr + 4);
  const T* th = tptr<T>(P.th_row) + i * P.Kr;
  const T* xg = tptr<T>(P.x) + i * P.p;
  const int p = P.p, d = P.d, KA = P.KA, q = P.q;
  for (int k = 0; k < NKr; ++k) {
    T v = T(0);
    if (k < p) v = xg[k];
    else if (k < p + d) v = th[q + (k - p)];
    else if (k < KA) v = th[k - p - d];
    row[k] = v;
  }
  row[NKr] = P.has_off ? tptr<T>(P.off)[i] : T(0);
  row[NKr + 1] = T(0); row[NKr + 2] = T(0); row[NKr + 3] = T(0);
}

// every tracked row's slot and every column's padded [b | v | z] (gmf_reset)
template <typename T>
__global__ void __launch_bounds__(kThreads) k_cache_fill(Params P) {
  const int64_t g = (int64_t)blockIdx.x * kThreads + threadIdx.x, gs = (int64_t)gridDim.x * kThreads;
  for (int64_t sl = g; sl < P.nslots; sl += gs) ecache_fill_rt<T>(P, sl, P.srow[sl]);
  const T* tc = tptr<T>(P.th_col);
  const T* zg = tptr<T>(P.z);
  for (int64_t e = g; e < P.m * P.nkb; e += gs) {
    const int64_t j = e / P.nkb;
    const int k = (int)(e % P.nkb);
    T v = T(0);
    if (k < P.Kc) v = tc[j * P.Kc + k];
    else if (k < P.KA) v = zg[j * P.q + (k - P.Kc)];
    tptr<T>(P.vpad)[e] = v;
  }
}

// deviance of entry en from the caches: eta = a_slot . c_j (16-byte loads,
// all in flight; nkb <= 64 in passes of 32)
template <typename T>
GMF_D double entry_dev_cached(const Params& P, int4 en, double alpha) {
  using V = typename std::conditional<sizeof(T) == 4, float4, double2>::type;
  constexpr int VN = 16 / sizeof(T);
  constexpr int MAXV = 32 / VN;   // 32 features per pass (nkb <= 64: two passes)
  const int nv = P.nkb / VN;
  const V* a = reinterpret_cast<const V*>(tptr<T>(P.ecache) + (int64_t)en.w * (P.nkb + 4));
  const V* c = reinterpret_cast<const V*>(tptr<T>(P.vpad) + (int64_t)en.y * P.nkb);
  const T off = tptr<T>(P.ecache)[(int64_t)en.w * (P.nkb + 4) + P.nkb];
  double eta = (double)off;
  for (int v0 = 0; v0 < nv; v0 += MAXV) {
    V av[MAXV], cv[MAXV];
    #pragma unroll
    for (int u = 0; u < MAXV; ++u) {   // loads all in flight (clamped index)
      const int uu = v0 + u < nv ? v0 + u : 0;
      av[u] = a[uu];
      cv[u] = __ldcg(c + uu);
    }
    #pragma unroll
    for (int u = 0; u < MAXV; ++u) {
      if (v0 + u < nv) {
        const T* ap = reinterpret_cast<const T*>(&av[u]);
        const T* cp = reinterpret_cast<const T*>(&cv[u]);
        #pragma unroll
        for (int k = 0; k < VN; ++k) eta += (double)ap[k] * (double)cp[k];
      }
    }
  }
  const double wv = P.has_w ? (double)tptr<T>(P.w)[(int64_t)en.x * P.m + en.y] : 1.0;
  if (P.gen)   // general mode: real-valued response, any link
    return wv * unit_deviance(P.fam, (double)tptr<T>(P.y_work)[(int64_t)en.x * P.m + en.y],
                              gen_mean<double>(P.link, eta), alpha);
  if (sizeof(T) == 4)
    return wv * (double)unit_deviance_f(P.fam, (float)en.z, __expf((float)eta), (float)alpha);
  return wv * unit_deviance(P.fam, (double)en.z, exp(eta), alpha);
}

template <typename T>
__global__ void __launch_bounds__(kThreads) k_obj(Params P) {
  __shared__ double scr5[5 * (kThreads / 32)];
  const Ctrl* C = P.ctrl;
  if (C->stopped || (C->t % P.S) != 0) return;
  double dpart = 0.0;
  for (int64_t e = (int64_t)blockIdx.x * kThreads + threadIdx.x; e < P.E;
       e += (int64_t)gridDim.x * kThreads)
    dpart += entry_dev_cached<T>(P, P.ep[e], C->nb_shape);
  obj_partial<T>(P, C->nb_shape, blockIdx.x, gridDim.x, P.objpart + OBJ_W * blockIdx.x, dpart);
  unsigned int* tk = P.tickets + 2 * P.CT + 1;
  if (!last_block_ticket(tk, gridDim.x)) return;
  // one pass over all five partial arrays, one block reduction
  double v5[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
  for (int i = threadIdx.x; i < (int)gridDim.x; i += kThreads) {
    const double* op = P.objpart + (int64_t)OBJ_W * i;
    v5[0] += __ldcg(op); v5[1] += __ldcg(op + 1); v5[2] += __ldcg(op + 2);
  }
  for (int64_t i = threadIdx.x; i < P.R; i += kThreads) {
    v5[3] += __ldcg(P.blocksum + 2 * i); v5[4] += __ldcg(P.blocksum + 2 * i + 1);
  }
  block_sum_vec<5>(v5, scr5);
  const double dev = v5[0], nb = v5[1], nv = v5[2], ng = v5[3], nu = v5[4];
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
  __shared__ double scr2[2 * (kThreads / 32)];
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
        const int32_t sl = P.rslot[i];   // the objective cache slot of this row
        if (sl >= 0) tptr<T>(P.ecache)[(int64_t)sl * (P.nkb + 4) + (k < P.q ? P.p + P.d + k : P.p + (k - P.q))] = nvv;
        const double sq = (double)nvv * (double)nvv;
        if (k < P.q) rg = sq; else ru = sq;
      }
    }
    double v2[2] = {rg, ru};
    block_sum_vec<2>(v2, scr2);
    if (threadIdx.x == 0) { P.rnpart[2 * bx] = v2[0]; P.rnpart[2 * bx + 1] = v2[1]; }
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
        const T nvv = ema_update<T>(P, th, tptr<T>(P.gb_col) + j * Kc + k,
                                    tptr<T>(P.hb_col) + j * Kc + k, gs, hs, P.rbscale[blk],
                                    k < P.p ? P.lam_b : P.lam_v, rho, at);
        tptr<T>(P.vpad)[j * P.nkb + k] = nvv;   // the objective's padded [b | v | z]
      }
    }
  }

  // ---------------- commit (last CTA) ----------------
  unsigned int* tk = P.tickets + 2 * P.CT + 2;
  if (!last_block_ticket(tk, gridDim.x)) return;
  double g2 = 0.0, u2 = 0.0;
  if (upd) {
    double v2[2] = {0.0, 0.0};
    for (int i = threadIdx.x; i < P.n_row_ctas; i += kThreads) {
      v2[0] += __ldcg(P.rnpart + 2 * i); v2[1] += __ldcg(P.rnpart + 2 * i + 1);
    }
    block_sum_vec<2>(v2, scr2);
    g2 = v2[0]; u2 = v2[1];
  }
  if (threadIdx.x != 0) return;
  if (D.boundary) {
    P.trace_obj[C.trace_len] = D.obj;
    P.trace_nb[C.trace_len] = C.nb_shape;
    P.trace_phi[C.trace_len] = C.phi;
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
// ||Gamma_r||^2 and ||U_r||^2 of every row block r (the per-block sums the
// tracked objective's penalty is kept in): grid (segments, blocks), each CTA
// a fixed segment of kBnRows rows (a thread per row, no division per
// element), its partials reduced in fixed segment order by k_blocknorm_fin
constexpr int kBnRows = 2048;

template <typename T>
__global__ void __launch_bounds__(kThreads) k_blocknorm(Params P, double* part, int nseg) {
  __shared__ double scr[kThreads / 32];
  const int64_t r = blockIdx.y, sg = blockIdx.x;
  const T* th = tptr<T>(P.th_row);
  const int64_t r0 = P.rbp[r], r1 = P.rbp[r + 1];
  const int64_t lo = r0 + sg * kBnRows, hi = lo + kBnRows < r1 ? lo + kBnRows : r1;
  const int Kr = P.Kr, q = P.q;
  double ng = 0.0, nu = 0.0;
  for (int64_t i = lo + threadIdx.x; i < hi; i += kThreads) {
    const T* row = th + i * Kr;
    for (int k = 0; k < Kr; ++k) {
      const double v = (double)row[k];
      if (k < q) ng += v * v; else nu += v * v;
    }
  }
  ng = block_sum<kThreads>(ng, scr);
  nu = block_sum<kThreads>(nu, scr);
  if (threadIdx.x == 0) {
    part[2 * (r * nseg + sg)] = ng;
    part[2 * (r * nseg + sg) + 1] = nu;
  }
}

__global__ void __launch_bounds__(32) k_blocknorm_fin(Params P, const double* part, int nseg) {
  const int64_t r = blockIdx.x;
  const int64_t nrows = P.rbp[r + 1] - P.rbp[r];
  const int used = (int)((nrows + kBnRows - 1) / kBnRows);
  double ng = 0.0, nu = 0.0;
  for (int sg = threadIdx.x; sg < used; sg += 32) {
    ng += part[2 * (r * nseg + sg)];
    nu += part[2 * (r * nseg + sg) + 1];
  }
  #pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ng += __shfl_xor_sync(0xffffffffu, ng, o);
    nu += __shfl_xor_sync(0xffffffffu, nu, o);
  }
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

// NB part of -2 log-likelihood beyond D/phi for one entry with y > 0
// (select.py:57-78 _dispersion_constant: sat + y log y; zeros contribute 0)
GMF_D double nb_loglik_term(double y, double a) {
  const double sat = lgamma(y + a) - lgamma(a) - lgamma(y + 1.0) - (y + a) * log(y + a) +
                     a * log(a);
  return sat + y * log(y);
}

// unit deviance at eta: fp64 on the fp64 path; on the fp32 path the fp32
// transcendentals of the tracked objective (gmf_common.cuh unit_deviance_f),
// accumulated in fp64 by the caller
template <typename T>
GMF_D double dev_at(int fam, double y, double eta, double alpha) {
  if constexpr (std::is_same<T, float>::value)
    return (double)unit_deviance_f(fam, (float)y, __expf((float)eta), (float)alpha);
  else
    return unit_deviance(fam, y, exp(eta), alpha);
}

// D(0, mu) -- the all-zero grid of a CSR pass.  NB: -2 alpha log1p(-mu / (mu + alpha))
// = 2 alpha log1p(mu / alpha) (no division; also exact where mu >> alpha);
// Poisson: 2 mu.
template <typename T>
GMF_D double dev0_at(int fam, double eta, double alpha, double inv_alpha) {
  if constexpr (std::is_same<T, float>::value) {
    const float mu = __expf((float)eta);
    if (fam == GMF_NEG_BINOMIAL) return (double)(2.f * (float)alpha * log1pf(mu * (float)inv_alpha));
    return (double)(2.f * mu);
  } else {
    const double mu = exp(eta);
    if (fam == GMF_NEG_BINOMIAL) return 2.0 * alpha * log1p(mu * inv_alpha);
    return 2.0 * mu;
  }
}

// full deviance over all local entries (model.py:268-276), tiled: a CTA
// takes 32 rows x 64 columns at a time with the rows' [u | x | gamma] and
// the columns' [v | b | z] staged in shared memory as fp64 (stride S = K | 1
// doubles: odd, so 32 lanes reading 32 columns do not collide), and each
// thread forms a 4-row x 2-column register tile of predictors (6 shared
// loads per 8 FMAs instead of 2 global loads per FMA).  Dense Y is read
// coalesced along the columns; CSR rows are treated as all-zero over the
// grid and corrected at the row tile's stored nonzeros (one contiguous
// range).  With `with_const` (NB only) the same pass also sums the
// dispersion constant of select.py:71-78 -> out[1] = -2 sum w (sat + y log y).
constexpr int kFullRows = 32, kFullCols = 64;

GMF_HD int full_stride(int K) { return K | 1; }
GMF_HD int full_smem_bytes(int K) { return (kFullRows + kFullCols) * full_stride(K) * 8; }

template <typename T, bool GEN = false>
__global__ void __launch_bounds__(kThreads) k_objfull(Params P, double alpha, int with_const,
                                                      double* part, unsigned int* ticket,
                                                      double* out) {
  extern __shared__ double fsm[];
  __shared__ double scr[kThreads / 32];
  __shared__ double offs[kFullRows];
  __shared__ int64_t rps[kFullRows + 1];
  const int d = P.d, p = P.p, q = P.q, K = d + p + q, S = full_stride(K);
  double* Rs = fsm;                     // [kFullRows][S]: u | x | gamma
  double* Cs = fsm + kFullRows * S;     // [kFullCols][S]: v | b | z
  const T* tr = tptr<T>(P.th_row);
  const T* tc = tptr<T>(P.th_col);
  const T* xg = tptr<T>(P.x);
  const T* zg = tptr<T>(P.z);
  const T* og = tptr<T>(P.off);
  const T* wg = tptr<T>(P.w);
  const bool dense = P.yfmt == GMF_Y_DENSE_I32;
  const double inv_alpha = 1.0 / alpha;
  const int lane = threadIdx.x & 31, rg = threadIdx.x >> 5;   // rows rg + 8r, columns lane, lane + 32
  double s = 0.0, c = 0.0;
  const int64_t ntiles = (P.n + kFullRows - 1) / kFullRows;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t i0 = t * kFullRows;
    const int nr = (int)min((int64_t)kFullRows, P.n - i0);
    __syncthreads();   // previous tile's readers are done with Rs / rps
    for (int e = threadIdx.x; e < nr * K; e += kThreads) {
      const int r = e / K, k = e - r * K;
      const int64_t i = i0 + r;
      double v;
      if (k < d) v = (double)tr[i * P.Kr + q + k];
      else if (k < d + p) v = (double)xg[i * p + (k - d)];
      else v = (double)tr[i * P.Kr + (k - d - p)];
      Rs[r * S + k] = v;
    }
    if (threadIdx.x < nr) offs[threadIdx.x] = P.has_off ? (double)og[i0 + threadIdx.x] : 0.0;
    if (!dense && threadIdx.x <= nr) rps[threadIdx.x] = P.rp[i0 + threadIdx.x];
    for (int64_t j0 = 0; j0 < P.m; j0 += kFullCols) {
      const int nc = (int)min((int64_t)kFullCols, P.m - j0);
      __syncthreads();
      for (int e = threadIdx.x; e < nc * K; e += kThreads) {
        const int cc = e / K, k = e - cc * K;
        const int64_t j = j0 + cc;
        double v;
        if (k < d) v = (double)tc[j * P.Kc + p + k];
        else if (k < d + p) v = (double)tc[j * P.Kc + (k - d)];
        else v = (double)zg[j * q + (k - d - p)];
        Cs[cc * S + k] = v;
      }
      __syncthreads();
      double acc[4][2];
#pragma unroll
      for (int r = 0; r < 4; ++r) acc[r][0] = acc[r][1] = 0.0;
      for (int k = 0; k < K; ++k) {
        const double c0 = Cs[lane * S + k], c1 = Cs[(lane + 32) * S + k];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const double a = Rs[(rg + 8 * r) * S + k];
          acc[r][0] = fma(a, c0, acc[r][0]);
          acc[r][1] = fma(a, c1, acc[r][1]);
        }
      }
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int rr = rg + 8 * r;
        if (rr >= nr) continue;
        const int64_t i = i0 + rr;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int cc = lane + 32 * h;
          if (cc >= nc) continue;
          const int64_t j = j0 + cc;
          const double eta = acc[r][h] + offs[rr];
          if constexpr (GEN) {   // general mode: real-valued response, any link
            const double w = P.has_w ? (double)wg[i * P.m + j] : 1.0;
            const T yt = tptr<T>(P.y_work)[i * P.m + j];
            // unobserved entries (last mantissa bit set) are not in the masked
            // deviance (model.py:268-276)
            if (!(P.holes && lsb_set(yt)))
              s += w * unit_deviance(P.fam, (double)yt, gen_mean<double>(P.link, eta), alpha);
          } else if (dense) {
            double w = P.has_w ? (double)wg[i * P.m + j] : 1.0;
            const double y = (double)P.y[i * P.m + j];
            // unobserved entries (negative working response) are not in the
            // masked deviance (model.py:268-276)
            if (P.holes && signbit(tptr<T>(P.y_work)[i * P.m + j])) w = 0.0;
            s += w * dev_at<T>(P.fam, y, eta, alpha);
            if (with_const && y > 0.0) c += w * nb_loglik_term(y, alpha);
          } else {
            s += dev0_at<T>(P.fam, eta, alpha, inv_alpha);
          }
        }
      }
    }
    if (!dense) {
      const int64_t lo = rps[0], hi = rps[nr];
      for (int64_t k = lo + threadIdx.x; k < hi; k += kThreads) {
        int a = 0, b = nr - 1;        // the row r with rps[r] <= k < rps[r + 1]
        while (a < b) {
          const int mid = (a + b + 1) >> 1;
          if (rps[mid] <= k) a = mid; else b = mid - 1;
        }
        const double* R = Rs + a * S;
        const int64_t j = csr_col_at(P, k);
        double eta = 0.0;
        for (int kk = 0; kk < d; ++kk) eta = fma(R[kk], (double)tc[j * P.Kc + p + kk], eta);
        for (int kk = 0; kk < p; ++kk) eta = fma(R[d + kk], (double)tc[j * P.Kc + kk], eta);
        for (int kk = 0; kk < q; ++kk) eta = fma(R[d + p + kk], (double)zg[j * q + kk], eta);
        eta += offs[a];
        const double y = (double)csr_val_at(P, k);
        s += dev_at<T>(P.fam, y, eta, alpha) - dev0_at<T>(P.fam, eta, alpha, inv_alpha);
        if (with_const && y > 0.0) c += nb_loglik_term(y, alpha);
      }
    }
  }
  s = block_sum<kThreads>(s, scr);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
  if (with_const) {
    c = block_sum<kThreads>(c, scr);
    if (threadIdx.x == 0) part[gridDim.x + blockIdx.x] = c;
  }
  if (last_block_ticket(ticket, gridDim.x)) {
    const double tot = sum_parts<kThreads>(part, gridDim.x, 1, scr);
    __syncthreads();
    const double ctot = with_const ? sum_parts<kThreads>(part + gridDim.x, gridDim.x, 1, scr) : 0.0;
    if (threadIdx.x == 0) {
      out[0] = tot;
      if (with_const) out[1] = -2.0 * ctot;
      *ticket = 0u;
    }
  }
}

// Held-out scoring at listed entries (select.py:141-145 _mu_at, then
// metrics.py:35-55): mu = exp(eta) at (rows[k], cols[k]) -- rows in the
// handle's local (block-major) numbering -- optionally stored, and with y
// the four sums of rel_deviance / rel_log_rmse (unit prior weights):
// out = [sum D(y, mu), sum D(y, ybar), sum log^2((1+y)/(1+mu)), sum log^2((1+y)/(1+ybar))].
GMF_D void score_entry(int fam, double y, double mu, double ybar, double alpha, double* s) {
  s[0] += unit_deviance(fam, y, mu, alpha);
  s[1] += unit_deviance(fam, y, ybar, alpha);
  const double a = log((1.0 + y) / (1.0 + mu)), b = log((1.0 + y) / (1.0 + ybar));
  s[2] += a * a;
  s[3] += b * b;
}

template <int NT>
GMF_D void publish4(const double* s, double* part, unsigned int* ticket, double* out, double* scr) {
  for (int c = 0; c < 4; ++c) {
    const double t = block_sum<NT>(s[c], scr);
    if (threadIdx.x == 0) part[c * gridDim.x + blockIdx.x] = t;
  }
  if (last_block_ticket(ticket, gridDim.x)) {
    for (int c = 0; c < 4; ++c) {
      __syncthreads();
      const double tot = sum_parts<NT>(part + c * gridDim.x, gridDim.x, 1, scr);
      if (threadIdx.x == 0) out[c] = tot;
    }
    if (threadIdx.x == 0) *ticket = 0u;
  }
}

template <typename T>
__global__ void __launch_bounds__(kThreads) k_entries(Params P, double alpha, const int64_t* rows,
                                                      const int32_t* cols, const double* y,
                                                      int64_t n, double ybar, double* mu_out,
                                                      double* part, unsigned int* ticket,
                                                      double* out) {
  __shared__ double scr[kThreads / 32];
  double s[4] = {0.0, 0.0, 0.0, 0.0};
  for (int64_t k = blockIdx.x * (int64_t)kThreads + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * kThreads) {
    const double mu = gen_mean<double>(P.link, eta_at<T>(P, rows[k], cols[k]));
    if (mu_out) mu_out[k] = mu;
    if (out) score_entry(P.fam, y[k], mu, ybar, alpha, s);
  }
  if (out) publish4<kThreads>(s, part, ticket, out, scr);
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

int blocknorm_segments(int64_t nstar_max) {
  const int64_t s = (nstar_max + kBnRows - 1) / kBnRows;
  return (int)(s > 0 ? s : 1);
}

int launch_blocknorm(const Params& P, int dtype, cudaStream_t st) {
  if (P.R <= 0) return GMF_OK;
  const int nseg = blocknorm_segments(P.nstar_max);
  const dim3 grid((unsigned)nseg, (unsigned)P.R);
  if (dtype == GMF_F64) k_blocknorm<double><<<grid, kThreads, 0, st>>>(P, P.bnpart, nseg);
  else k_blocknorm<float><<<grid, kThreads, 0, st>>>(P, P.bnpart, nseg);
  GMF_LAUNCH_CHECK("k_blocknorm");
  k_blocknorm_fin<<<(unsigned)P.R, 32, 0, st>>>(P, P.bnpart, nseg);
  GMF_LAUNCH_CHECK("k_blocknorm_fin");
  return GMF_OK;
}

// Per-row tile index of a column-sorted CSR (J = all columns): thread per
// (row, tile boundary ct): the number of the row's nonzeros with column
// < ct * TC (lower bound); the ct = 0 thread also checks that the row's
// columns increase, else flags the index unusable.
__global__ void __launch_bounds__(kThreads) k_tile_index(Params P, int32_t* tidx,
                                                           unsigned int* unsorted) {
  const int CT1 = P.CT + 1;
  const int64_t total = P.n * CT1;
  for (int64_t g = (int64_t)blockIdx.x * kThreads + threadIdx.x; g < total;
       g += (int64_t)gridDim.x * kThreads) {
    const int64_t i = g / CT1;
    const int ct = (int)(g - i * CT1);
    const int64_t lo = P.rp[i], hi = P.rp[i + 1];
    const int64_t bound = (int64_t)ct * P.TC;
    int64_t a = lo, b = hi;   // first k in [lo, hi) with col >= bound
    while (a < b) {
      const int64_t mid = (a + b) >> 1;
      if (csr_col_at(P, mid) < bound) a = mid + 1; else b = mid;
    }
    tidx[g] = (int32_t)((ct == P.CT ? hi : a) - lo);
    if (ct == 0)
      for (int64_t k = lo + 1; k < hi; ++k)
        if (csr_col_at(P, k) <= csr_col_at(P, k - 1)) { atomicOr(unsorted, 1u); break; }
  }
}

// tile-CSR for K1 v2: the nonzeros of column tile ct (TC columns) of every
// row, tile-major, each carrying its row: (row, count << 8 | column - ct TC).
// lens[ct][i] = nonzeros of row i in tile ct (from the tile index)
__global__ void __launch_bounds__(kThreads) k_tcsr_len(Params P, const int32_t* tidx, int32_t* lens) {
  const int CT1 = P.CT + 1;
  for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < P.n; i += (int64_t)gridDim.x * kThreads)
    for (int ct = 0; ct < P.CT; ++ct) lens[(int64_t)ct * P.n + i] = tidx[i * CT1 + ct + 1] - tidx[i * CT1 + ct];
}

__global__ void __launch_bounds__(kThreads) k_tcsr_fill(Params P, const int32_t* tidx, const int64_t* tptr,
                                                          int32_t* tent, unsigned int* too_big) {
  const int CT1 = P.CT + 1;
  for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < P.n; i += (int64_t)gridDim.x * kThreads) {
    const int64_t k0 = P.rp[i];
    for (int ct = 0; ct < P.CT; ++ct) {
      const int64_t base = tptr[(int64_t)ct * (P.n + 1) + i];
      const int a = tidx[i * CT1 + ct], b = tidx[i * CT1 + ct + 1];
      for (int k = a; k < b; ++k) {
        const int col = csr_col_at(P, k0 + k), val = csr_val_at(P, k0 + k);
        if (val >= (1 << 23)) atomicOr(too_big, 1u);
        tent[2 * (base + k - a)] = (int32_t)i;
        tent[2 * (base + k - a) + 1] = (int32_t)(((uint32_t)val << 8) | (uint32_t)(col - ct * P.TC));
      }
    }
  }
}

int launch_tcsr(const Params& P, const int32_t* tidx, int32_t* lens, int64_t* tptr, int32_t* tent,
                unsigned int* too_big, cudaStream_t st) {
  const unsigned b = (unsigned)((P.n + kThreads - 1) / kThreads < 4096 ? (P.n + kThreads - 1) / kThreads : 4096);
  k_tcsr_len<<<b > 0 ? b : 1, kThreads, 0, st>>>(P, tidx, lens);
  GMF_LAUNCH_CHECK("k_tcsr_len");
  // exclusive scan in tile-major order on the host (once per handle)
  std::vector<int32_t> h((size_t)P.CT * P.n);
  GMF_CUDA(cudaMemcpyAsync(h.data(), lens, h.size() * 4, cudaMemcpyDeviceToHost, st));
  GMF_CUDA(cudaStreamSynchronize(st));
  std::vector<int64_t> tp((size_t)P.CT * (P.n + 1));
  int64_t run = 0;
  for (int ct = 0; ct < P.CT; ++ct) {
    for (int64_t i = 0; i < P.n; ++i) {
      tp[(size_t)ct * (P.n + 1) + i] = run;
      run += h[(size_t)ct * P.n + i];
    }
    tp[(size_t)ct * (P.n + 1) + P.n] = run;
  }
  GMF_CUDA(cudaMemcpyAsync(tptr, tp.data(), tp.size() * 8, cudaMemcpyHostToDevice, st));
  k_tcsr_fill<<<b > 0 ? b : 1, kThreads, 0, st>>>(P, tidx, tptr, tent, too_big);
  GMF_LAUNCH_CHECK("k_tcsr_fill");
  GMF_CUDA(cudaStreamSynchronize(st));
  return GMF_OK;
}

int launch_tile_index(const Params& P, int32_t* tidx, unsigned int* unsorted, cudaStream_t st) {
  const int64_t total = P.n * (P.CT + 1);
  unsigned b = (unsigned)((total + kThreads - 1) / kThreads);
  if (b > 8 * kSMs) b = 8 * kSMs;
  if (b < 1) b = 1;
  k_tile_index<<<b, kThreads, 0, st>>>(P, tidx, unsorted);
  GMF_LAUNCH_CHECK("k_tile_index");
  return GMF_OK;
}

int launch_cache_fill(const Params& P, int dtype, cudaStream_t st) {
  const int64_t work = P.nslots > P.m * P.nkb ? P.nslots : P.m * P.nkb;
  unsigned b = (unsigned)((work + kThreads - 1) / kThreads);
  if (b > 4 * kSMs) b = 4 * kSMs;
  if (b < 1) b = 1;
  if (dtype == GMF_F64) k_cache_fill<double><<<b, kThreads, 0, st>>>(P);
  else k_cache_fill<float><<<b, kThreads, 0, st>>>(P);
  GMF_LAUNCH_CHECK("k_cache_fill");
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

int launch_objfull(const Params& P, int dtype, double alpha, int with_const, double* part,
                   unsigned int* ticket, double* out, cudaStream_t st) {
  const int grid = 8 * kSMs;
  const int K = P.d + P.p + P.q;
  const int smem = full_smem_bytes(K);
  if (dtype == GMF_F64) {
    if (P.gen) {
      GMF_CUDA(cudaFuncSetAttribute(k_objfull<double, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      k_objfull<double, true><<<grid, kThreads, smem, st>>>(P, alpha, with_const, part, ticket, out);
    } else {
    GMF_CUDA(cudaFuncSetAttribute(k_objfull<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    k_objfull<double><<<grid, kThreads, smem, st>>>(P, alpha, with_const, part, ticket, out);
    }
  } else {
    if (P.gen) {
      GMF_CUDA(cudaFuncSetAttribute(k_objfull<float, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      k_objfull<float, true><<<grid, kThreads, smem, st>>>(P, alpha, with_const, part, ticket, out);
    } else {
    GMF_CUDA(cudaFuncSetAttribute(k_objfull<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    k_objfull<float><<<grid, kThreads, smem, st>>>(P, alpha, with_const, part, ticket, out);
    }
  }
  GMF_LAUNCH_CHECK("k_objfull");
  return GMF_OK;
}

int launch_entries(const Params& P, int dtype, double alpha, const int64_t* rows,
                   const int32_t* cols, const double* y, int64_t n, double ybar, double* mu_out,
                   double* part, unsigned int* ticket, double* out, cudaStream_t st) {
  int64_t b = (n + kThreads - 1) / kThreads;
  if (b > 2 * kSMs) b = 2 * kSMs;
  if (b < 1) b = 1;
  if (dtype == GMF_F64)
    k_entries<double><<<(unsigned)b, kThreads, 0, st>>>(P, alpha, rows, cols, y, n, ybar, mu_out,
                                                         part, ticket, out);
  else
    k_entries<float><<<(unsigned)b, kThreads, 0, st>>>(P, alpha, rows, cols, y, n, ybar, mu_out,
                                                        part, ticket, out);
  GMF_LAUNCH_CHECK("k_entries");
  return GMF_OK;
}

}  // namespace gmf
