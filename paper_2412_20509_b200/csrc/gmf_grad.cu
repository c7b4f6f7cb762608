// K1: fused minibatch gradient for one aSGD step (sm_100a, CUDA cores).
//
// One CTA owns a tile of TC columns of the column block J and a contiguous
// range of row chunks (TR rows each) of the row block I.  Per entry:
//   eta = offset_i + [x_i|u_i|gamma_i] . [b_j|v_j|z_j]       (model.py:229-256)
//   mu  = exp(eta)                                             (_ref.py:21-32)
//   dotD, ddotD  (Poisson / NB with log link)                  (_core.pyx:79-103)
// Column side  sum_i dotD_ij [x_i, u_i], ddotD_ij [x_i^2, u_i^2] accumulates in
// registers (thread == column) across all of the CTA's rows; the row side
// sum_j dotD_ij [z_j, v_j] (and ddotD with squares) is a small smem GEMM over
// the chunk's P tile (gradients.py:102-113).  eta and mu never leave
// registers; P lives only in shared memory.  Cross-CTA reductions are
// fixed-order (determinism contract): per-CTA partials plus a
// "last CTA" ticket, never float atomics.
#include "gmf_engine.cuh"

namespace gmf {

struct GradSmem {
  int64_t rd, a, cd2, off, y, w, P, red, cp, total;
};

// byte offsets of the dynamic shared-memory carve-up (host + device)
GMF_HD GradSmem grad_smem(int NK, int tsz, int has_w, int Kr, int Kc) {
  GradSmem s;
  int64_t o = 0;
  auto al = [](int64_t v) { return (v + 15) & ~int64_t(15); };
  s.rd = o; o = al(o + (int64_t)2 * TC * NK * tsz);
  s.P = o; o = al(o + (int64_t)2 * TC * (TR + 1) * tsz);
  const int64_t region = o;
  int64_t r = region;
  s.a = r; r = al(r + (int64_t)TR * NK * tsz);
  s.cd2 = r; r = al(r + (int64_t)TR * NK * tsz);
  s.off = r; r = al(r + (int64_t)TR * tsz);
  s.y = r; r = al(r + (int64_t)TR * TC * tsz);
  s.w = r; r = al(r + (has_w ? (int64_t)TR * TC * tsz : 0));
  const int64_t p1 = r - region;
  const int64_t red = al((int64_t)NQ * 2 * Kr * (TR + 1) * tsz);
  const int64_t cp = al((int64_t)TC * (2 * Kc + 1) * tsz);
  s.red = region;
  s.cp = region;
  int64_t mx = p1 > red ? p1 : red;
  mx = mx > cp ? mx : cp;
  s.total = region + mx;
  return s;
}

template <typename T, int FAM, int NK>
__global__ void __launch_bounds__(kThreads, 1)
k_grad(Params P, long long xb, long long xs, double xalpha) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ double red_scr[kThreads / 32];
  const int tid = threadIdx.x;
  const Ctrl* C = P.ctrl;

  long long blk, s;
  double alpha;
  if (xb >= 0) {
    blk = xb; s = xs; alpha = xalpha;
  } else {
    const long long t = C->t;
    if (C->stopped || t >= P.max_steps) return;   // uniform across the grid
    blk = P.bseq[t];
    s = t % P.S;
    alpha = C->nb_shape;
  }
  const int Kr = P.Kr, Kc = P.Kc, KA = P.KA, p = P.p, q = P.q, d = P.d;
  const int64_t r0 = P.rbp[blk], nI = P.rbp[blk + 1] - r0;
  const int64_t j0 = P.cbp[s], nJ = P.cbp[s + 1] - j0;
  const int ct = blockIdx.y, rs = blockIdx.x, RS = gridDim.x;
  const int64_t nchunks = (nI + TR - 1) / TR;
  const int64_t cpr = (nchunks + RS - 1) / RS;
  const int64_t ch_lo = rs * cpr, ch_hi = ch_lo + cpr < nchunks ? ch_lo + cpr : nchunks;

  const GradSmem L = grad_smem(NK, sizeof(T), P.has_w, Kr, Kc);
  T* rd_s = reinterpret_cast<T*>(smem + L.rd);
  T* P_s = reinterpret_cast<T*>(smem + L.P);
  T* a_s = reinterpret_cast<T*>(smem + L.a);
  T* cd2_s = reinterpret_cast<T*>(smem + L.cd2);
  T* off_s = reinterpret_cast<T*>(smem + L.off);
  T* y_s = reinterpret_cast<T*>(smem + L.y);
  T* w_s = reinterpret_cast<T*>(smem + L.w);
  T* red_s = reinterpret_cast<T*>(smem + L.red);
  T* cp_s = reinterpret_cast<T*>(smem + L.cp);

  const T* th_row = tptr<T>(P.th_row);
  const T* th_col = tptr<T>(P.th_col);
  const T* xg = tptr<T>(P.x);
  const T* zg = tptr<T>(P.z);
  const T* offg = tptr<T>(P.off);
  const T* wg = tptr<T>(P.w);

  // ---- column features of this thread's column (phase 1) ----
  const int c = tid % TC, g = tid / TC;
  const int64_t pos = (int64_t)ct * TC + c;
  const bool col_ok = pos < nJ;
  const int64_t j = col_ok ? (P.col_identity ? pos : (int64_t)P.cidx[j0 + pos]) : 0;
  T cf[NK];
  #pragma unroll
  for (int k = 0; k < NK; ++k) {
    T v = T(0);
    if (col_ok) {
      if (k < Kc) v = th_col[j * Kc + k];
      else if (k < KA) v = zg[j * q + (k - Kc)];
    }
    cf[k] = v;
  }
  // ---- row-side design [z_j | v_j] and squares for the tile (phase 2) ----
  for (int e = tid; e < TC * NK; e += kThreads) {
    const int cc = e / NK, k = e % NK;
    const int64_t pp = (int64_t)ct * TC + cc;
    T v = T(0);
    if (pp < nJ && k < Kr) {
      const int64_t jj = P.col_identity ? pp : (int64_t)P.cidx[j0 + pp];
      v = k < q ? zg[jj * q + k] : th_col[jj * Kc + p + (k - q)];
    }
    rd_s[cc * NK + k] = v;
    rd_s[(TC + cc) * NK + k] = v * v;
  }

  T gacc[NK], hacc[NK];
  #pragma unroll
  for (int k = 0; k < NK; ++k) { gacc[k] = T(0); hacc[k] = T(0); }
  double nb_num = 0.0, nb_den = 0.0;
  const T rphi = T(1.0 / P.phi);
  const T ralpha = T(1.0 / alpha);

  // phase-2 role
  const int pr = tid % TR, ph = (tid / TR) & 1, pq = tid / (2 * TR);
  constexpr int TCQ = TC / NQ;
  const int rkk = 2 * Kr;

  for (int64_t ch = ch_lo; ch < ch_hi; ++ch) {
    const int64_t rowbase = ch * TR;                       // within block
    const int rows = (int)((nI - rowbase) < TR ? (nI - rowbase) : TR);
    __syncthreads();   // previous chunk's red_s reads are done
    // ---- load row features [x | u | gamma], squares, offset ----
    for (int e = tid; e < TR * NK; e += kThreads) {
      const int rr = e / NK, k = e % NK;
      T v = T(0);
      if (rr < rows) {
        const int64_t i = r0 + rowbase + rr;
        if (k < p) v = xg[i * p + k];
        else if (k < p + d) v = th_row[i * Kr + q + (k - p)];
        else if (k < KA) v = th_row[i * Kr + (k - p - d)];
      }
      a_s[rr * NK + k] = v;
      cd2_s[rr * NK + k] = k < Kc ? v * v : T(0);
    }
    if (tid < TR) {
      T v = T(0);
      if (tid < rows && P.has_off) v = offg[r0 + rowbase + tid];
      off_s[tid] = v;
    }
    // ---- response tile ----
    if (P.yfmt == GMF_Y_DENSE_I32) {
      for (int e = tid; e < TR * TC; e += kThreads) {
        const int rr = e / TC, cc = e % TC;
        const int64_t pp = (int64_t)ct * TC + cc;
        T v = T(0), wv = T(0);
        if (rr < rows && pp < nJ) {
          const int64_t jj = P.col_identity ? pp : (int64_t)P.cidx[j0 + pp];
          const int64_t i = r0 + rowbase + rr;
          v = (T)P.y[i * P.m + jj];
          if (P.has_w) wv = wg[i * P.m + jj];
        }
        y_s[e] = v;
        if (P.has_w) w_s[e] = wv;
      }
    } else {
      for (int e = tid; e < TR * TC; e += kThreads) y_s[e] = T(0);
      __syncthreads();
      const int lane = tid & 31, warp = tid >> 5;
      for (int rr = warp; rr < rows; rr += kThreads / 32) {
        const int64_t i = r0 + rowbase + rr;
        const int64_t a = P.rp[i], b = P.rp[i + 1];
        for (int64_t k = a + lane; k < b; k += 32) {
          const int col = P.ci[k];
          int64_t pp;
          if (P.col_identity) pp = col;
          else pp = (P.cbof[col] == s) ? (int64_t)P.cpos[col] : -1;
          const int64_t cl = pp - (int64_t)ct * TC;
          if (pp >= 0 && cl >= 0 && cl < TC) y_s[rr * TC + cl] = (T)P.cv[k];
        }
      }
    }
    __syncthreads();

    // ---- phase 1: eta, mu, dotD, ddotD; column side in registers ----
    T cn = T(0), cd = T(0);
    #pragma unroll 2
    for (int rr = g; rr < TR; rr += NG) {
      const T* a = a_s + rr * NK;
      T eta = off_s[rr];
      #pragma unroll
      for (int k = 0; k < NK; ++k) eta = fma(a[k], cf[k], eta);
      const T mu = exp_t(eta);
      const T yv = y_s[rr * TC + c];
      const T wv = P.has_w ? w_s[rr * TC + c] : T(1);
      const T r = yv - mu;
      T dd, hh;
      if (FAM == 0) {
        dd = -wv * r * rphi;
        hh = wv * mu * rphi;
      } else {
        const T inv = rcp_t(T(P.phi) * fma(mu, ralpha, T(1)));
        dd = -wv * r * inv;
        hh = wv * mu * inv;
      }
      const bool ok = col_ok && rr < rows;
      if (!ok) { dd = T(0); hh = T(0); }
      const T* a2 = cd2_s + rr * NK;
      #pragma unroll
      for (int k = 0; k < NK; ++k) {
        gacc[k] = fma(dd, a[k], gacc[k]);
        hacc[k] = fma(hh, a2[k], hacc[k]);
      }
      P_s[c * (TR + 1) + rr] = dd;
      P_s[(TC + c) * (TR + 1) + rr] = hh;
      if (FAM == 1 && ok) {
        cn = fma(wv * mu, mu, cn);
        cd = fma(wv, fma(r, r, -mu), cd);
      }
    }
    nb_num += (double)cn;
    nb_den += (double)cd;
    __syncthreads();

    // ---- phase 2: row side  P (TR x TC) . rd (TC x Kr) ----
    T acc[NK];
    #pragma unroll
    for (int k = 0; k < NK; ++k) acc[k] = T(0);
    {
      const T* Pp = P_s + ph * TC * (TR + 1);
      const T* rdp = rd_s + ph * TC * NK;
      #pragma unroll 4
      for (int cc = pq * TCQ; cc < (pq + 1) * TCQ; ++cc) {
        const T pv = Pp[cc * (TR + 1) + pr];
        const T* rd = rdp + cc * NK;
        #pragma unroll
        for (int k = 0; k < NK; ++k) acc[k] = fma(pv, rd[k], acc[k]);
      }
    }
    // red_s aliases the phase-1 tile region: every thread finished phase 1
    // before the barrier above, so it is free now.
    #pragma unroll
    for (int k = 0; k < NK; ++k)
      if (k < Kr) red_s[((pq * 2 + ph) * Kr + k) * (TR + 1) + pr] = acc[k];
    __syncthreads();
    {
      T* outp = tptr<T>(P.rowpart) + ((int64_t)ct * P.nstar_max + rowbase) * rkk;
      for (int o = tid; o < rows * rkk; o += kThreads) {
        const int rr = o / rkk, hk = o % rkk;
        const int h = hk / Kr, k = hk % Kr;
        T sum = T(0);
        #pragma unroll
        for (int qq = 0; qq < NQ; ++qq) sum += red_s[((qq * 2 + h) * Kr + k) * (TR + 1) + rr];
        outp[o] = sum;
      }
    }
  }
  __syncthreads();

  // ---- column partials: fixed-order sum over the NG row groups ----
  const int ck = 2 * Kc + 1;
  for (int round = 0; round < NG; ++round) {
    if (g == round) {
      #pragma unroll
      for (int k = 0; k < NK; ++k) {
        if (k < Kc) {
          if (round == 0) { cp_s[c * ck + k] = gacc[k]; cp_s[c * ck + Kc + k] = hacc[k]; }
          else { cp_s[c * ck + k] += gacc[k]; cp_s[c * ck + Kc + k] += hacc[k]; }
        }
      }
    }
    __syncthreads();
  }
  const int kk = 2 * Kc;
  T* colpart = tptr<T>(P.colpart);
  const int64_t cbase = ((int64_t)ct * RS + rs) * TC * kk;
  for (int e = tid; e < TC * kk; e += kThreads) colpart[cbase + e] = cp_s[(e / kk) * ck + (e % kk)];

  // NB moment partials (optim.py:225-226)
  const double bn = block_sum<kThreads>(nb_num, red_scr);
  const double bd = block_sum<kThreads>(nb_den, red_scr);
  if (tid == 0) {
    P.nbpart[2 * ((int64_t)ct * RS + rs)] = bn;
    P.nbpart[2 * ((int64_t)ct * RS + rs) + 1] = bd;
  }

  // ---- last CTA of this column tile: rank-level column partial ----
  if (last_block_ticket(P.tickets + ct, RS)) {
    T* recp = reinterpret_cast<T*>(P.rec + REC_HDR);
    for (int e = tid; e < TC * kk; e += kThreads) {
      const int64_t pp = (int64_t)ct * TC + e / kk;
      if (pp >= nJ) continue;
      T sum = T(0);
      for (int r2 = 0; r2 < RS; ++r2) {
        const T* src = colpart + ((int64_t)ct * RS + r2) * TC * kk + e;
        sum += sizeof(T) == 8 ? (T)__ldcg((const double*)src) : (T)__ldcg((const float*)src);
      }
      recp[pp * kk + (e % kk)] = sum;
    }
    if (tid == 0) P.tickets[ct] = 0u;
  }
  // ---- last CTA overall: NB sums in fixed CTA order ----
  const unsigned int total = (unsigned int)(RS * gridDim.y);
  if (last_block_ticket(P.tickets + P.CT, total)) {
    if (tid == 0) {
      double sn = 0.0, sd = 0.0;
      for (unsigned int b = 0; b < total; ++b) {
        sn += __ldcg(P.nbpart + 2 * b);
        sd += __ldcg(P.nbpart + 2 * b + 1);
      }
      P.rec[R_NBNUM] = sn;
      P.rec[R_NBDEN] = sd;
      P.tickets[P.CT] = 0u;
    }
  }
}

template <typename T, int FAM, int NK>
static int launch_one(const Params& P, dim3 grid, size_t smem, cudaStream_t st, long long xb,
                      long long xs, double xalpha) {
  k_grad<T, FAM, NK><<<grid, kThreads, smem, st>>>(P, xb, xs, xalpha);
  GMF_LAUNCH_CHECK("k_grad");
  return GMF_OK;
}

template <typename T, int FAM>
static int launch_nk(const Params& P, int NK, dim3 grid, size_t smem, cudaStream_t st,
                     long long xb, long long xs, double xa) {
  switch (NK) {
    case 8: return launch_one<T, FAM, 8>(P, grid, smem, st, xb, xs, xa);
    case 12: return launch_one<T, FAM, 12>(P, grid, smem, st, xb, xs, xa);
    case 16: return launch_one<T, FAM, 16>(P, grid, smem, st, xb, xs, xa);
    case 24: return launch_one<T, FAM, 24>(P, grid, smem, st, xb, xs, xa);
    case 32: return launch_one<T, FAM, 32>(P, grid, smem, st, xb, xs, xa);
    default: set_error("unsupported feature bucket %d", NK); return GMF_ERR_UNSUPPORTED;
  }
}

template <typename T, int FAM>
static int prepare_nk(int NK) {
  cudaError_t e = cudaSuccess;
  switch (NK) {
    case 8: e = cudaFuncSetAttribute(k_grad<T, FAM, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024); break;
    case 12: e = cudaFuncSetAttribute(k_grad<T, FAM, 12>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024); break;
    case 16: e = cudaFuncSetAttribute(k_grad<T, FAM, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024); break;
    case 24: e = cudaFuncSetAttribute(k_grad<T, FAM, 24>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024); break;
    case 32: e = cudaFuncSetAttribute(k_grad<T, FAM, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024); break;
    default: set_error("unsupported feature bucket %d", NK); return GMF_ERR_UNSUPPORTED;
  }
  if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(k_grad)");
  return GMF_OK;
}

// opt in to >48 KB dynamic shared memory once per handle (outside graph capture)
int prepare_grad(int dtype, int family, int NK) {
  const int fam = family == GMF_NEG_BINOMIAL ? 1 : 0;
  if (dtype == GMF_F64) return fam ? prepare_nk<double, 1>(NK) : prepare_nk<double, 0>(NK);
  return fam ? prepare_nk<float, 1>(NK) : prepare_nk<float, 0>(NK);
}

int grad_bucket(int KA) {
  if (KA <= 8) return 8;
  if (KA <= 12) return 12;
  if (KA <= 16) return 16;
  if (KA <= 24) return 24;
  if (KA <= 32) return 32;
  return -1;
}

int64_t grad_smem_bytes(int dtype, int NK, int has_w, int Kr, int Kc) {
  return grad_smem(NK, dtype == GMF_F64 ? 8 : 4, has_w, Kr, Kc).total;
}

int launch_grad(const Params& P, int dtype, int NK, cudaStream_t st, long long xb, long long xs,
                double xalpha) {
  dim3 grid(P.RS, P.CT);
  const size_t smem = (size_t)grad_smem_bytes(dtype, NK, P.has_w, P.Kr, P.Kc);
  const int fam = P.fam == GMF_NEG_BINOMIAL ? 1 : 0;
  if (dtype == GMF_F64)
    return fam ? launch_nk<double, 1>(P, NK, grid, smem, st, xb, xs, xalpha)
               : launch_nk<double, 0>(P, NK, grid, smem, st, xb, xs, xalpha);
  return fam ? launch_nk<float, 1>(P, NK, grid, smem, st, xb, xs, xalpha)
             : launch_nk<float, 0>(P, NK, grid, smem, st, xb, xs, xalpha);
}

}  // namespace gmf
