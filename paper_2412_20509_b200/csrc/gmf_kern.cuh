// Device bodies shared by the per-step kernels (multi-rank path) and the
// persistent fit kernel (single-rank path).
#pragma once
#include "gmf_engine.cuh"

namespace gmf {

// ---------------------------------------------------------------------------
// value of Y and eta at a tracked entry (optim.py:274-280)
// ---------------------------------------------------------------------------
// stored nonzero k of the CSR formats: column and count
GMF_D int csr_col_at(const Params& P, int64_t k) {
  const int32_t w = P.ci[k];
  return P.yfmt == GMF_Y_CSR_PACK32 ? (int)((uint32_t)w & 0xFFFFu) : (int)w;
}
GMF_D int csr_val_at(const Params& P, int64_t k) {
  return P.yfmt == GMF_Y_CSR_PACK32 ? (int)((uint32_t)P.ci[k] >> 16) : (int)P.cv[k];
}
// a staged word pair (col, val) of either CSR format
GMF_D int stg_col(int pack, int32_t w) { return pack ? (int)((uint32_t)w & 0xFFFFu) : (int)w; }
GMF_D int stg_val(int pack, int32_t w, int32_t v) { return pack ? (int)((uint32_t)w >> 16) : (int)v; }

GMF_D double y_lookup(const Params& P, int64_t i, int64_t j) {
  if (P.gen) return 0.0;   // real-valued responses are read from y_work where needed
  if (P.yfmt == GMF_Y_DENSE_I32) return (double)P.y[i * P.m + j];
  int64_t lo = P.rp[i], hi = P.rp[i + 1];
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    const int cm = csr_col_at(P, mid);
    if (cm == j) return (double)csr_val_at(P, mid);
    if (cm < j) lo = mid + 1; else hi = mid;
  }
  return 0.0;
}

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
// K3 body: this CTA's share of the tracked objective of the current state
// (optim.py:283-290) -> out[0] deviance, out[1] ||B||^2, out[2] ||V||^2.
// ---------------------------------------------------------------------------
template <typename T>
GMF_D void obj_partial(const Params& P, double alpha, int cta, int ncta, double* out,
                       double dev_partial) {
  __shared__ double scr[3 * (kThreads / 32)];
  (void)alpha;
  double s = dev_partial;   // this CTA's deviance share (gmf_step.cu: entry_dev_cached)
  const int64_t stride = (int64_t)ncta * kThreads;
  const T* tc = tptr<T>(P.th_col);
  double nb = 0.0, nv = 0.0;
  for (int64_t e = (int64_t)cta * kThreads + threadIdx.x; e < P.m * P.Kc; e += stride) {
    const double v = (double)tc[e];
    if ((int)(e % P.Kc) < P.p) nb += v * v; else nv += v * v;
  }
  double v3[3] = {s, nb, nv};
  block_sum_vec<3>(v3, scr);
  if (threadIdx.x == 0) { out[0] = v3[0]; out[1] = v3[1]; out[2] = v3[2]; }
}

// ---------------------------------------------------------------------------
// cp.async (LDGSTS) helpers: 4/8-byte copies with zero fill
// ---------------------------------------------------------------------------
template <int BYTES>
GMF_D void cp_async(void* sdst, const void* gsrc, bool valid) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(sdst);
  const int n = valid ? BYTES : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;" ::"r"(s), "l"(gsrc), "n"(BYTES),
               "r"(n)
               : "memory");
}
GMF_D void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
GMF_D void cp_async_wait0() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// ---------------------------------------------------------------------------
// K1 body: fused minibatch gradient for one CTA tile.
//
// The CTA owns TC columns (column tile `ct` of block J) and a contiguous,
// balanced row range of block I (row split `rs` of RS), walked in TR-row
// chunks.  Per entry:
//   eta = offset_i + [x_i|u_i|gamma_i] . [b_j|v_j|z_j]       (model.py:229-256)
//   mu  = exp(eta)                                             (_ref.py:21-32)
//   dotD, ddotD  (Poisson / NB with log link)                  (_core.pyx:79-103)
// Column side sum_i dotD_ij [x_i, u_i] (ddotD with squares) accumulates in
// registers (thread == column) across all rows of the CTA; the row side
// sum_j dotD_ij [z_j, v_j] is a small shared-memory GEMM over the chunk's P
// tile (gradients.py:102-113).  eta and mu stay in registers.
//
// Software pipeline: the next chunk's row features, offsets and Y (the
// chunk's CSR nonzeros are one contiguous range; dense rows are contiguous)
// are copied into the other staging buffer with cp.async while the current
// chunk computes, so global latency overlaps the FMA work.
// Outputs: rowpart[ct][row][2Kr], colpart[ct][rs][c][2Kc], nbpart[ct*RS+rs][2].
// ---------------------------------------------------------------------------
constexpr int kStageCap = 2048;   // CSR nonzeros staged per chunk (else direct path)
constexpr int kRpMax = 192;       // CSR row pointers staged per CTA row range

struct GradSmem {
  int64_t rd, P, red, rp, ytile, stage[2], a[2], cd2[2], off[2], wt[2], total, stage_bytes;
};

GMF_HD GradSmem grad_smem(int TC, int NK, int tsz, int has_w, int Kr, int Kc) {
  GradSmem s;
  int64_t o = 0;
  auto al = [](int64_t v) { return (v + 15) & ~int64_t(15); };
  s.rd = o; o = al(o + (int64_t)2 * TC * NK * tsz);
  s.P = o; o = al(o + (int64_t)2 * TC * (TR + 1) * tsz);
  // fp64 at K > 32: the row-side reduction runs in two passes over halves of
  // the Kr features so its buffer (and the tile) fits in shared memory
  const int KrR = (tsz == 8 && NK > 32) ? (Kr + 1) / 2 : Kr;
  const int64_t red = (int64_t)NQ * 2 * KrR * (TR + 1) * tsz;
  const int64_t cp = (int64_t)TC * (2 * Kc + 1) * tsz;
  s.red = o; o = al(o + red);   // (column partials reuse the P region at the end)
  (void)cp;
  s.rp = o; o = al(o + (int64_t)(kRpMax + 1) * 8);
  s.ytile = o; o = al(o + (int64_t)TR * TC * 4);
  // a stage holds either the dense int32 Y tile or the CSR (col, val) range
  const int64_t dense = (int64_t)TR * TC * tsz, csr = (int64_t)kStageCap * 8;   // int32 or T (holes)
  s.stage_bytes = dense > csr ? dense : csr;
  for (int b = 0; b < 2; ++b) {
    s.stage[b] = o; o = al(o + s.stage_bytes);
    s.a[b] = o; o = al(o + (int64_t)TR * NK * tsz);
    s.cd2[b] = o; o = al(o + (int64_t)TR * NK * tsz);
    s.off[b] = o; o = al(o + (int64_t)TR * tsz);
    s.wt[b] = o; o = al(o + (has_w ? (int64_t)TR * TC * tsz : 0));
  }
  s.total = o;
  return s;
}

// exp of a predictor that the caller pre-scaled by log2(e) (fp32: MUFU ex2)
GMF_D float exp_pre(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
GMF_D double exp_pre(double x) { return exp(x); }
template <typename T> struct Pre { static constexpr double s = 1.4426950408889634; };
template <> struct Pre<double> { static constexpr double s = 1.0; };

GMF_D float rcp_fast(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
GMF_D double rcp_fast(double x) { return 1.0 / x; }

// phase 1 of one chunk: eta, mu, dotD, ddotD per entry; column side into
// registers; P tile into shared memory.  Branch-free: invalid rows/columns
// carry weight 0, which zeroes dotD, ddotD and the NB moment terms.
// HOLES: the staged Y tile holds the working response (T): observed values
// >= 0, an unobserved entry as -(its imputed mean).  hmode 1 (the fit):
// holes enter with their imputed mean, refilled with this step's mu when
// `fill` (optim.py:430-436, the refill written back through ywg); hmode 2
// (standalone minibatch gradients, gradients.py:66-88): holes carry weight 0.
template <typename T, int FAM, int NK, int TC, bool HW, bool HOLES = false>
GMF_D void phase1(const T* __restrict__ a_s, const T* __restrict__ cd2_s,
                  const T* __restrict__ off_s, const int32_t* __restrict__ y_s,
                  const T* __restrict__ w_s, T* __restrict__ P_s, const T (&cf)[NK],
                  T (&gacc)[NK], T (&hacc)[NK], T cm, int c, int g, int rows, T rphi, T tphi,
                  T ralpha, T& cn, T& cd, int hmode = 0, bool fill = false, T* ywg = nullptr,
                  int64_t ystride = 0, int fcode = 0, int lcode = 0) {
  constexpr int NG = kThreads / TC;
  #pragma unroll 2
  for (int rr = g; rr < rows; rr += NG) {
    const T* a = a_s + rr * NK;
    T e0 = off_s[rr], e1 = T(0);
    #pragma unroll
    for (int k = 0; k < NK; k += 2) {
      e0 = fma(a[k], cf[k], e0);
      e1 = fma(a[k + 1], cf[k + 1], e1);
    }
    // FAM 2 (general mode): the features are not pre-scaled, any link
    const T mu = FAM == 2 ? gen_mean<T>(lcode, e0 + e1) : exp_pre(e0 + e1);
    T yv;
    T wv = HW ? w_s[rr * TC + c] : cm;
    if constexpr (HOLES) {
      // hmode 3: y_work is a plain real-valued response (no holes)
      const T v = reinterpret_cast<const T*>(y_s)[rr * TC + c];
      // count paths: a hole is minus its imputed mean; general mode (FAM 2):
      // the imputed mean with its last mantissa bit set
      const bool hole = hmode != 3 && (FAM == 2 ? lsb_set(v) : signbit(v));
      yv = (hole && FAM != 2) ? -v : v;
      if (hole && hmode == 2) wv = T(0);
      if (hole && hmode == 1 && fill && cm != T(0)) {
        yv = mu;
        ywg[(int64_t)rr * ystride] = FAM == 2 ? with_lsb(mu) : -mu;
      }
    } else {
      yv = (T)y_s[rr * TC + c];
    }
    const T r = yv - mu;
    T dd, hh;
    if (FAM == 2) {
      T pear;
      gen_derivs<T>(fcode, lcode, yv, mu, wv, tphi, T(1) / ralpha, dd, hh, pear);
      if (wv == T(0)) { dd = T(0); hh = T(0); pear = T(0); }   // outside the block: no NaNs
      cn += pear;
    } else if (FAM == 0) {
      const T ws = wv * rphi;
      dd = -ws * r;
      hh = ws * mu;
    } else {
      const T inv = wv * rcp_fast(tphi * fma(mu, ralpha, T(1)));
      dd = -r * inv;
      hh = mu * inv;
      cn = fma(wv * mu, mu, cn);
      cd = fma(wv, fma(r, r, -mu), cd);
    }
    const T* a2 = cd2_s + rr * NK;
    #pragma unroll
    for (int k = 0; k < NK; ++k) {
      gacc[k] = fma(dd, a[k], gacc[k]);
      hacc[k] = fma(hh, a2[k], hacc[k]);
    }
    P_s[c * (TR + 1) + rr] = dd;
    P_s[(TC + c) * (TR + 1) + rr] = hh;
  }
}

template <typename T, int FAM, int NK, int TC>
GMF_D void grad_cta(const Params& P, long long blk, long long s, double alpha, int rs, int ct,
                    int RS, unsigned char* smem, int hmode = 0, bool fill = false,
                    double phi = -1.0) {
  if (phi < 0.0) phi = P.phi;   // the fit passes the live dispersion (Ctrl.phi)
  constexpr int NG = kThreads / TC;
  constexpr int TCQ = TC / NQ;
  __shared__ double red_scr[kThreads / 32];
  __shared__ int stage_n[2];   // staged CSR nonzeros per buffer, -1 = overflow
  const int tid = threadIdx.x;
  const int Kr = P.Kr, Kc = P.Kc, KA = P.KA, p = P.p, q = P.q, d = P.d;
  const int64_t r0 = P.rbp[blk], nI = P.rbp[blk + 1] - r0;
  const int64_t j0 = P.cbp[s], nJ = P.cbp[s + 1] - j0;
  // this row split's contiguous rows of block I, balanced to within one row
  const int64_t rlo = nI * rs / RS, rhi = nI * (rs + 1) / RS;
  const int64_t nrows = rhi - rlo;
  const bool csr = P.yfmt != GMF_Y_DENSE_I32;
  const bool rp_staged = csr && nrows <= kRpMax;
  const int64_t cbase = (int64_t)ct * TC;

  const GradSmem L = grad_smem(TC, NK, sizeof(T), P.has_w, Kr, Kc);
  T* rd_s = reinterpret_cast<T*>(smem + L.rd);
  T* P_s = reinterpret_cast<T*>(smem + L.P);
  T* red_s = reinterpret_cast<T*>(smem + L.red);
  T* cp_s = reinterpret_cast<T*>(smem + L.P);
  int64_t* rp_s = reinterpret_cast<int64_t*>(smem + L.rp);
  int32_t* ytile = reinterpret_cast<int32_t*>(smem + L.ytile);

  const T* th_row = tptr<T>(P.th_row);
  const T* th_col = tptr<T>(P.th_col);
  const T* xg = tptr<T>(P.x);
  const T* zg = tptr<T>(P.z);
  const T* offg = tptr<T>(P.off);
  const T* wg = tptr<T>(P.w);
  const T pre = FAM == 2 ? T(1) : T(Pre<T>::s);

  // ---- this thread's column features [b | v | z] (phase 1), pre-scaled ----
  const int c = tid % TC, g = tid / TC;
  const int64_t pos = cbase + c;
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
    cf[k] = v * pre;
  }
  const T cm = col_ok ? T(1) : T(0);
  __syncthreads();   // smem reuse across calls (persistent kernel)
  // ---- row-side design [z_j | v_j] and squares of the tile (phase 2) ----
  for (int e = tid; e < TC * NK; e += kThreads) {
    const int cc = e / NK, k = e % NK;
    const int64_t pp = cbase + cc;
    T v = T(0);
    if (pp < nJ && k < Kr) {
      const int64_t jj = P.col_identity ? pp : (int64_t)P.cidx[j0 + pp];
      v = k < q ? zg[jj * q + k] : th_col[jj * Kc + p + (k - q)];
    }
    rd_s[cc * NK + k] = v;
    rd_s[(TC + cc) * NK + k] = v * v;
  }
  if (rp_staged)
    for (int64_t e = tid; e <= nrows; e += kThreads) rp_s[e] = P.rp[r0 + rlo + e];
  if (csr)
    for (int e = tid; e < TR * TC; e += kThreads) ytile[e] = 0;
  __syncthreads();

  // ---- asynchronous staging of one chunk into buffer b ----
  auto issue = [&](int b, int64_t rowbase) {
    const int rows = (int)((rhi - rowbase) < TR ? (rhi - rowbase) : TR);
    const int64_t i0 = r0 + rowbase;
    T* a_b = reinterpret_cast<T*>(smem + L.a[b]);
    T* off_b = reinterpret_cast<T*>(smem + L.off[b]);
    for (int e = tid; e < TR * NK; e += kThreads) {
      const int rr = e / NK, k = e % NK;
      const T* src = xg;
      bool ok = false;
      if (rr < rows) {
        const int64_t i = i0 + rr;
        if (k < p) { src = xg + i * p + k; ok = true; }
        else if (k < p + d) { src = th_row + i * Kr + q + (k - p); ok = true; }
        else if (k < KA) { src = th_row + i * Kr + (k - p - d); ok = true; }
      }
      cp_async<sizeof(T)>(a_b + e, src, ok);
    }
    if (tid < TR) {
      const bool ok = tid < rows && P.has_off;
      cp_async<sizeof(T)>(off_b + tid, ok ? offg + i0 + tid : offg, ok);
    }
    if (P.has_w) {
      T* w_b = reinterpret_cast<T*>(smem + L.wt[b]);
      for (int e = tid; e < TR * TC; e += kThreads) {
        const int rr = e / TC, cc = e % TC;
        const int64_t pp = cbase + cc;
        const bool ok = rr < rows && pp < nJ;
        const int64_t jj = ok ? (P.col_identity ? pp : (int64_t)P.cidx[j0 + pp]) : 0;
        cp_async<sizeof(T)>(w_b + e, ok ? wg + (i0 + rr) * P.m + jj : wg, ok);
      }
    }
    unsigned char* st = smem + L.stage[b];
    if (!csr && (FAM == 2 || P.holes)) {   // working / real-valued response (T)
      T* y_b = reinterpret_cast<T*>(st);
      const T* yw = tptr<T>(P.y_work);
      for (int e = tid; e < TR * TC; e += kThreads) {
        const int rr = e / TC, cc = e % TC;
        const int64_t pp = cbase + cc;
        const bool ok = rr < rows && pp < nJ;
        const int64_t jj = ok ? (P.col_identity ? pp : (int64_t)P.cidx[j0 + pp]) : 0;
        cp_async<sizeof(T)>(y_b + e, ok ? yw + (i0 + rr) * P.m + jj : yw, ok);
      }
    } else if (!csr) {
      int32_t* y_b = reinterpret_cast<int32_t*>(st);
      for (int e = tid; e < TR * TC; e += kThreads) {
        const int rr = e / TC, cc = e % TC;
        const int64_t pp = cbase + cc;
        const bool ok = rr < rows && pp < nJ;
        const int64_t jj = ok ? (P.col_identity ? pp : (int64_t)P.cidx[j0 + pp]) : 0;
        cp_async<4>(y_b + e, ok ? P.y + (i0 + rr) * P.m + jj : P.y, ok);
      }
    } else if (rp_staged) {
      const int64_t lo = rp_s[rowbase - rlo], hi = rp_s[rowbase - rlo + rows];
      const int64_t nnz = hi - lo;
      if (nnz <= kStageCap) {
        int32_t* col_b = reinterpret_cast<int32_t*>(st);
        int32_t* val_b = col_b + kStageCap;
        const bool pack = P.yfmt == GMF_Y_CSR_PACK32;
        for (int64_t e = tid; e < nnz; e += kThreads) {
          cp_async<4>(col_b + e, P.ci + lo + e, true);
          if (!pack) cp_async<4>(val_b + e, P.cv + lo + e, true);
        }
        if (tid == 0) stage_n[b] = (int)nnz;
      } else if (tid == 0) {
        stage_n[b] = -1;
      }
    } else if (tid == 0) {
      stage_n[b] = -1;
    }
    cp_async_commit();
  };

  T gacc[NK], hacc[NK];
  #pragma unroll
  for (int k = 0; k < NK; ++k) { gacc[k] = T(0); hacc[k] = T(0); }
  double nb_num = 0.0, nb_den = 0.0;
  const T rphi = T(1.0 / phi);
  const T ralpha = T(1.0 / alpha);
  const T tphi = T(phi);
  const int pr = tid % TR, ph = (tid / TR) & 1, pq = tid / (2 * TR);
  const int rkk = 2 * Kr;
  // incremental (row, component) walk of the row-partial output loop
  const int o_rr0 = tid / rkk, o_hk0 = tid % rkk, o_dq = kThreads / rkk, o_dr = kThreads % rkk;

  if (nrows > 0) issue(0, rlo);
  int b = 0;
  for (int64_t rowbase = rlo; rowbase < rhi; rowbase += TR, b ^= 1) {
    const int rows = (int)((rhi - rowbase) < TR ? (rhi - rowbase) : TR);
    const int64_t i0 = r0 + rowbase;
    T* a_s = reinterpret_cast<T*>(smem + L.a[b]);
    T* cd2_s = reinterpret_cast<T*>(smem + L.cd2[b]);
    T* off_s = reinterpret_cast<T*>(smem + L.off[b]);
    T* w_s = reinterpret_cast<T*>(smem + L.wt[b]);
    unsigned char* st = smem + L.stage[b];
    cp_async_wait0();
    __syncthreads();   // chunk b landed; previous chunk fully consumed
    // ---- post-process the staged chunk ----
    for (int e = tid; e < TR * NK; e += kThreads) {
      const T v = a_s[e];
      cd2_s[e] = (e % NK) < Kc ? v * v : T(0);
    }
    if (tid < TR) off_s[tid] *= pre;
    const int32_t* y_s;
    if (!csr) {
      y_s = reinterpret_cast<const int32_t*>(st);
    } else {
      y_s = ytile;
      const int n_st = stage_n[b];
      if (n_st >= 0) {
        // warp per row: the row index is known, no search per nonzero
        const int32_t* col_b = reinterpret_cast<const int32_t*>(st);
        const int32_t* val_b = col_b + kStageCap;
        const int64_t* rpc = rp_s + (rowbase - rlo);
        const int lo = (int)rpc[0];
        const int lane = tid & 31;
        for (int rr = tid >> 5; rr < rows; rr += kThreads / 32) {
          const int a = (int)rpc[rr] - lo, bnd = (int)rpc[rr + 1] - lo;
          const int pack = P.yfmt == GMF_Y_CSR_PACK32;
          for (int e = a + lane; e < bnd; e += 32) {
            const int32_t w = col_b[e];
            const int col = stg_col(pack, w);
            const int pp = P.col_identity ? col : ((P.cbof[col] == s) ? P.cpos[col] : -1);
            const int cl = pp - (int)cbase;
            if (pp >= 0 && cl >= 0 && cl < TC) ytile[rr * TC + cl] = stg_val(pack, w, pack ? 0 : val_b[e]);
          }
        }
      } else {   // row range too long or chunk too dense: direct loads (this tile's range)
        const bool tix = P.tidx != nullptr && !P.stream_mode;
        for (int rr = tid >> 5; rr < rows; rr += kThreads / 32) {
          const int64_t i = i0 + rr;
          int64_t k0 = P.rp[i], k1 = P.rp[i + 1];
          if (tix) {
            const int32_t* tr = P.tidx + i * (P.CT + 1) + ct;
            k1 = k0 + tr[1];
            k0 += tr[0];
          }
          for (int64_t k = k0 + (tid & 31); k < k1; k += 32) {
            const int col = csr_col_at(P, k);
            const int64_t pp = P.col_identity ? col : ((P.cbof[col] == s) ? (int64_t)P.cpos[col] : -1);
            const int64_t cl = pp - cbase;
            if (pp >= 0 && cl >= 0 && cl < TC) ytile[rr * TC + cl] = csr_val_at(P, k);
          }
        }
      }
    }
    __syncthreads();
    // ---- next chunk's loads fly while this one computes ----
    if (rowbase + TR < rhi) issue(b ^ 1, rowbase + TR);

    // ---- phase 1 ----
    T cn = T(0), cd = T(0);
    if (FAM == 2 || P.holes) {
      T* ywg = tptr<T>(P.y_work) + i0 * P.m + j;   // the chunk's first row, this thread's column j
      if (P.has_w)
        phase1<T, FAM, NK, TC, true, true>(a_s, cd2_s, off_s, y_s, w_s, P_s, cf, gacc, hacc, cm, c,
                                           g, rows, rphi, tphi, ralpha, cn, cd, hmode, fill, ywg,
                                           P.m, P.fam, P.link);
      else
        phase1<T, FAM, NK, TC, false, true>(a_s, cd2_s, off_s, y_s, w_s, P_s, cf, gacc, hacc, cm,
                                            c, g, rows, rphi, tphi, ralpha, cn, cd, hmode, fill,
                                            ywg, P.m, P.fam, P.link);
    } else if (P.has_w) {
      phase1<T, FAM, NK, TC, true>(a_s, cd2_s, off_s, y_s, w_s, P_s, cf, gacc, hacc, cm, c, g,
                                   rows, rphi, tphi, ralpha, cn, cd);
    } else {
      phase1<T, FAM, NK, TC, false>(a_s, cd2_s, off_s, y_s, w_s, P_s, cf, gacc, hacc, cm, c, g,
                                    rows, rphi, tphi, ralpha, cn, cd);
    }
    nb_num += (double)cn;
    nb_den += (double)cd;
    __syncthreads();
    if (csr) {   // clear the Y tile for the next scatter (phase 2 does not read it)
      for (int e = tid; e < rows * TC; e += kThreads) ytile[e] = 0;
    }

    // ---- phase 2: row side  P (rows x TC) . rd (TC x Kr) ----
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
    constexpr bool kSplit = sizeof(T) == 8 && NK > 32;
    const int KrR = kSplit ? (Kr + 1) / 2 : Kr;
    #pragma unroll
    for (int pass = 0; pass < (kSplit ? 2 : 1); ++pass) {
      const int k0 = pass * KrR, k1 = min(Kr, k0 + KrR);
      if (pass) __syncthreads();   // previous pass's readers are done with red_s
      #pragma unroll
      for (int k = 0; k < NK; ++k)
        if (k >= k0 && k < k1) red_s[((pq * 2 + ph) * KrR + (k - k0)) * (TR + 1) + pr] = acc[k];
      __syncthreads();
      // o = rr * rkk + hk walked incrementally (no runtime division per element)
      T* outp = tptr<T>(P.rowpart) + ((int64_t)ct * P.nstar_max + rowbase) * rkk;
      int rr = o_rr0, hk = o_hk0;
      for (int o = tid; o < rows * rkk; o += kThreads) {
        const int h = hk >= Kr ? 1 : 0, k = hk - h * Kr;
        if (!kSplit || (k >= k0 && k < k1)) {
          T sum = T(0);
          #pragma unroll
          for (int qq = 0; qq < NQ; ++qq)
            sum += red_s[((qq * 2 + h) * KrR + (k - k0)) * (TR + 1) + rr];
          outp[o] = sum;
        }
        rr += o_dq;
        hk += o_dr;
        if (hk >= rkk) { hk -= rkk; ++rr; }
      }
    }
  }
  cp_async_wait0();
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
  const int64_t cbase2 = ((int64_t)ct * RS + rs) * TC * kk;
  {
    int cc = tid / kk, kx = tid % kk;
    const int dq = kThreads / kk, dr = kThreads % kk;
    for (int e = tid; e < TC * kk; e += kThreads) {
      colpart[cbase2 + e] = cp_s[cc * ck + kx];
      cc += dq;
      kx += dr;
      if (kx >= kk) { kx -= kk; ++cc; }
    }
  }
  const double bn = block_sum<kThreads>(nb_num, red_scr);
  const double bd = block_sum<kThreads>(nb_den, red_scr);
  if (tid == 0) {
    P.nbpart[2 * ((int64_t)ct * RS + rs)] = bn;
    P.nbpart[2 * ((int64_t)ct * RS + rs) + 1] = bd;
  }
}

// column-side gradient sums of element (pos, k) of column block J from the
// per-CTA K1 partials (fixed rs order)
template <typename T>
GMF_D void colpart_sum(const Params& P, int64_t pos, int k, int RS, T& gs, T& hs) {
  const int TC = P.TC, kk = 2 * P.Kc;
  const int64_t ct = pos / TC, c = pos % TC;
  const T* base = tptr<T>(P.colpart) + (ct * RS * TC + c) * kk + k;
  const int64_t stride = (int64_t)TC * kk;
  T g = T(0), h = T(0);
  #pragma unroll 8
  for (int r = 0; r < RS; ++r) {
    g += ldcg_t<T>(base + r * stride);
    h += ldcg_t<T>(base + r * stride + P.Kc);
  }
  gs = g;
  hs = h;
}

// row-side sums of (row il of the block, k) over the CT column tiles
template <typename T, int W = 4>
GMF_D void rowpart_sum(const Params& P, int64_t il, int k, T& gs, T& hs) {
  // the column tiles' loads issued together, W per pass, fixed-order adds
  // (the sum is sequential in the tile index whatever W is)
  const T* rp = tptr<T>(P.rowpart);
  const int64_t cstride = P.nstar_max * (2 * P.Kr);
  const T* src = rp + il * (2 * P.Kr) + k;
  T g = T(0), h = T(0);
  for (int c0 = 0; c0 < P.CT; c0 += W) {
    T gv[W], hv[W];
    gather_vec_cg<W>(src + c0 * cstride, cstride, P.CT - c0, gv);
    gather_vec_cg<W>(src + c0 * cstride + P.Kr, cstride, P.CT - c0, hv);
    #pragma unroll
    for (int ct = 0; ct < W; ++ct) { g += gv[ct]; h += hv[ct]; }
  }
  gs = g;
  hs = h;
}

}  // namespace gmf
