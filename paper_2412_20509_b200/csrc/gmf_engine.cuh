// Device-side state, launch parameters and the shared per-element step
// algebra of the aSGD fit engine.
#pragma once
#include "gmf_common.cuh"

namespace gmf {

constexpr int TR = 32;                    // rows per chunk (K1)
constexpr int NQ = kThreads / (2 * TR);   // column slices in K1 phase 2 (4)
constexpr int REC_HDR = 8;                // doubles in the rank-record header
constexpr int kSnapCtas = 32;
constexpr int OBJ_W = 3;                  // objective partial: (deviance, ||B||^2, ||V||^2)

// column tile width of K1: 128 columns for fp32 (2 row groups of 128
// threads), 64 for fp64 (4 row groups; register/smem budget)
template <typename T> struct Tile { static constexpr int TC = 128; };
template <> struct Tile<double> { static constexpr int TC = 64; };
// the 64-feature bucket (K in (32, 64], fp32 only) halves the CUDA-core K1's
// column tile so its shared memory fits
template <typename T, int NK> struct TileK {
  static constexpr int TC = NK > 32 ? Tile<T>::TC / 2 : Tile<T>::TC;
};

// rank record header slots (doubles)
enum { R_DEV = 0, R_NGAM = 1, R_NU = 2, R_NB = 3, R_NV = 4, R_NBNUM = 5, R_NBDEN = 6 };

// Fit control block.  Per-step kernels read it at entry and only the last
// CTA of k_apply writes it; the persistent kernel keeps an identical copy in
// every CTA (redundant, deterministic computation) and CTA 0 publishes it.
struct Ctrl {
  long long t;                  // steps applied
  long long trace_len;          // objective_trace entries
  long long snap_period;        // number of snapshot points passed (copy-on-write epoch)
  long long snapshot_trace_len;
  double nb_shape;
  double phi;
  double last_obj;
  int streak, converged, diverged, diverged_init, stopped;
};

struct Params {
  int64_t n, m;
  int p, q, d, KA, Kr, Kc;
  int fam, yfmt, has_w, has_off;
  int holes;            // unobserved entries: y_work carries them (negative = imputed mean)
  int gen;              // general mode: runtime family / link, y_work = the real-valued response
  int link;             // gmf_link (general mode; the fused count paths are log-link)
  int est_phi;          // Pearson dispersion update every step (optim.py:175-202)
  double inv_dof;       // 1 / (nm - mp - nq - (n+m)d - 1)   (optim.py:171-172)
  int nafill;           // refill period (optim.py:432)
  void* y_work;         // [n][m] T working response (holes only)
  const int32_t* y;
  const int64_t* rp;
  int64_t nnz;          // rp[n] (CSR)
  const int32_t* ci;
  const int32_t* cv;
  const void* w;
  const void* x;
  const void* z;
  const void* off;
  void* th_row;
  void* th_col;
  void* gb_row;
  void* hb_row;
  void* gb_col;
  void* hb_col;
  void* sn_row;
  void* sn_col;
  const int64_t* rbp;
  const double* rbscale;
  int64_t R;
  const int32_t* cidx;
  const int64_t* cbp;
  const int32_t* cpos;
  const int32_t* cbof;
  int64_t S;
  int col_identity;   // S == 1 and col_idx == arange(m)
  const int32_t* bseq;
  int64_t max_steps;
  const int64_t* erow;
  const int32_t* ecol;
  const int4* ep;     // tracked entries packed (row, col, y, 0), built once
  int64_t E;
  // config
  double a1, a2, damp, tol;
  double lam_b, lam_g, lam_u, lam_v;
  double nbfloor, nbceil, escale, phi;
  int est_alpha, snap_stride, world;
  int tcm;             // K1 on the tensor cores: 1 gmf_tc.cuh, 2 gmf_tc2.cuh (warp-specialized)
  int k1_cap;          // K1 v2: tile-CSR entries staged per chunk slot
  int k1_na1;          // K1 v2: A1 operand buffers (1 or 2)
  void* rimg;                // K1 v2 operand-row images [RS][rimg_nch][tc2::rimg_bytes]
  unsigned int* rimg_flag;   // [RS][rimg_nch] epoch of the last build of each image
  unsigned int* rimg_epoch;  // builds epoch (one per step; device counter)
  int rimg_nch;              // 64-row chunks per row split (max over blocks)
  int ep_cap;          // tracked entries cached per fit CTA in shared memory (0 = none)
  int64_t ep_soff;     // their shared-memory offset (bytes, after K1's region)
  // tracked-objective caches of the persistent kernel (entries sorted by row):
  const int32_t* rslot;  // [n] cache slot of row i (-1: no tracked entry)
  const int64_t* srow;   // [nslots] row of each cache slot
  const int32_t* eslot;  // [E] cache slot of each tracked entry (packed into ep.w)
  int64_t nslots;
  void* ecache;          // [nslots][NK+4] T: a_i = [x | u | gamma | 0..] then offset_i
  void* vpad;            // [m][NK]   T: c_j = [b | v | z | 0..] (16-byte rows)
  int nkb;               // NK, the feature bucket (cache row strides at run time)
  // streaming mode (gmf_run_stream): step t's row block is uploaded while the
  // kernel runs; the copy stream then sets *ready = t + 1, which K1 waits for;
  // each step's status word is written to mapped pinned host memory
  int stream_mode;
  const int64_t* tptr;     // tile-CSR (K1 v2): [CT][n+1] start of tile ct's entries of row i
  const int32_t* tent;     // tile-CSR entries, int32 pairs (row, count << 8 | tile column)
  const int32_t* tidx;     // [n][CT+1] per-row start of each column tile's nonzeros (CSR,
                           // J = all columns, rows sorted by column), else null
  // tensor-core K1 column operands (R | B1h | B1l per column tile, bf16, in the
  // shared-memory byte layout), kept current by the persistent kernel's column
  // updates when every step uses all columns; colimg_on only inside k_fit
  void* colimg;
  int colimg_on;
  const unsigned long long* ready;
  void* host_status;
  const double* rho_tab;     // learning_rate(t)        (optim.py:130-134)
  const double* alpt_tab;    // bias_correction(t + 1)  (optim.py:142-148)
  // workspace
  Ctrl* ctrl;
  double* trace_obj;
  double* trace_nb;
  double* trace_phi;   // dispersion at each trace point (optim.py:326)
  void* rowpart;       // [CT][nstar_max][2 Kr]          T
  void* colpart;       // [CT][RS][TC][2 Kc]            T
  double* nbpart;      // [CT * RS][2]
  unsigned int* tickets;   // [CT] col tiles, [CT] grad-global, [CT+1] obj, [CT+2] apply
  double* totals;          // [7] phase-2 totals, reduced once by the barrier's last arriver
  unsigned int* gbar;      // software grid barrier of the tensor-core fit kernel: count, generation, abort
  double* rec;         // rank record: REC_HDR doubles + [jmax][2 Kc] T
  int64_t rec_stride;  // bytes between gathered records
  double* objpart;     // [n_obj_ctas][OBJ_W]
  double* rnpart;      // [n_row_ctas][2]
  double* cnpart;      // [fit CTAs][2] column-norm partials (persistent kernel)
  double* blocksum;    // [R][2] (gamma, u) squared norms per row block
  double* bnpart;      // [R][segments][2] partials of k_blocknorm
  // Divergence snapshots are copy-on-write: snap_ver[r] is the snapshot
  // period in which block r's pre-snapshot rows were saved to sn_row.  The
  // snapshot of period k is sn_row for blocks with snap_ver == k and the
  // live theta_row for the others (untouched since the snapshot point).
  long long* snap_ver; // [R]
  int TC, RS, CT;
  int64_t nstar_max, jmax;
  int n_obj_ctas, n_row_ctas, n_col_ctas;
  unsigned long long* prof;   // optional phase timers of k_fit (ns, CTA 0)
};

GMF_D unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

template <typename T>
GMF_D T* tptr(void* p) { return reinterpret_cast<T*>(p); }
template <typename T>
GMF_D const T* tptr(const void* p) { return reinterpret_cast<const T*>(p); }

template <typename T>
GMF_D T ldcg_t(const T* p);
template <>
GMF_D float ldcg_t<float>(const float* p) { return __ldcg(p); }
template <>
GMF_D double ldcg_t<double>(const double* p) { return __ldcg(p); }

// N-wide gathers with branch-free bounds: out-of-range lanes read a clamped
// valid address and are zeroed by a select, so the compiler issues every
// load before the first use (one round trip instead of N)
template <int N, typename T>
GMF_D void gather_vec(const T* base, int count, T (&out)[N]) {
  if (count <= 0) {
    #pragma unroll
    for (int k = 0; k < N; ++k) out[k] = T(0);
    return;
  }
  #pragma unroll
  for (int k = 0; k < N; ++k) {
    const int kk = k < count ? k : 0;
    const T v = base[kk];
    out[k] = k < count ? v : T(0);
  }
}
template <int N, typename T>
GMF_D void gather_vec_cg(const T* base, int64_t stride, int count, T (&out)[N]) {
  #pragma unroll
  for (int k = 0; k < N; ++k) {
    const int kk = k < count ? k : 0;
    const T v = ldcg_t<T>(base + kk * stride);
    out[k] = k < count ? v : T(0);
  }
}

// block-wide sum with the result broadcast to every thread (fixed order)
template <int NT>
GMF_D double block_sum_all(double v, double* scr) {
  double s = block_sum<NT>(v, scr);
  __syncthreads();
  if (threadIdx.x == 0) scr[0] = s;
  __syncthreads();
  s = scr[0];
  __syncthreads();
  return s;
}

// block-wide sums of N values at once (blocks of kThreads), broadcast to every thread; xor
// butterflies give bitwise-identical lane results (a+b == b+a), then a fixed
// warp order (scr >= N * warps doubles)
template <int N, int NT = kThreads>
GMF_D void block_sum_vec(double (&v)[N], double* scr) {
  #pragma unroll
  for (int i = 0; i < N; ++i) {
    #pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[i] += __shfl_xor_sync(0xffffffffu, v[i], o);
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) {
    #pragma unroll
    for (int i = 0; i < N; ++i) scr[wid * N + i] = v[i];
  }
  __syncthreads();
  // warps outer, values inner: N independent add chains (same order per value)
  double s[N];
  #pragma unroll
  for (int i = 0; i < N; ++i) s[i] = 0.0;
  #pragma unroll
  for (int w = 0; w < NT / 32; ++w) {
    #pragma unroll
    for (int i = 0; i < N; ++i) s[i] += scr[w * N + i];
  }
  #pragma unroll
  for (int i = 0; i < N; ++i) v[i] = s[i];
  __syncthreads();
}

// sum of n strided partials published by other CTAs, identical in every
// thread and every CTA that calls it (fixed assignment + fixed tree)
template <int NT>
GMF_D double sum_parts(const double* parts, int64_t n, int64_t stride, double* scr) {
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += NT) s += __ldcg(parts + i * stride);
  return block_sum_all<NT>(s, scr);
}

// ---------------------------------------------------------------------------
// general mode: any family / link at run time (kernels/_ref.py:21-32, 96-117;
// canonical pairs use the reference's simplified forms, the rest the generic
// -w r / (phi nu g'), w / (phi nu g'^2)); pear = w r^2 / nu (optim.py:196-199)
// ---------------------------------------------------------------------------
// general mode marks an unobserved entry of the working response by the least
// significant mantissa bit (observed values have it cleared by the caller: at
// most one ulp; the sign is taken by real-valued responses)
GMF_D bool lsb_set(float v) { return (__float_as_uint(v) & 1u) != 0u; }
GMF_D bool lsb_set(double v) { return (__double_as_longlong(v) & 1ll) != 0ll; }
GMF_D float with_lsb(float v) { return __uint_as_float(__float_as_uint(v) | 1u); }
GMF_D double with_lsb(double v) { return __longlong_as_double(__double_as_longlong(v) | 1ll); }

GMF_D float gexp(float x) { return expf(x); }
GMF_D double gexp(double x) { return exp(x); }
GMF_D float grsqrt(float x) { return 1.f / sqrtf(x); }
GMF_D double grsqrt(double x) { return 1.0 / sqrt(x); }

template <typename T>
GMF_D T gen_mean(int lcode, T eta) {
  switch (lcode) {
    case GMF_IDENTITY: return eta;
    case GMF_LOG: return gexp(eta);
    case GMF_LOGIT: return T(1) / (T(1) + gexp(-eta));
    case GMF_INVERSE: return T(1) / eta;
    default: return grsqrt(eta);
  }
}

template <typename T>
GMF_D T gen_variance(int fcode, T mu, T alpha) {
  switch (fcode) {
    case GMF_GAUSSIAN: return T(1);
    case GMF_GAMMA: return mu * mu;
    case GMF_INV_GAUSSIAN: return mu * mu * mu;
    case GMF_POISSON: return mu;
    case GMF_BERNOULLI: return mu * (T(1) - mu);
    default: return mu * (T(1) + mu / alpha);
  }
}

template <typename T>
GMF_D void gen_derivs(int fcode, int lcode, T y, T mu, T w, T phi, T alpha, T& dd, T& hh, T& pear) {
  const T r = y - mu;
  const T nu = gen_variance<T>(fcode, mu, alpha);
  pear = w * r * r / nu;
  if (fcode == GMF_POISSON && lcode == GMF_LOG) { dd = -w * r / phi; hh = w * mu / phi; return; }
  if (fcode == GMF_BERNOULLI && lcode == GMF_LOGIT) {
    dd = -w * r / phi; hh = w * mu * (T(1) - mu) / phi; return;
  }
  if (fcode == GMF_GAUSSIAN && lcode == GMF_IDENTITY) { dd = -w * r / phi; hh = w / phi; return; }
  if (fcode == GMF_GAMMA && lcode == GMF_INVERSE) { dd = w * r / phi; hh = w * mu * mu / phi; return; }
  if (fcode == GMF_INV_GAUSSIAN && lcode == GMF_INVERSE_SQUARED) {
    dd = w * r / (T(2) * phi); hh = w * mu * mu * mu / (T(4) * phi); return;
  }
  if (fcode == GMF_NEG_BINOMIAL && lcode == GMF_LOG) {
    const T den = T(1) + mu / alpha;
    dd = -w * r / (phi * den); hh = w * mu / (phi * den); return;
  }
  T g1;
  switch (lcode) {
    case GMF_IDENTITY: g1 = T(1); break;
    case GMF_LOG: g1 = T(1) / mu; break;
    case GMF_LOGIT: g1 = T(1) / (mu * (T(1) - mu)); break;
    case GMF_INVERSE: g1 = T(-1) / (mu * mu); break;
    default: g1 = T(-2) / (mu * mu * mu);
  }
  dd = -w * r / (phi * nu * g1);
  hh = w / (phi * nu * g1 * g1);
}

// ---------------------------------------------------------------------------
// tracker decision (optim.py:301-338), from objective totals
// ---------------------------------------------------------------------------
// a mod b for a, b >= 0 through the 32-bit path whenever both fit (a 64-bit
// remainder by a runtime divisor is a long software sequence)
GMF_D long long mod_nn(long long a, long long b) {
  if ((((unsigned long long)a | (unsigned long long)b) >> 32) == 0)
    return (long long)((unsigned int)a % (unsigned int)b);
  return a % b;
}

struct Decision {
  double obj;
  int boundary, snap, stop, conv, div, div_init, streak;
};

GMF_D Decision decide_from(const Params& P, const Ctrl& C, double dev, double ng, double nu,
                           double nb, double nv) {
  Decision D;
  D.obj = 0.0;
  D.boundary = mod_nn(C.t, P.S) == 0;
  D.snap = 0; D.stop = 0; D.conv = C.converged; D.div = 0; D.div_init = 0; D.streak = C.streak;
  if (D.boundary) {
    D.obj = P.escale * dev / (2.0 * C.phi) +
            0.5 * (P.lam_b * nb + P.lam_g * ng + P.lam_u * nu + P.lam_v * nv);
    if (C.t == 0) {
      if (!isfinite(D.obj)) { D.div_init = 1; D.stop = 1; }
      else D.snap = 1;
    } else if (!isfinite(D.obj)) {
      D.div = 1; D.stop = 1;
    } else {
      if (mod_nn(C.trace_len + 1, P.snap_stride) == 0) D.snap = 1;
      const double rel = fabs(D.obj - C.last_obj) / (fabs(C.last_obj) + 1e-12);
      D.streak = rel < P.tol ? D.streak + 1 : 0;
      if (D.streak >= 2) { D.conv = 1; D.stop = 1; }
    }
  }
  if (C.t >= P.max_steps) D.stop = 1;
  return D;
}

// next control block after the decision (and the step, if applied)
GMF_D Ctrl advance(const Params& P, const Ctrl& C, const Decision& D, double nb_num,
                   double nb_den) {
  Ctrl N = C;
  if (D.boundary) {
    N.trace_len = C.trace_len + 1;
    N.last_obj = D.obj;
    N.streak = D.streak;
    N.converged = D.conv;
    N.diverged = D.div;
    N.diverged_init = D.div_init;
  }
  if (D.snap) {
    N.snap_period = C.snap_period + 1;
    N.snapshot_trace_len = N.trace_len;
  }
  if (!D.stop) {
    if (P.est_alpha) {   // optim.py:205-229
      const double rho = P.rho_tab[C.t];
      double ah = nb_den > 0.0 ? nb_num / nb_den : P.nbceil;
      ah = fmin(fmax(P.nbfloor, ah), P.nbceil);
      N.nb_shape = (1.0 - rho) * C.nb_shape + rho * ah;
    }
    if (P.est_phi) {     // optim.py:175-202: nb_num carries sum_B w (y - mu)^2 / nu(mu)
      const double rho = P.rho_tab[C.t];
      const long long s = mod_nn(C.t, P.S);
      const double nJ = (double)(P.cbp[s + 1] - P.cbp[s]);
      const double ph = nb_num * P.rbscale[P.bseq[C.t]] * ((double)P.m / nJ) * P.inv_dof;
      N.phi = (1.0 - rho) * C.phi + rho * ph;
    }
    N.t = C.t + 1;
  }
  N.stopped = D.stop;
  return N;
}

// ---------------------------------------------------------------------------
// EMA + adaptive update of one coordinate (optim.py:450-462)
// ---------------------------------------------------------------------------
// same, with the old theta / EMA values already loaded (prefetched)
template <typename T>
GMF_D T ema_update_from(const Params& P, T* th, T* gb, T* hb, T old, T ogb, T ohb, T gsum, T hsum,
                        double scale, double lam, double rho, double at) {
  const T G = T(scale) * gsum + T(lam) * old;
  const T H = T(scale) * hsum + T(lam);
  const T gn = (T(1) - T(P.a1)) * ogb + T(P.a1) * G;
  const T hn = (T(1) - T(P.a2)) * ohb + T(P.a2) * H;
  *gb = gn;
  *hb = hn;
  const T delta = -T(at) * gn / (hn + T(P.damp));
  const T nv = old + T(rho) * delta;
  *th = nv;
  return nv;
}

template <typename T>
GMF_D T ema_update(const Params& P, T* th, T* gb, T* hb, T gsum, T hsum, double scale, double lam,
                   double rho, double at) {
  return ema_update_from<T>(P, th, gb, hb, *th, *gb, *hb, gsum, hsum, scale, lam, rho, at);
}

}  // namespace gmf
