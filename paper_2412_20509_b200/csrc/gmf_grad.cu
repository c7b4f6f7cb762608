// K1 (fused minibatch gradient) kernels and the persistent fit kernel.
//
//  * k_grad  -- one launch per step (multi-rank path and the standalone
//               minibatch_gradients): K1 tiles + fixed-order reductions into
//               the rank record via "last CTA" tickets.
//  * k_fit   -- single-rank path: ONE cooperative launch runs many aSGD steps;
//               every step is phase 1 (tracked objective partials + K1 tiles),
//               a grid-wide barrier, phase 2 (tracker decision computed
//               redundantly in every CTA, EMA/adaptive updates of rows I and
//               columns J, NB shape), and a second barrier.  Steps are
//               microseconds long and strictly sequential through V, so
//               removing per-kernel launch/drain gaps is the first-order win.
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>

#include "gmf_tc2.cuh"

namespace cg = cooperative_groups;

namespace gmf {

// CTAs per SM the register allocation targets: two for fp32 (the tensor-core
// K1 and the narrow CUDA-core buckets), one for fp64 and for the 64-feature
// bucket, whose shared-memory tile allows one CTA per SM anyway (so it may
// use up to 255 registers instead of spilling at 128)
template <typename T, int NK> struct MinBlocks {
  static constexpr int v = (sizeof(T) == 8 || NK > 32) ? 1 : 2;
};

// threads per CTA of the fit kernel: tc2::NT (320) for the warp-specialized K1 v2
template <int TCM> struct FitNT { static constexpr int v = TCM == 2 ? tc2::NT : kThreads; };

template <typename T, int FAM, int NK, bool TCM>
__global__ void __launch_bounds__(kThreads, MinBlocks<T, NK>::v)
k_grad(Params P, long long xb, long long xs, double xalpha) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ double scr[kThreads / 32];
  __shared__ uint32_t s_tmem;
  __shared__ __align__(8) uint64_t s_bar[2];
  constexpr int TC = TileK<T, NK>::TC;
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
  const int ct = blockIdx.y, rs = blockIdx.x, RS = gridDim.x;
  if constexpr (TCM) {
    tc::Ctx tcx;
    tc::ctx_open(tcx, &s_tmem, s_bar);
    tc::grad_cta<FAM, NK>(P, blk, s, alpha, rs, ct, RS, smem, tcx, nullptr);
    tc::ctx_close(tcx);
  } else {
    // holes: a standalone gradient masks them (gradients.py:66-88); inside
    // the fit they carry the imputed mean, refilled every nafill steps
    // general mode without holes: hmode 3 (y_work is the plain response)
    const int hmode = P.holes ? (xb >= 0 ? 2 : 1) : (FAM == 2 ? 3 : 0);
    const bool fill = hmode == 1 && mod_nn(P.ctrl->t, P.nafill) == 0;
    grad_cta<T, FAM, NK, TC>(P, blk, s, alpha, rs, ct, RS, smem, hmode, fill,
                             xb >= 0 ? P.phi : C->phi);
  }

  (void)TC;
  // (the rank-level column partials are reduced by k_colrec, many CTAs wide)
  // last CTA overall: NB moment sums in fixed CTA order (parallel)
  const unsigned int total = (unsigned int)(RS * gridDim.y);
  if (last_block_ticket(P.tickets + P.CT, total)) {
    const double sn = sum_parts<kThreads>(P.nbpart, total, 2, scr);
    const double sd = sum_parts<kThreads>(P.nbpart + 1, total, 2, scr);
    if (threadIdx.x == 0) {
      P.rec[R_NBNUM] = sn;
      P.rec[R_NBDEN] = sd;
      P.tickets[P.CT] = 0u;
    }
  }
}

// K1 v2 (warp-specialized tensor-core pipeline, gmf_tc2.cuh) for one step:
// one CTA per SM walks the (column tile, row split) units; the last CTA sums
// the per-CTA NB moment partials in fixed order
template <int FAM, int NK>
__global__ void __launch_bounds__(tc2::NT, 1)
k_grad2(Params P, long long xb, long long xs, double xalpha) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ double scr[tc2::NT / 32];
  __shared__ uint32_t s_tmem;
  __shared__ __align__(8) tc2::Bars s_bars;
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
  tc2::Ctx X;
  tc2::ctx_open(X, &s_tmem, &s_bars);
  const unsigned int epoch = *P.rimg_epoch + 1u;   // one image build per launch
  tc2::build_images<NK>(P, blk, P.RS, epoch);
  tc2::grad_units<FAM, NK>(P, blk, s, alpha, P.RS, smem, X, epoch);
  tc2::ctx_close(X);
  const unsigned int total = gridDim.x;
  if (last_block_ticket(P.tickets + P.CT, total)) {
    const double sn = sum_parts<tc2::NT>(P.nbpart, total, 2, scr);
    const double sd = sum_parts<tc2::NT>(P.nbpart + 1, total, 2, scr);
    if (threadIdx.x == 0) {
      P.rec[R_NBNUM] = sn;
      P.rec[R_NBDEN] = sd;
      P.tickets[P.CT] = 0u;
      *P.rimg_epoch = epoch;   // every CTA has read the old value (ticket)
    }
  }
}

// rank-level column partials of the step's column block into the rank record
// (per-step path): a group of 8 lanes per coordinate sums the K1 row splits'
// partials (all loads in flight, fixed xor-butterfly order inside the group)
template <typename T>
__global__ void __launch_bounds__(kThreads) k_colrec(Params P, long long xs) {
  long long s;
  if (xs >= 0) {
    s = xs;
  } else {
    const Ctrl* C = P.ctrl;
    const long long t = C->t;
    if (C->stopped || t >= P.max_steps) return;
    s = t % P.S;
  }
  const int64_t nJ = P.cbp[s + 1] - P.cbp[s];
  const int Kc = P.Kc, kk = 2 * Kc, TC = P.TC, RS = P.RS;
  const int64_t gtid = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  const int sub = threadIdx.x & 7;
  const int64_t e = gtid >> 3;
  const bool live = e < nJ * Kc;
  const uint32_t ue = (uint32_t)(live ? e : 0), pos = ue / (uint32_t)Kc;
  const int k = (int)(ue - pos * (uint32_t)Kc);
  const T* base = tptr<T>(P.colpart) + ((int64_t)(pos / TC) * RS * TC + (pos % TC)) * kk + k;
  const int64_t rstride = (int64_t)TC * kk;
  constexpr int MAXU = 16;
  T g = T(0), h = T(0);
  for (int r0 = 0; r0 < RS; r0 += 8 * MAXU) {
    T gv[MAXU], hv[MAXU];
    #pragma unroll
    for (int u = 0; u < MAXU; ++u) {
      const int r = r0 + sub + 8 * u;
      const int rc = r < RS ? r : 0;
      const T gx = ldcg_t<T>(base + rc * rstride);
      const T hx = ldcg_t<T>(base + rc * rstride + Kc);
      gv[u] = r < RS ? gx : T(0);
      hv[u] = r < RS ? hx : T(0);
    }
    #pragma unroll
    for (int u = 0; u < MAXU; ++u) { g += gv[u]; h += hv[u]; }
  }
  #pragma unroll
  for (int o = 4; o > 0; o >>= 1) {
    g += __shfl_xor_sync(0xffffffffu, g, o);
    h += __shfl_xor_sync(0xffffffffu, h, o);
  }
  if (live && sub == 0) {
    T* recp = reinterpret_cast<T*>(P.rec + REC_HDR);
    recp[(int64_t)pos * kk + k] = g;
    recp[(int64_t)pos * kk + Kc + k] = h;
  }
}

// ---------------------------------------------------------------------------
// persistent fit kernel (single rank)
// ---------------------------------------------------------------------------

// tracked objective of the persistent kernel (optim.py:283-290).  Every row
// with a tracked entry owns a cache slot a_i = [x | u | gamma | 0 | offset]
// (entries carry their slot in ep.w) and the columns' [b | v | z] sit in
// 16-byte padded rows; phase 2 writes both together with theta (one store
// per updated coordinate), so eta is a few 16-byte loads per entry instead of
// ~2K scattered words.  fp64 predictor, fixed order.
template <typename T, int NK>
GMF_D void ecache_fill(const Params& P, int64_t slot, int64_t i) {
  T* row = tptr<T>(P.ecache) + slot * (NK + 4);
  const T* th = tptr<T>(P.th_row) + i * P.Kr;
  const T* xg = tptr<T>(P.x) + i * P.p;
  const int p = P.p, d = P.d, KA = P.KA, q = P.q;
  #pragma unroll
  for (int k = 0; k < NK; ++k) {
    T v = T(0);
    if (k < p) v = xg[k];
    else if (k < p + d) v = th[q + (k - p)];
    else if (k < KA) v = th[k - p - d];
    row[k] = v;
  }
  row[NK] = P.has_off ? tptr<T>(P.off)[i] : T(0);
  row[NK + 1] = T(0); row[NK + 2] = T(0); row[NK + 3] = T(0);
}

template <typename T>
struct Vec16;   // 16-byte vector of T
template <> struct Vec16<float> { using V = float4; static constexpr int N = 4; };
template <> struct Vec16<double> { using V = double2; static constexpr int N = 2; };

template <typename T, int NK, int NT = kThreads, bool GEN = false>
GMF_D double obj_dev_partial(const Params& P, double alpha, const int4* ents, int64_t lo,
                             int64_t hi) {
  using V = typename Vec16<T>::V;
  constexpr int VN = Vec16<T>::N;
  double s = 0.0;
  for (int64_t e = lo + threadIdx.x; e < hi; e += NT) {
    const int4 en = ents[e - lo];
    const int64_t i = en.x, j = en.y;
    const V* a = reinterpret_cast<const V*>(tptr<T>(P.ecache) + (int64_t)en.w * (NK + 4));
    const V* c = reinterpret_cast<const V*>(tptr<T>(P.vpad) + j * NK);
    T av[NK + 4], cv[NK];
    #pragma unroll
    for (int u = 0; u < (NK + 4) / VN; ++u) *reinterpret_cast<V*>(av + VN * u) = a[u];
    #pragma unroll
    for (int u = 0; u < NK / VN; ++u) *reinterpret_cast<V*>(cv + VN * u) = __ldcg(c + u);
    double eta = (double)av[NK];
    #pragma unroll
    for (int k = 0; k < NK; ++k) eta += (double)av[k] * (double)cv[k];
    const double wv = P.has_w ? (double)tptr<T>(P.w)[i * P.m + j] : 1.0;
    if constexpr (GEN)   // general mode: real-valued response, any link (fp64 per-entry algebra)
      s += wv * unit_deviance(P.fam, (double)tptr<T>(P.y_work)[i * P.m + j],
                              gen_mean<double>(P.link, eta), alpha);
    else if (sizeof(T) == 4)   // fp32 path: fp32 transcendentals, fp64 accumulation
      s += wv * (double)unit_deviance_f(P.fam, (float)en.z, __expf((float)eta), (float)alpha);
    else
      s += wv * unit_deviance(P.fam, (double)en.z, exp(eta), alpha);
  }
  return s;
}

// Grid-wide barrier of the tensor-core persistent kernel.  The occupancy
// calculator (and so cudaLaunchCooperativeKernel) caps kernels that allocate
// tensor memory at one CTA per SM, so that kernel is launched normally with
// every CTA co-resident (two per SM: 256 TMEM columns each) and synchronises
// through this counter/generation barrier.  A residency probe at launch
// (short timeout) and a long timeout on every barrier turn a lost CTA into an
// abort flag instead of a hang; the host falls back to one CTA per SM.
GMF_D unsigned int ld_acquire_u32(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

GMF_D unsigned int ld_relaxed_u32(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

GMF_D unsigned long long ld_relaxed_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Barrier state (P.gbar, zeroed at every launch): u32 [1] generation,
// [2] abort flag, u64 at [4] arrivals (monotonic: the k-th barrier of a
// launch completes at G * k arrivals, so no reset RMW is needed).  Every CTA
// counts its barriers in `gen`.  Release: fence.acq_rel + the counting
// atomic; the completing arrival opens the barrier with one generation
// increment after its own fence; waiters spin on relaxed loads (an acquire
// load per iteration would invalidate the SM's L1 every time) and fence once.
GMF_D void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
GMF_D unsigned long long* gbar_count(unsigned int* gb) {
  return reinterpret_cast<unsigned long long*>(gb + 4);
}

GMF_D bool soft_spin(unsigned int* gb, unsigned int gen, unsigned long long timeout_ns) {
  const unsigned long long t0 = gtimer();
  while (ld_relaxed_u32(gb + 1) == gen) {
    if (ld_relaxed_u32(gb + 2)) return false;
    if (gtimer() - t0 > timeout_ns) { atomicExch(gb + 2, 1u); return false; }
  }
  return true;
}

GMF_D bool soft_grid_sync(unsigned int* gb, unsigned int G, unsigned int& gen,
                          unsigned long long timeout_ns) {
  __shared__ int ok;
  __syncthreads();
  if (threadIdx.x == 0) {
    int res = 1;
    fence_acq_rel_gpu();   // release this CTA's writes
    const unsigned long long target = (unsigned long long)G * (gen + 1);
    if (atomicAdd(gbar_count(gb), 1ull) == target - 1) {
      fence_acq_rel_gpu();   // everyone's writes (acquire) -> the opening (release)
      atomicAdd(gb + 1, 1u);
    } else {
      res = soft_spin(gb, gen, timeout_ns) ? 1 : 0;
      fence_acq_rel_gpu();   // acquire: later loads see other CTAs' writes
    }
    ok = res;
  }
  ++gen;
  __syncthreads();
  return ok != 0;
}

// Split form: arrive (release this CTA's writes, count in) and wait (spin,
// acquire).  Loads issued between the two -- inputs of the next phase that
// the current phase does not write -- overlap the barrier.
struct SoftArrival { unsigned int gen; int last; };

GMF_D void soft_grid_release(unsigned int* gb) {   // one thread of the last arriver
  fence_acq_rel_gpu();
  atomicAdd(gb + 1, 1u);
}

// hold: the last arriver does not open the barrier; it sees every other
// CTA's released writes (fence after its counting atomic), does work the
// whole grid needs once, and opens the barrier with soft_grid_release
GMF_D void soft_grid_arrive(unsigned int* gb, unsigned int G, unsigned int& gen, SoftArrival& a,
                            bool hold = false) {
  __shared__ SoftArrival s_a;
  __syncthreads();
  if (threadIdx.x == 0) {
    SoftArrival r;
    r.gen = gen;
    fence_acq_rel_gpu();   // release this CTA's writes
    const unsigned long long target = (unsigned long long)G * (gen + 1);
    r.last = atomicAdd(gbar_count(gb), 1ull) == target - 1;
    if (r.last) {
      if (hold) fence_acq_rel_gpu();   // acquire side of the other CTAs' releases
      else soft_grid_release(gb);
    }
    s_a = r;
  }
  ++gen;
  __syncthreads();
  a = s_a;
}

GMF_D bool soft_grid_wait(unsigned int* gb, const SoftArrival& a, unsigned long long timeout_ns) {
  __shared__ int ok;
  if (threadIdx.x == 0) {
    int res = 1;
    if (!a.last) {
      res = soft_spin(gb, a.gen, timeout_ns) ? 1 : 0;
      fence_acq_rel_gpu();   // acquire
    }
    ok = res;
  }
  __syncthreads();
  return ok != 0;
}

#ifndef GMF_TOTALS_HOLD
#define GMF_TOTALS_HOLD 1   // the barrier's last arriver reduces the phase-2 totals once
#endif

constexpr unsigned long long kProbeTimeoutNs = 50ull * 1000 * 1000;        // residency probe
constexpr unsigned long long kBarrierTimeoutNs = 10ull * 1000 * 1000 * 1000;  // hang guard

template <typename T>
GMF_D T warp_sum(T v) {
  #pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <typename T, int FAM, int NK, int TCM>
__global__ void __launch_bounds__(FitNT<TCM>::v, TCM == 2 ? 1 : MinBlocks<T, NK>::v)
k_fit(Params P, long long n_steps) {
  constexpr int NT = FitNT<TCM>::v;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ double scr[8 * (NT / 32)];
  __shared__ double s_tot[8];
  __shared__ uint32_t s_tmem;
  __shared__ __align__(8) uint64_t s_bar[2];
  __shared__ __align__(8) tc2::Bars s_bars;
  constexpr int TC = TileK<T, NK>::TC;
  Ctrl C = *P.ctrl;
  if (C.stopped) return;
  tc::Ctx tcx;
  tc2::Ctx tcx2;
  const int G = gridDim.x;
  unsigned int bgen = 0;   // software barriers passed by this CTA (P.gbar zeroed per launch)
  auto gsync = [&](unsigned long long timeout) -> bool {
    if constexpr (TCM) {
      return soft_grid_sync(P.gbar, (unsigned int)G, bgen, timeout);
    } else {
      (void)timeout;
      cg::this_grid().sync();
      return true;
    }
  };
  if constexpr (TCM == 1) {
    tc::ctx_open(tcx, &s_tmem, s_bar);
    // residency probe: a CTA that timed out raised the abort flag before the
    // last arrival could open the barrier, or after it -- every CTA re-reads
    // the flag once the barrier opened, so the launch aborts as a whole
    bool resident = gsync(kProbeTimeoutNs);
    if (resident) {
      __shared__ int s_abort;
      if (threadIdx.x == 0) s_abort = (int)ld_acquire_u32(P.gbar + 2);
      __syncthreads();
      resident = s_abort == 0;
    }
    if (!resident) {   // not every CTA resident: abort, host falls back to one CTA per SM
      tc::ctx_close(tcx);
      return;
    }
  } else if constexpr (TCM == 2) {
    tc2::ctx_open(tcx2, &s_tmem, &s_bars);   // cooperative launch: co-resident by construction
  }
  // K1 v2 operand-row images: one build epoch per step (every CTA reads the
  // counter before the first grid barrier, CTA 0 advances it at the end)
  const unsigned int epoch0 = TCM == 2 ? *P.rimg_epoch : 0u;
  unsigned int epoch_n = epoch0;
  // K1 v1 / CUDA cores: one (column tile, row split) per CTA; v2: units looped
  const int ct = blockIdx.x % P.CT, rs = blockIdx.x / P.CT;
  const int RS = TCM == 2 ? P.RS : G / P.CT;
  const int64_t gstride = (int64_t)G * NT;
  const int64_t gtid = (int64_t)blockIdx.x * NT + threadIdx.x;
  const int lane = threadIdx.x & 31;
  const int64_t gw = gtid >> 5, nw = gstride >> 5;
  const int Kr = P.Kr, Kc = P.Kc, kk = 2 * Kc;
  long long prev_blk = -1;

  // column-norm partials of the current state (phase 2 keeps them current)
  {
    double v[2] = {0.0, 0.0};
    const T* tc = tptr<T>(P.th_col);
    for (int64_t e = gtid; e < P.m * Kc; e += gstride) {
      const double x = (double)tc[e];
      v[(int)(e % Kc) < P.p ? 0 : 1] += x * x;
    }
    block_sum_vec<2, NT>(v, scr);
    if (threadIdx.x == 0) { P.cnpart[2 * blockIdx.x] = v[0]; P.cnpart[2 * blockIdx.x + 1] = v[1]; }
  }

  // this CTA's tracked entries (static for the whole fit) cached in shared memory
  const bool ep_cached = P.ep_cap > 0;
  const int4* ep_src = P.ep;
  if (ep_cached) {
    int4* ep_s = reinterpret_cast<int4*>(smem + P.ep_soff);
    const int64_t per = (P.E + G - 1) / G;
    const int64_t lo = per * blockIdx.x, hi = lo + per < P.E ? lo + per : P.E;
    for (int64_t e = threadIdx.x; e < hi - lo; e += NT) ep_s[e] = P.ep[lo + e];
    __syncthreads();
    ep_src = ep_s;
  }
  const int64_t e_per = (P.E + G - 1) / G;
  const int64_t e_lo = e_per * blockIdx.x < P.E ? e_per * blockIdx.x : P.E;
  const int64_t e_hi = e_lo + e_per < P.E ? e_lo + e_per : P.E;
  {
    // objective caches: every tracked row's slot, every column's padded features
    for (int64_t sl = gtid; sl < P.nslots; sl += gstride) ecache_fill<T, NK>(P, sl, P.srow[sl]);
    const T* tc = tptr<T>(P.th_col);
    const T* zg = tptr<T>(P.z);
    for (int64_t e = gtid; e < P.m * NK; e += gstride) {
      const int64_t j = e / NK;
      const int k = (int)(e % NK);
      T v = T(0);
      if (k < Kc) v = tc[j * Kc + k];
      else if (k < P.KA) v = zg[j * P.q + (k - Kc)];
      tptr<T>(P.vpad)[e] = v;
    }
    if constexpr (TCM == 1) {
      if (P.colimg_on) {   // K1's column-operand images, one task per thread
        const int nt = tc::colimg_tasks<NK>();
        for (int64_t e = gtid; e < (int64_t)P.CT * nt; e += gstride)
          tc::colimg_task<NK>(P, (int)(e / nt), (int)(e % nt));
      }
    } else if constexpr (TCM == 2) {
      if (P.colimg_on) {
        const int nt = tc2::colimg_tasks<NK>();
        for (int64_t e = gtid; e < (int64_t)P.CT * nt; e += gstride)
          tc2::colimg_task<NK>(P, (int)(e / nt), (int)(e % nt));
      }
    }
    if (!gsync(kBarrierTimeoutNs)) n_steps = 0;   // vpad / images complete before the first step
  }
  const bool prof = P.prof != nullptr && blockIdx.x == 0 && threadIdx.x == 0;
  // per-CTA stamps of the last profiled step (block-uniform condition)
  const bool profc = P.prof != nullptr;
  unsigned long long t_a = prof ? gtimer() : 0, t_b;
  for (long long it = 0; it < n_steps; ++it) {
    const long long t = C.t;
    if (profc) { __syncthreads(); if (threadIdx.x == 0) P.prof[16 + 32 * blockIdx.x + 0] = gtimer(); }
    const long long sidx = mod_nn(t, P.S);
    const bool boundary = sidx == 0;
    const bool run_grad = t < P.max_steps;
    const long long blk = run_grad ? (long long)P.bseq[t] : -1;
    const unsigned long long rdy_pre =
        (P.stream_mode && threadIdx.x == 0) ? ld_relaxed_u64(P.ready) : 0ull;
    // ------------------------- phase 1 -------------------------
    if (blockIdx.x == 0 && prev_blk >= 0) {   // row norms of the block updated last step
      double v[2] = {0.0, 0.0};
      for (int i = threadIdx.x; i < G; i += NT) {
        v[0] += __ldcg(P.rnpart + 2 * i);
        v[1] += __ldcg(P.rnpart + 2 * i + 1);
      }
      block_sum_vec<2, NT>(v, scr);
      if (threadIdx.x == 0) { P.blocksum[2 * prev_blk] = v[0]; P.blocksum[2 * prev_blk + 1] = v[1]; }
    }
    if (boundary) {
      // contiguous, equal entry ranges per CTA keep the objective balanced
      double v[1] = {0.0};
      const long long c0 = profc ? clock64() : 0;
      v[0] = obj_dev_partial<T, NK, NT, FAM == 2>(P, C.nb_shape, ep_src + (ep_cached ? 0 : e_lo),
                                                   e_lo, e_hi);
      const long long c1 = profc ? clock64() : 0;
      block_sum_vec<1, NT>(v, scr);
      if (threadIdx.x == 0) P.objpart[OBJ_W * blockIdx.x] = v[0];
      if (profc && threadIdx.x == 0) {   // objective sub-phases (SM clocks): loop, reduction
        atomicAdd(P.prof + 16 + 32 * blockIdx.x + 5, (unsigned long long)(c1 - c0));
        atomicAdd(P.prof + 16 + 32 * blockIdx.x + 6, (unsigned long long)(clock64() - c1));
      }
    }
    if (prof) { t_b = gtimer(); atomicAdd(P.prof + 0, t_b - t_a); t_a = t_b; }
    if (profc) { __syncthreads(); if (threadIdx.x == 0) P.prof[16 + 32 * blockIdx.x + 1] = gtimer(); }
    if constexpr (TCM == 2) {   // this step's operand-row images (before the objective: overlap)
      if (run_grad && !P.stream_mode) tc2::build_images<NK>(P, blk, RS, ++epoch_n);
    }
    if (P.stream_mode && run_grad) {
      // streaming: this step's row block is being uploaded; wait for its flag
      // (read at the start of the step, so a block that arrived long ago
      // costs no round trip here)
      if (threadIdx.x == 0) {
        const unsigned long long want = (unsigned long long)t + 1;
        if (rdy_pre < want) {
          const unsigned long long t0 = gtimer();
          while (ld_relaxed_u64(P.ready) < want) {
            if (gtimer() - t0 > kBarrierTimeoutNs) { atomicExch(P.gbar + 2, 1u); break; }
          }
        }
        fence_acq_rel_gpu();   // acquire: the uploaded block is visible
      }
      __syncthreads();
    }
    if constexpr (TCM == 2) {
      if (run_grad) {
        if (P.stream_mode) tc2::build_images<NK>(P, blk, RS, ++epoch_n);   // after the block arrived
        tc2::grad_units<FAM, NK>(P, blk, sidx, C.nb_shape, RS, smem, tcx2, epoch_n,
                                 profc ? P.prof + 16 + 32 * blockIdx.x + 8 : nullptr);
      }
    } else if (run_grad && rs < RS) {
      if constexpr (TCM == 1)
        tc::grad_cta<FAM, NK>(P, blk, sidx, C.nb_shape, rs, ct, RS, smem, tcx,
                              profc ? P.prof + 16 + 32 * blockIdx.x + 8 : nullptr);
      else grad_cta<T, FAM, NK, TC>(P, blk, sidx, C.nb_shape, rs, ct, RS, smem,
                                    P.holes ? 1 : (FAM == 2 ? 3 : 0),
                                    P.holes && mod_nn(t, P.nafill) == 0, C.phi);
    }
    if (prof) { t_b = gtimer(); atomicAdd(P.prof + 1, t_b - t_a); t_a = t_b; }
    if (profc) { __syncthreads(); if (threadIdx.x == 0) P.prof[16 + 32 * blockIdx.x + 2] = gtimer(); }
    // Phase-2 inputs that phase 1 does not write are read across the barrier
    // so their latency hides behind it: this thread's first two row
    // coordinates (theta, EMA state) and the block's snapshot version.  The
    // tensor-core kernel's split barrier arrives first, so these loads do not
    // hold up the arriving thread's release fence.
    // totals: deviance, ||B||^2, ||V||^2, ||Gamma||^2, ||U||^2, NB moment
    // sums (one merged reduction of the per-CTA partials, fixed order)
    auto phase2_totals = [&](double (&v7)[7]) {
      #pragma unroll
      for (int k = 0; k < 7; ++k) v7[k] = 0.0;
      {   // two slots per thread per pass, every load of a pass in flight together
        const bool tb = boundary, tn = run_grad && (P.est_alpha || P.est_phi);
        const int64_t nmax = (int64_t)G > P.R ? (int64_t)G : P.R;
        for (int64_t i = threadIdx.x; i < nmax; i += 2 * NT) {
          double l[2][7];
          #pragma unroll
          for (int u = 0; u < 2; ++u) {
            const int64_t ii = i + u * NT;
            const bool ig = ii < G, ir = ii < P.R;
            const int64_t ic = ig ? ii : 0, irc = ir ? ii : 0;
            const double o0 = __ldcg(P.objpart + OBJ_W * ic);
            const double c0 = __ldcg(P.cnpart + 2 * ic), c1 = __ldcg(P.cnpart + 2 * ic + 1);
            const double b0 = __ldcg(P.blocksum + 2 * irc), b1 = __ldcg(P.blocksum + 2 * irc + 1);
            const double n0 = __ldcg(P.nbpart + 2 * ic), n1 = __ldcg(P.nbpart + 2 * ic + 1);
            l[u][0] = tb && ig ? o0 : 0.0;
            l[u][1] = tb && ig ? c0 : 0.0;
            l[u][2] = tb && ig ? c1 : 0.0;
            l[u][3] = tb && ir ? b0 : 0.0;
            l[u][4] = tb && ir ? b1 : 0.0;
            l[u][5] = tn && ig ? n0 : 0.0;
            l[u][6] = tn && ig ? n1 : 0.0;
          }
          #pragma unroll
          for (int u = 0; u < 2; ++u) {
            #pragma unroll
            for (int k = 0; k < 7; ++k) v7[k] += l[u][k];
          }
        }
      }
      block_sum_vec<7, NT>(v7, scr);
    };
    SoftArrival arr;
    if constexpr (TCM) {
      // the last CTA to arrive reduces the totals once for the grid, then
      // opens the barrier; the others read 7 doubles after their wait
      soft_grid_arrive(P.gbar, (unsigned int)G, bgen, arr, GMF_TOTALS_HOLD != 0);
      if (GMF_TOTALS_HOLD && arr.last) {
        double t7[7];
        phase2_totals(t7);
        if (threadIdx.x == 0) {
          #pragma unroll
          for (int k = 0; k < 7; ++k) { s_tot[k] = t7[k]; P.totals[k] = t7[k]; }
          soft_grid_release(P.gbar);   // fence, then open
        }
        __syncthreads();
      }
    }
    const long long sv = blk >= 0 ? __ldcg(P.snap_ver + blk) : 0;
    const int64_t rI0 = blk >= 0 ? P.rbp[blk] : 0;
    const int64_t nIK = blk >= 0 ? (P.rbp[blk + 1] - rI0) * Kr : 0;
    T pth[2], pgb[2], phb[2];
    int32_t prs[2];
    #pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int64_t e = gtid + u * gstride;
      const int64_t ec = e < nIK ? e : 0;
      const int64_t o = (rI0 * Kr) + ec;
      pth[u] = ldcg_t<T>(tptr<T>(P.th_row) + o);
      pgb[u] = ldcg_t<T>(tptr<T>(P.gb_row) + o);
      phb[u] = ldcg_t<T>(tptr<T>(P.hb_row) + o);
      const int64_t ii = rI0 + (int64_t)((uint32_t)ec / (uint32_t)Kr);
      prs[u] = P.rslot[ii];
    }
    // and every scalar phase 2 reads (constant through the step)
    const int64_t j0s = blk >= 0 ? P.cbp[sidx] : 0;
    const int64_t nJs = blk >= 0 ? P.cbp[sidx + 1] - j0s : 1;
    const double s_col_pre = blk >= 0 ? P.rbscale[blk] : 0.0;
    const double rho_pre = run_grad ? P.rho_tab[t] : 0.0;
    const double at_pre = run_grad ? P.alpt_tab[t] : 0.0;
    if constexpr (TCM) {
      if (!soft_grid_wait(P.gbar, arr, kBarrierTimeoutNs)) break;
    } else {
      if (!gsync(kBarrierTimeoutNs)) break;
    }
    if (profc) { __syncthreads(); if (threadIdx.x == 0) P.prof[16 + 32 * blockIdx.x + 3] = gtimer(); }
    if (prof) { t_b = gtimer(); atomicAdd(P.prof + 2, t_b - t_a); t_a = t_b; }
    // ------------------------- phase 2 -------------------------
    // totals, redundantly in every CTA: deviance, ||B||^2, ||V||^2,
    // ||Gamma||^2, ||U||^2, NB moment sums (one merged reduction)
    const long long ct0 = profc ? clock64() : 0;
    double v7[7];
    if constexpr (TCM && !GMF_TOTALS_HOLD) {
      phase2_totals(v7);
    } else if constexpr (TCM) {
      if (arr.last) {
        #pragma unroll
        for (int k = 0; k < 7; ++k) v7[k] = s_tot[k];
      } else {
        if (threadIdx.x < 7) s_tot[threadIdx.x] = __ldcg(P.totals + threadIdx.x);
        __syncthreads();
        #pragma unroll
        for (int k = 0; k < 7; ++k) v7[k] = s_tot[k];
      }
    } else {
      phase2_totals(v7);
    }
    if (profc && threadIdx.x == 0)   // phase-2 totals (SM clocks)
      atomicAdd(P.prof + 16 + 32 * blockIdx.x + 7, (unsigned long long)(clock64() - ct0));
    if (prof) { t_b = gtimer(); atomicAdd(P.prof + 6, t_b - t_a); }
    const Decision D = decide_from(P, C, v7[0], v7[3], v7[4], v7[1], v7[2]);
    const bool upd = !D.stop;
    const double rho = upd ? rho_pre : 0.0;
    const double at = upd ? at_pre : 0.0;
    // copy-on-write snapshot of block I (first update after a snapshot point)
    const long long per_now = C.snap_period + (D.snap ? 1 : 0);
    const bool cow = upd && sv != per_now;
    double nrm[4] = {0.0, 0.0, 0.0, 0.0};   // new ||Gamma_I||, ||U_I||, ||B||, ||V|| partials
    // rows of block I
    if (upd) {
      const double s_row = (double)P.m / (double)nJs;
      // the first two elements' row partials, all loads in flight together
      constexpr int RTW = 4;
      T rg[2][RTW], rh[2][RTW];
      {
        const T* rpb = tptr<T>(P.rowpart);
        const int64_t cstride = P.nstar_max * (2 * Kr);
        #pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int64_t e = gtid + u * gstride;
          const uint32_t ue = (uint32_t)(e < nIK ? e : 0), il32 = ue / (uint32_t)Kr;
          const T* src = rpb + (int64_t)il32 * (2 * Kr) + (ue - il32 * (uint32_t)Kr);
          gather_vec_cg<RTW>(src, cstride, P.CT, rg[u]);
          gather_vec_cg<RTW>(src + Kr, cstride, P.CT, rh[u]);
        }
      }
      for (int64_t e = gtid, u = 0; e < nIK; e += gstride, ++u) {
        // 32-bit index split (a 64-bit division by a runtime divisor is a
        // long software sequence); e < |I| (q+d) < 2^31
        const uint32_t ue = (uint32_t)e, il32 = ue / (uint32_t)Kr;
        const int64_t il = il32;
        const int k = (int)(ue - il32 * (uint32_t)Kr);
        const int64_t o = rI0 * Kr + e;
        T gs, hs;
        if (u < 2) {   // tiles in the same fixed order as rowpart_sum
          gs = T(0);
          hs = T(0);
          #pragma unroll
          for (int c = 0; c < RTW; ++c) { gs += rg[u][c]; hs += rh[u][c]; }
          for (int c0 = RTW; c0 < P.CT; c0 += RTW) {
            T gv[RTW], hv[RTW];
            const int64_t cstride = P.nstar_max * (2 * Kr);
            const T* src = tptr<T>(P.rowpart) + il * (2 * Kr) + k + c0 * cstride;
            gather_vec_cg<RTW>(src, cstride, P.CT - c0, gv);
            gather_vec_cg<RTW>(src + Kr, cstride, P.CT - c0, hv);
            #pragma unroll
            for (int c = 0; c < RTW; ++c) { gs += gv[c]; hs += hv[c]; }
          }
        } else {
          rowpart_sum<T>(P, il, k, gs, hs);
        }
        const T old = u < 2 ? pth[u] : ldcg_t<T>(tptr<T>(P.th_row) + o);
        const T ogb = u < 2 ? pgb[u] : ldcg_t<T>(tptr<T>(P.gb_row) + o);
        const T ohb = u < 2 ? phb[u] : ldcg_t<T>(tptr<T>(P.hb_row) + o);
        if (cow) tptr<T>(P.sn_row)[o] = old;
        const double lam = k < P.q ? P.lam_g : P.lam_u;
        const T G_ = T(s_row) * gs + T(lam) * old;
        const T H_ = T(s_row) * hs + T(lam);
        const T gn = (T(1) - T(P.a1)) * ogb + T(P.a1) * G_;
        const T hn = (T(1) - T(P.a2)) * ohb + T(P.a2) * H_;
        const T nvv = old + T(rho) * (-T(at) * gn / (hn + T(P.damp)));
        tptr<T>(P.gb_row)[o] = gn;
        tptr<T>(P.hb_row)[o] = hn;
        tptr<T>(P.th_row)[o] = nvv;
        {   // the objective's cache rows of this row's tracked entries
          const int64_t i = rI0 + il;
          const int apos = k < P.q ? P.p + P.d + k : P.p + (k - P.q);   // a = [x | u | gamma]
          const int32_t sl = u < 2 ? prs[u] : P.rslot[i];
          if (sl >= 0) tptr<T>(P.ecache)[(int64_t)sl * (NK + 4) + apos] = nvv;
        }
        const double sq = (double)nvv * (double)nvv;   // register selects, no local array
        if (k < P.q) nrm[0] += sq; else nrm[1] += sq;
      }
    }
    if (prof) { t_b = gtimer(); atomicAdd(P.prof + 7, t_b - t_a); }
    // columns of block J.  A task is CG whole columns of one K1 column tile:
    // their partials are CG * 2Kc contiguous values per row split, so the
    // CTA's lanes read them coalesced (lane -> value, S lane groups -> row
    // splits, all of a thread's loads in flight), reduce across the S groups
    // in shared memory (K1's, idle in phase 2) in a fixed order, and the
    // first CG * Kc threads update one coordinate each
    if (upd) {
      const int64_t j0 = j0s, nJ = nJs;
      const double s_col = s_col_pre;
      const T* cpart = tptr<T>(P.colpart);
      const int64_t rstride = (int64_t)TC * kk;
      int CG = 1;
      while (2 * CG * kk <= 64 && 2 * CG <= TC) CG *= 2;   // divides TC (a power of two)
      const int EQ = CG * kk, S = NT / EQ;
      const int qv = threadIdx.x % EQ, sg = threadIdx.x / EQ;
      T* red = reinterpret_cast<T*>(smem);
      const int64_t ntask = (nJ + CG - 1) / CG;
      constexpr int MAXU = 16;
      for (int64_t task = blockIdx.x; task < ntask; task += G) {
        const int64_t pos0 = task * CG;
        if (sg < S) {
          const T* base = cpart + ((pos0 / TC) * RS * TC + (pos0 % TC)) * kk + qv;
          T acc = T(0);
          for (int r0 = sg; r0 < RS; r0 += S * MAXU) {
            T v[MAXU];
            #pragma unroll
            for (int u = 0; u < MAXU; ++u) {
              const int r = r0 + u * S;
              v[u] = r < RS ? ldcg_t<T>(base + r * rstride) : T(0);
            }
            #pragma unroll
            for (int u = 0; u < MAXU; ++u) acc += v[u];
          }
          red[sg * EQ + qv] = acc;
        }
        __syncthreads();
        if (threadIdx.x < CG * Kc) {
          const int c = threadIdx.x / Kc, k = threadIdx.x - c * Kc;
          const int64_t pos = pos0 + c;
          if (pos < nJ) {
            T g = T(0), h = T(0);
            for (int ss = 0; ss < S; ++ss) {
              g += red[ss * EQ + c * kk + k];
              h += red[ss * EQ + c * kk + Kc + k];
            }
            const int64_t j = P.col_identity ? pos : (int64_t)P.cidx[j0 + pos];
            T* th = tptr<T>(P.th_col) + j * Kc + k;
            if (D.snap) tptr<T>(P.sn_col)[j * Kc + k] = *th;
            const T nvv = ema_update<T>(P, th, tptr<T>(P.gb_col) + j * Kc + k,
                                        tptr<T>(P.hb_col) + j * Kc + k, g, h, s_col,
                                        k < P.p ? P.lam_b : P.lam_v, rho, at);
            tptr<T>(P.vpad)[j * NK + k] = nvv;   // the objective's padded copy of [b | v | z]
            if constexpr (TCM == 1) {
              if (P.colimg_on) tc::colimg_write<NK>(P, j, k, (float)nvv);
            } else if constexpr (TCM == 2) {
              if (P.colimg_on) tc2::colimg_write<NK>(P, j, k, (float)nvv);
            }
            const double sq = (double)nvv * (double)nvv;
            if (k < P.p) nrm[2] += sq; else nrm[3] += sq;
          }
        }
        __syncthreads();
      }
    }
    if (prof) { t_b = gtimer(); atomicAdd(P.prof + 8, t_b - t_a); }
    // columns outside J: snapshot and norms (nothing to do when J = all)
    if ((upd || D.snap) && !(upd && P.col_identity)) {
      const T* tc = tptr<T>(P.th_col);
      for (int64_t e = gtid; e < P.m * Kc; e += gstride) {
        const int64_t j = (int64_t)((uint64_t)e / (uint64_t)Kc);
        if (upd && P.cbof[j] == sidx) continue;
        const T x = tc[e];
        if (D.snap) tptr<T>(P.sn_col)[e] = x;
        const double sq = (double)x * (double)x;
        if ((int)(e - j * Kc) < P.p) nrm[2] += sq; else nrm[3] += sq;
      }
    }
    if (prof) { t_b = gtimer(); atomicAdd(P.prof + 9, t_b - t_a); }
    block_sum_vec<4, NT>(nrm, scr);
    if (prof) { t_b = gtimer(); atomicAdd(P.prof + 10, t_b - t_a); }
    if (threadIdx.x == 0) {
      P.rnpart[2 * blockIdx.x] = nrm[0];
      P.rnpart[2 * blockIdx.x + 1] = nrm[1];
      if (upd) {
        P.cnpart[2 * blockIdx.x] = nrm[2];
        P.cnpart[2 * blockIdx.x + 1] = nrm[3];
      }
    }
    const Ctrl N = advance(P, C, D, v7[5], v7[6]);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      if (D.boundary) {
        P.trace_obj[C.trace_len] = D.obj;
        P.trace_nb[C.trace_len] = C.nb_shape;
    P.trace_phi[C.trace_len] = C.phi;
      }
      if (cow) P.snap_ver[blk] = per_now;
      *P.ctrl = N;
    }
    C = N;
    prev_blk = upd ? blk : -1;
    if (prof) { t_b = gtimer(); atomicAdd(P.prof + 3, t_b - t_a); t_a = t_b; }
    if (profc) { __syncthreads(); if (threadIdx.x == 0) P.prof[16 + 32 * blockIdx.x + 4] = gtimer(); }
    // per-step status word to pinned host memory, written after the barrier:
    // a system-memory store ahead of a barrier's gpu-scope fence would hold
    // that fence for a PCIe round trip
    const bool host_w = P.host_status && blockIdx.x == 0 && threadIdx.x == 0;
    if (D.stop) {
      if (host_w) reinterpret_cast<Ctrl*>(P.host_status)[it] = N;
      break;
    }
    if (!gsync(kBarrierTimeoutNs)) break;
    if (host_w) reinterpret_cast<Ctrl*>(P.host_status)[it] = N;
    if (prof) { t_b = gtimer(); atomicAdd(P.prof + 4, t_b - t_a); t_a = t_b; atomicAdd(P.prof + 5, 1ull); }
  }
  if (blockIdx.x == 0 && prev_blk >= 0) {
    double v[2] = {0.0, 0.0};
    for (int i = threadIdx.x; i < G; i += NT) {
      v[0] += __ldcg(P.rnpart + 2 * i);
      v[1] += __ldcg(P.rnpart + 2 * i + 1);
    }
    block_sum_vec<2, NT>(v, scr);
    if (threadIdx.x == 0) { P.blocksum[2 * prev_blk] = v[0]; P.blocksum[2 * prev_blk + 1] = v[1]; }
  }
  if constexpr (TCM == 1) tc::ctx_close(tcx);
  else if constexpr (TCM == 2) {
    tc2::ctx_close(tcx2);
    if (blockIdx.x == 0 && threadIdx.x == 0) *P.rimg_epoch = epoch_n;
  }
}

// ---------------------------------------------------------------------------
// host side: dispatch over (dtype, family, feature bucket)
// ---------------------------------------------------------------------------
template <typename T, int FAM, int NK, int TCM>
struct Inst {
  static void* grad() {
    if constexpr (TCM == 2) return (void*)k_grad2<FAM, NK>;
    else return (void*)k_grad<T, FAM, NK, TCM != 0>;
  }
  static void* fit() { return (void*)k_fit<T, FAM, NK, TCM>; }
};

template <typename T, int FAM, int TCM>
static void* pick(int NK, bool fit) {
  if constexpr (FAM == 2) {   // general mode: two feature buckets (build time)
    switch (NK) {
      case 16: return fit ? Inst<T, 2, 16, 0>::fit() : Inst<T, 2, 16, 0>::grad();
      case 32: return fit ? Inst<T, 2, 32, 0>::fit() : Inst<T, 2, 32, 0>::grad();
      default: return nullptr;
    }
  } else {
  switch (NK) {
    case 8: return fit ? Inst<T, FAM, 8, TCM>::fit() : Inst<T, FAM, 8, TCM>::grad();
    case 12: return fit ? Inst<T, FAM, 12, TCM>::fit() : Inst<T, FAM, 12, TCM>::grad();
    case 16: return fit ? Inst<T, FAM, 16, TCM>::fit() : Inst<T, FAM, 16, TCM>::grad();
    case 24: return fit ? Inst<T, FAM, 24, TCM>::fit() : Inst<T, FAM, 24, TCM>::grad();
    case 32: return fit ? Inst<T, FAM, 32, TCM>::fit() : Inst<T, FAM, 32, TCM>::grad();
    case 64:   // K = p+q+d in (32, 64]: CUDA-core K1 only (c5's rank 50)
      if constexpr (!TCM)
        return fit ? Inst<T, FAM, 64, 0>::fit() : Inst<T, FAM, 64, 0>::grad();
      return nullptr;
    default: return nullptr;
  }
  }
}

// tcm: K1 on the tensor cores (fp32 only; gmf_tc.cuh)
static void* kernel_for(int dtype, int family, int NK, bool fit, int tcm, int gen = 0) {
  if (gen) return dtype == GMF_F64 ? pick<double, 2, 0>(NK, fit) : pick<float, 2, 0>(NK, fit);
  const int fam = family == GMF_NEG_BINOMIAL ? 1 : 0;
  if (dtype == GMF_F64) return fam ? pick<double, 1, 0>(NK, fit) : pick<double, 0, 0>(NK, fit);
  if (tcm == 2) return fam ? pick<float, 1, 2>(NK, fit) : pick<float, 0, 2>(NK, fit);
  if (tcm) return fam ? pick<float, 1, 1>(NK, fit) : pick<float, 0, 1>(NK, fit);
  return fam ? pick<float, 1, 0>(NK, fit) : pick<float, 0, 0>(NK, fit);
}

static int k1_threads(int tcm) { return tcm == 2 ? tc2::NT : kThreads; }

int64_t rimg_bytes_of(int NK) { return tc2::rimg_bytes(NK); }

int tc_eligible(int dtype, int has_w, int Kr, int Kc, int KA, int holes) {
  return dtype == GMF_F32 && !has_w && !holes && Kr <= 16 && Kc <= 16 && KA <= 32;
}

int grad_bucket_gen(int KA) { return KA <= 16 ? 16 : (KA <= 32 ? 32 : -1); }

int grad_bucket(int KA) {
  if (KA <= 8) return 8;
  if (KA <= 12) return 12;
  if (KA <= 16) return 16;
  if (KA <= 24) return 24;
  if (KA <= 32) return 32;
  if (KA <= 64) return 64;
  return -1;
}

int tile_cols(int dtype, int NK) {
  if (NK > 32) return dtype == GMF_F64 ? TileK<double, 64>::TC : TileK<float, 64>::TC;
  return dtype == GMF_F64 ? Tile<double>::TC : Tile<float>::TC;
}

int64_t colimg_bytes_total(int NK, int CT, int tcm) {
  return (int64_t)CT * (tcm == 2 ? tc2::colimg_bytes(NK) : tc::colimg_bytes(NK));
}

static int csr_kind(int yfmt) { return yfmt == GMF_Y_DENSE_I32 ? 0 : (yfmt == GMF_Y_CSR_PACK32 ? 2 : 1); }

// dynamic shared memory of K1 (the fit kernel adds its cached tracked entries)
int64_t grad_smem_bytes(const Params& P, int dtype, int NK) {
  if (P.tcm == 2) return tc2::layout(NK, P.Kr, P.p, csr_kind(P.yfmt), P.k1_cap, P.k1_na1).total;
  if (P.tcm) return tc::smem_layout(NK).total;
  return grad_smem(tile_cols(dtype, NK), NK, dtype == GMF_F64 ? 8 : 4, P.has_w, P.Kr, P.Kc).total;
}

// opt in to >48 KB dynamic shared memory (outside any graph capture) and
// report how many k_fit CTAs can be co-resident per SM
int prepare_grad(const Params& P, int dtype, int NK, int fit_extra_smem, int* fit_blocks_per_sm) {
  const int tcm = P.tcm;
  void* g = kernel_for(dtype, P.fam, NK, false, tcm, P.gen);
  void* f = kernel_for(dtype, P.fam, NK, true, tcm, P.gen);
  if (!g || !f) { set_error("unsupported feature bucket %d", NK); return GMF_ERR_UNSUPPORTED; }
  const int nt = k1_threads(tcm);
  const int smem_g = (int)grad_smem_bytes(P, dtype, NK);
  const int smem = smem_g + fit_extra_smem;
  GMF_CUDA(cudaFuncSetAttribute(g, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_g));
  GMF_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  int nb = 0;
  GMF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, f, nt, smem));
  if (tcm == 1) {
    // The occupancy calculator caps kernels that allocate tensor memory at one
    // CTA per SM; each K1 v1 CTA takes 256 of the 512 TMEM columns, so the SM
    // holds as many as registers and shared memory allow, up to two.
    cudaFuncAttributes a;
    GMF_CUDA(cudaFuncGetAttributes(&a, f));
    int dev = 0, smem_sm = 0, regs_sm = 0;
    GMF_CUDA(cudaGetDevice(&dev));
    GMF_CUDA(cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev));
    GMF_CUDA(cudaDeviceGetAttribute(&regs_sm, cudaDevAttrMaxRegistersPerMultiprocessor, dev));
    const int by_smem = smem_sm / (int)(smem + a.sharedSizeBytes + 1024);
    const int by_regs = regs_sm / (((a.numRegs + 7) / 8) * 8 * kThreads);
    int v = by_smem < by_regs ? by_smem : by_regs;
    if (v > (int)(512 / tc::kCols)) v = (int)(512 / tc::kCols);
    if (v > nb) nb = v;
  }
  *fit_blocks_per_sm = nb;
  if (getenv("GMF_VERBOSE")) {
    for (void* k : {g, f}) {
      cudaFuncAttributes a;
      cudaFuncGetAttributes(&a, k);
      int n1 = 0, n2 = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n1, k, nt, smem);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n2, k, nt, 0);
      fprintf(stderr, "[gmf] %s kernel (K1 %s): regs %d static smem %zu dyn smem %d (max %d) local %zu maxthreads %d -> %d CTAs/SM (%d without dyn smem)\n",
              k == f ? "fit" : "grad", tcm == 2 ? "tc v2" : (tcm ? "tc v1" : "cuda cores"), a.numRegs,
              a.sharedSizeBytes, smem, a.maxDynamicSharedSizeBytes, a.localSizeBytes,
              a.maxThreadsPerBlock, n1, n2);
    }
  }
  return GMF_OK;
}

int launch_grad(const Params& P, int dtype, int NK, cudaStream_t st, long long xb, long long xs,
                double xalpha) {
  void* f = kernel_for(dtype, P.fam, NK, false, P.tcm, P.gen);
  if (!f) { set_error("unsupported feature bucket %d", NK); return GMF_ERR_UNSUPPORTED; }
  dim3 grid(P.RS, P.CT);
  if (P.tcm == 2) {   // one CTA per SM walking the CT x RS units
    int dev = 0, n_sm = kSMs;
    GMF_CUDA(cudaGetDevice(&dev));
    GMF_CUDA(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev));
    const int64_t units = (int64_t)P.RS * P.CT;
    grid = dim3((unsigned)(units < n_sm ? units : n_sm));
  }
  const size_t smem = (size_t)grad_smem_bytes(P, dtype, NK);
  void* args[] = {(void*)&P, (void*)&xb, (void*)&xs, (void*)&xalpha};
  GMF_CUDA(cudaLaunchKernel(f, grid, dim3(k1_threads(P.tcm)), args, smem, st));
  return GMF_OK;
}

int launch_colrec(const Params& P, int dtype, cudaStream_t st, long long xs) {
  const int64_t ne = P.jmax * P.Kc;
  const unsigned blocks = (unsigned)((ne * 8 + kThreads - 1) / kThreads);
  void* args[] = {(void*)&P, (void*)&xs};
  void* f = dtype == GMF_F64 ? (void*)k_colrec<double> : (void*)k_colrec<float>;
  GMF_CUDA(cudaLaunchKernel(f, dim3(blocks > 0 ? blocks : 1), dim3(kThreads), args, 0, st));
  return GMF_OK;
}

int launch_fit(const Params& P, int dtype, int NK, int grid, long long n_steps, cudaStream_t st) {
  void* f = kernel_for(dtype, P.fam, NK, true, P.tcm, P.gen);
  if (!f) { set_error("unsupported feature bucket %d", NK); return GMF_ERR_UNSUPPORTED; }
  const size_t smem = (size_t)grad_smem_bytes(P, dtype, NK) + (size_t)P.ep_cap * sizeof(int4);
  Params Q = P;
  Q.colimg_on = P.tcm && P.colimg != nullptr;   // images maintained by k_fit's own updates
  void* args[] = {(void*)&Q, (void*)&n_steps};
  if (P.tcm == 1) {   // software grid barrier (soft_grid_sync): plain launch, fresh counters
    GMF_CUDA(cudaMemsetAsync(P.gbar, 0, 32, st));
    GMF_CUDA(cudaLaunchKernel(f, dim3(grid), dim3(kThreads), args, smem, st));
  } else {
    // cooperative launch: every CTA co-resident by construction (K1 v2 runs
    // one CTA per SM and synchronises through the software barrier)
    if (P.tcm == 2) GMF_CUDA(cudaMemsetAsync(P.gbar, 0, 32, st));
    GMF_CUDA(cudaLaunchCooperativeKernel(f, dim3(grid), dim3(k1_threads(P.tcm)), args, smem, st));
  }
  return GMF_OK;
}

}  // namespace gmf
