// K1 v2 on the 5th-generation tensor cores (fp32 path): a warp-specialized
// tcgen05 pipeline, one CTA (320 threads: 8 elementwise warps, the MMA warp,
// the loader warp) per SM.
//
// Same contract as tc::grad_cta / grad_cta: for every work unit (column tile
// ct of block J x a balanced contiguous row range rs of block I) it writes
// rowpart[ct][row][2Kr] and colpart[ct][rs][c][2Kc]; the NB moment sums go to
// nbpart[blockIdx.x] (one pair per CTA, summed over its units).  A CTA walks
// units blockIdx.x, +G, ... and each unit in 64-row chunks.  Per chunk:
//
//   GEMM1  eta[128 x 128] = A1 . B1^T      M = the chunk's 64 rows twice (TMEM
//          lanes 0-63 and 64-127 hold the same rows, so warps of lane quarters
//          0-1 read tile columns 0-63 and warps of quarters 2-3 columns
//          64-127), N = 128 tile columns, K = the features
//          a = [x | u | gamma | offset], c = [b | v | z | 1] * log2 e.
//          fp32 accuracy from a three-way bf16 split x = x0 + x1 + x2:
//          x0y0 + x0y1 + x1y0 + x0y2 + x1y1 + x2y0 (error ~2^-24 |x||y|)
//   elementwise (8 warps, thread = one chunk row x 32 tile columns):
//          mu = 2^eta, dotD / ddotD (NB or Poisson, log link), NB moments,
//          written as two stacked bf16 tiles P_g (g = rows 0-31, 32-63; each
//          dd rows then hh rows, hi and lo split rows 8 apart: tc::stack_hi)
//   GEMM2  D2_g[128 x 64] = P_g . R        row side, K = tile columns
//   GEMM3  D3[128 x 64]  += P_g^T . [A3_g | A3sq_g]   column side, K = rows,
//          accumulated over every chunk of the unit (TMEM)
//
// Roles (mbarrier hand-offs, no CTA-wide barrier inside a unit):
//   warps 0-7  elementwise; they also build the next chunk's A1 (right after
//              reading this chunk's eta, so GEMM1 of c+1 overlaps chunk c)
//              and A3, read D2 (row partials) and, at the unit's end, D3
//              (column partials); dense Y is loaded straight into registers
//              one chunk ahead (the loader prefetches it into L2 two ahead)
//   warp 8     TMEM owner; lane 0 issues every MMA: GEMM1(c) then GEMM2/3(c-1)
//   warp 9     loader: TMA bulk copies of the row features and of the
//              chunk's tile-CSR entries two chunks ahead (a few copies per
//              chunk), and the lane-parallel scatter of the entries into the
//              Y tile
// Buffers: eta double-buffered in TMEM (the elementwise pass of chunk c
// overlaps GEMM1 of c+1), A3 double-buffered, staging ring of 3, A1 / P /
// D2 / Y single.
//
// TMEM (512 columns, one CTA per SM): eta 0 / 128, D2_0 256, D2_1 320, D3 384.
// Shared-memory operand layouts are tc::'s (verified: tools/umma_test.cu).
#pragma once
#include "gmf_tc.cuh"

namespace gmf {
namespace tc2 {

using tc::kofs;
using tc::a1ofs;
using tc::stack_hi;
using tc::smem_addr;
using tc::sdesc;
using tc::idesc;
using tc::umma;
using tc::umma_commit;
using tc::fence_before;
using tc::fence_after;
using tc::fence_async_smem;
using tc::SBO_P;

constexpr int NT = 320;              // threads per CTA
constexpr int NEW = 8;               // elementwise warps 0..7
constexpr int MMA_WARP = 8;
constexpr int LDW = 9;               // loader warp
constexpr int CR = 64;               // distinct rows per chunk
constexpr int TCC = 128;             // tile columns
constexpr int YP = 132;              // Y tile pitch (floats)
constexpr int NSLOT = 3;             // staging ring depth (chunks in flight)
constexpr uint32_t kCols = 512;
constexpr uint32_t T_D2 = 256, T_D3 = 384;
constexpr float kLog2e = 1.4426950408889634f;

// ---------------------------------------------------------------------------
// shared-memory layout (host and device compute it identically)
// ---------------------------------------------------------------------------
struct Lay {
  int64_t R, B1, A1, A3, P, Y, nstage, total;
  int nka, cap, nslot_bytes, na1;
};

GMF_HD int64_t al128(int64_t v) { return (v + 127) & ~int64_t(127); }
GMF_HD int64_t al16(int64_t v) { return (v + 15) & ~int64_t(15); }

// bytes of one chunk's operand-row image (K1 v2 pre-pass): A1 of the
// chunk's 64 rows (three splits) then A3 / A3sq, the shared-memory layouts
GMF_HD int64_t rimg_bytes(int NK) {
  const int nka = NK <= 16 ? 16 : 32;
  return (int64_t)3 * CR * nka * 2 + 8192;
}

// csr: 0 dense, 1 CSR (col + val words), 2 packed CSR; cap = staged nonzeros per
// slot; na1 = A1 buffers (2: the builders run a chunk ahead of GEMM1)
GMF_HD Lay layout(int NK, int Kr, int p, int csr, int cap, int na1) {
  Lay L;
  L.nka = NK <= 16 ? 16 : 32;
  L.cap = csr ? cap : 0;
  L.na1 = na1;
  int64_t o = 0;
  L.R = o; o = al128(o + 64 * TCC * 2);
  L.B1 = o; o = al128(o + 3 * TCC * L.nka * 2);          // three splits
  L.A1 = o; o = al128(o + (int64_t)na1 * 3 * 128 * L.nka * 2);   // three splits, 128 M rows
  L.A3 = o; o = al128(o + 2 * 2 * 4096);                  // 2 slots x (a0|a1, sq0|sq1)
  L.P = o; o = al128(o + 2 * 32768);                       // two stacked 32-row groups
  L.Y = o; o = al128(o + (csr ? 2 : 1) * CR * YP * 4);   // CSR: two Y tiles (scatter a chunk ahead)
  // CSR staging slot: meta (8 int32: entry offset, count, fits, -, first entry
  // int64) | cap tile-CSR entries (int2)
  L.nslot_bytes = csr ? (int)al16(8 * 4 + (int64_t)cap * 8) : 0;
  L.nstage = o; o = al128(o + (int64_t)NSLOT * L.nslot_bytes);
  L.total = o;
  return L;
}

// column-operand image of one tile: R | B1 (3 splits), the shared-memory bytes
GMF_HD int64_t colimg_bytes(int NK) {
  const int nka = NK <= 16 ? 16 : 32;
  return (int64_t)64 * TCC * 2 + 3 * (int64_t)TCC * nka * 2;
}

using tc::split3_8;

GMF_D void split3_1(float x, __nv_bfloat16& a, __nv_bfloat16& b, __nv_bfloat16& c) {
  a = __float2bfloat16_rn(x);
  const float r = x - __bfloat162float(a);
  b = __float2bfloat16_rn(r);
  c = __float2bfloat16_rn(r - __bfloat162float(b));
}

// Two sentinel features after [x | u | gamma | offset] make eta of an entry
// outside the block -1000 (mu = 2^-1000 = 0 after ftz), so the elementwise
// pass needs no masks: feature kone = 1 for every row and 0 / -1000 for a
// valid / invalid column; feature kone + 1 = 0 / -1000 for a valid / invalid
// row and 1 for every column.
constexpr float kSentinel = -1000.f;
GMF_HD int kone_of(const Params& P) { return P.KA + (P.has_off ? 1 : 0); }

// B1 entry of column j (feature k), prescaled by log2 e; ok: column inside the block
GMF_D float b1_value(const Params& P, int64_t j, int k, bool ok) {
  const int kone = kone_of(P);
  if (k == kone) return ok ? 0.f : kSentinel;
  if (k == kone + 1) return 1.f;
  if (!ok) return 0.f;
  const float* th_col = tptr<float>(P.th_col);
  const float* zg = tptr<float>(P.z);
  float x = 0.f;
  if (k < P.Kc) x = th_col[j * P.Kc + k];
  else if (k < P.KA) x = zg[j * P.q + (k - P.Kc)];
  else if (k == P.KA && P.has_off) x = 1.f;
  return x * kLog2e;
}

// ---- column-operand images (persistent kernel, all columns every step) ----
template <int NK>
GMF_HD int colimg_tasks() { return 16 * (TCC / 8) + TCC * ((NK <= 16 ? 16 : 32) / 8); }

// task t of column tile ct: R rows (feature k, 8 columns) then B1 rows
// (column, 8 features), written into the tile's image (dst: image base) or
// straight into shared memory (same byte layout)
template <int NK>
GMF_D void colop_task(const Params& P, unsigned char* dst, int64_t cbase, int ncv, int t,
                      const int32_t* cmap = nullptr) {
  // cmap: column of each block position (null: identity, J = all columns)
  auto col = [&](int c) -> int64_t { return cmap ? (int64_t)cmap[cbase + c] : cbase + c; };
  constexpr int nka = NK <= 16 ? 16 : 32, ng1 = nka / 8;
  constexpr uint32_t sbo1 = (uint32_t)ng1 * 128u;
  constexpr int64_t b1sz = (int64_t)TCC * nka * 2;
  const float* th_col = tptr<float>(P.th_col);
  const float* zg = tptr<float>(P.z);
  const int Kr = P.Kr, Kc = P.Kc, p = P.p, q = P.q;
  if (t < 16 * (TCC / 8)) {
    const int rk = t / (TCC / 8), rcg = t % (TCC / 8);
    float v[8], v2[8];
    #pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int c = 8 * rcg + u;
      const bool ok = c < ncv && rk < Kr;
      const int64_t j = ok ? col(c) : 0;
      v[u] = !ok ? 0.f : (rk < q ? zg[j * q + rk] : th_col[j * Kc + p + (rk - q)]);
      v2[u] = v[u] * v[u];
    }
    uint4 h, l, h2, l2;
    tc::split8(v, h, l);
    tc::split8(v2, h2, l2);
    *reinterpret_cast<uint4*>(dst + kofs(rk, 8 * rcg, SBO_P)) = h;
    *reinterpret_cast<uint4*>(dst + kofs(16 + rk, 8 * rcg, SBO_P)) = l;
    *reinterpret_cast<uint4*>(dst + kofs(32 + rk, 8 * rcg, SBO_P)) = h2;
    *reinterpret_cast<uint4*>(dst + kofs(48 + rk, 8 * rcg, SBO_P)) = l2;
    return;
  }
  t -= 16 * (TCC / 8);
  if (t >= TCC * ng1) return;
  const int c = t / ng1, g = t % ng1;
  const bool ok = c < ncv;
  float v[8];
  #pragma unroll
  for (int u = 0; u < 8; ++u) v[u] = b1_value(P, ok ? col(c) : 0, 8 * g + u, ok);
  uint4 s0, s1, s2;
  split3_8(v, s0, s1, s2);
  unsigned char* B1 = dst + 64 * TCC * 2;
  *reinterpret_cast<uint4*>(B1 + kofs(c, 8 * g, sbo1)) = s0;
  *reinterpret_cast<uint4*>(B1 + b1sz + kofs(c, 8 * g, sbo1)) = s1;
  *reinterpret_cast<uint4*>(B1 + 2 * b1sz + kofs(c, 8 * g, sbo1)) = s2;
}

template <int NK>
GMF_D void colimg_task(const Params& P, int ct, int t) {
  unsigned char* img = reinterpret_cast<unsigned char*>(P.colimg) + (int64_t)ct * colimg_bytes(NK);
  const int64_t cbase = (int64_t)ct * TCC;
  const int ncv = (int)(P.m - cbase < TCC ? P.m - cbase : TCC);
  colop_task<NK>(P, img, cbase, ncv, t);
}

// column j's coordinate k (of [b | v]) changed to v: its B1 and R entries
template <int NK>
GMF_D void colimg_write(const Params& P, int64_t j, int k, float v) {
  constexpr int nka = NK <= 16 ? 16 : 32;
  constexpr uint32_t sbo1 = (uint32_t)(nka / 8) * 128u;
  constexpr int64_t b1sz = (int64_t)TCC * nka * 2;
  const int ct = (int)(j / TCC), c = (int)(j % TCC);
  unsigned char* img = reinterpret_cast<unsigned char*>(P.colimg) + (int64_t)ct * colimg_bytes(NK);
  unsigned char* B1 = img + 64 * TCC * 2;
  __nv_bfloat16 a, b, e;
  split3_1(v * kLog2e, a, b, e);
  *reinterpret_cast<__nv_bfloat16*>(B1 + kofs(c, k, sbo1)) = a;
  *reinterpret_cast<__nv_bfloat16*>(B1 + b1sz + kofs(c, k, sbo1)) = b;
  *reinterpret_cast<__nv_bfloat16*>(B1 + 2 * b1sz + kofs(c, k, sbo1)) = e;
  if (k >= P.p) {
    const int kr = P.q + (k - P.p);
    __nv_bfloat16 h, l, h2, l2;
    tc::split_bf16(v, h, l);
    tc::split_bf16(v * v, h2, l2);
    *reinterpret_cast<__nv_bfloat16*>(img + kofs(kr, c, SBO_P)) = h;
    *reinterpret_cast<__nv_bfloat16*>(img + kofs(16 + kr, c, SBO_P)) = l;
    *reinterpret_cast<__nv_bfloat16*>(img + kofs(32 + kr, c, SBO_P)) = h2;
    *reinterpret_cast<__nv_bfloat16*>(img + kofs(48 + kr, c, SBO_P)) = l2;
  }
}

// ---------------------------------------------------------------------------
// barriers and per-CTA state
// ---------------------------------------------------------------------------
struct Bars {
  uint64_t eta_full[2], eta_free[2];
  uint64_t staged[3];       // tile-CSR staging slot landed (TMA bulk copies, byte count)
  uint64_t cimg;            // column-operand image landed (unit prologue)
  uint64_t a1_full[2], a3_full[2];   // operand rows of a chunk landed (byte count)
  uint64_t a1_free[2], a3_free[2];   // GEMM1 / GEMM3 done with an operand slot
  uint64_t p_full, p_free, y_full[2], y_free[2];
};

GMF_D void mbar_init_n(uint64_t* bar, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(n) : "memory");
}
GMF_D void mbar_arrive(uint64_t* bar) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.release.cta.shared::cta.b64 st, [%0];\n\t}" ::"r"(
                   smem_addr(bar))
               : "memory");
}

// mbarrier phase wait with a hang guard: a protocol error traps (the launch
// fails with an error) instead of spinning forever.  No global state is read
// here: a __device__ switch consulted per wait costs the single-thread roles
// (MMA issuer, loader) a dependent global load each time.
GMF_D void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  unsigned long long t0 = 0;
  for (;;) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(done)
        : "r"(smem_addr(bar)), "r"(parity)
        : "memory");
    if (done) break;
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    if (t0 == 0) t0 = t;
    else if (t - t0 > 4000000000ull) __trap();   // 4 s
  }
}

struct Ctx {
  uint32_t tmem;
  Bars* b;
  uint32_t gc;   // chunks this CTA has pipelined since launch (mbarrier phases)
  uint32_t nu;   // units this CTA has started since launch (image barrier phase)
};

GMF_D void ctx_open(Ctx& X, uint32_t* s_tmem, Bars* s_b) {
  const int warp = threadIdx.x >> 5;
  if (warp == MMA_WARP) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_addr(s_tmem)),
                 "n"(kCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init_n(&s_b->eta_full[i], 1);
      mbar_init_n(&s_b->eta_free[i], NEW);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init_n(&s_b->a1_full[i], 1);
      mbar_init_n(&s_b->a3_full[i], 1);
      mbar_init_n(&s_b->a1_free[i], 1);
      mbar_init_n(&s_b->a3_free[i], 1);
    }
    mbar_init_n(&s_b->p_full, NEW);
    mbar_init_n(&s_b->p_free, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init_n(&s_b->y_full[i], 1);
      mbar_init_n(&s_b->y_free[i], NEW);
    }
    for (int i = 0; i < 3; ++i) mbar_init_n(&s_b->staged[i], 1);
    mbar_init_n(&s_b->cimg, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  fence_before();
  __syncthreads();
  fence_after();
  X.tmem = *s_tmem;
  X.b = s_b;
  X.gc = 0;
  X.nu = 0;
}

GMF_D void ctx_close(const Ctx& X) {
  fence_before();
  __syncthreads();
  fence_after();
  if ((threadIdx.x >> 5) == MMA_WARP)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(X.tmem), "n"(kCols)
                 : "memory");
}

// 32 lanes x 32 consecutive TMEM columns -> 32 registers per thread; the wait
// carries the registers so no use is scheduled before the data lands
GMF_D void tmem_ld32(uint32_t addr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
        "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
        "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(addr)
      : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]),
                 "+r"(v[6]), "+r"(v[7]), "+r"(v[8]), "+r"(v[9]), "+r"(v[10]), "+r"(v[11]),
                 "+r"(v[12]), "+r"(v[13]), "+r"(v[14]), "+r"(v[15]), "+r"(v[16]), "+r"(v[17]),
                 "+r"(v[18]), "+r"(v[19]), "+r"(v[20]), "+r"(v[21]), "+r"(v[22]), "+r"(v[23]),
                 "+r"(v[24]), "+r"(v[25]), "+r"(v[26]), "+r"(v[27]), "+r"(v[28]), "+r"(v[29]),
                 "+r"(v[30]), "+r"(v[31])
               :
               : "memory");
}


GMF_D void prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// TMA bulk copy global -> shared (16-byte aligned, size a multiple of 16),
// completion counted in bytes on an mbarrier
GMF_D void bulk_g2s(void* sdst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(sdst)),
      "l"(gsrc), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}
GMF_D void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(
                   smem_addr(bar)),
               "r"(bytes)
               : "memory");
}
// 16-byte aligned superset [lo, hi) (elements of 4 bytes) of [b, e)
GMF_D int64_t lo4(int64_t b) { return b & ~int64_t(3); }
GMF_D int64_t hi4(int64_t e) { return (e + 3) & ~int64_t(3); }
// 16 fp32 values -> bf16 hi (8 words) and lo = bf16(x - hi) (8 words), both
// rounded to nearest (ties away) with integer ops: the elementwise pass is
// bound by the quarter-rate pipe (ex2, rcp), so the split stays off it
GMF_D uint32_t rn_hi(float x) { return (__float_as_uint(x) + 0x8000u) & 0xffff0000u; }
GMF_D uint32_t pack_hi(uint32_t a, uint32_t b) {   // upper halves of a, b -> (b:a)
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, 0x7632;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}
GMF_D void split16_alu(const float* x, uint32_t* hi, uint32_t* lo) {
  #pragma unroll
  for (int u = 0; u < 8; ++u) {
    const float a = x[2 * u], b = x[2 * u + 1];
    const uint32_t ha = rn_hi(a), hb = rn_hi(b);
    const float ra = a - __uint_as_float(ha), rb = b - __uint_as_float(hb);
    hi[u] = pack_hi(ha, hb);
    lo[u] = pack_hi(__float_as_uint(ra) + 0x8000u, __float_as_uint(rb) + 0x8000u);
  }
}

// 16 fp32 values -> bf16 hi (8 words) and lo = bf16(x - hi) (8 words)
GMF_D void split16(const float* x, uint32_t* hi, uint32_t* lo) {
  #pragma unroll
  for (int u = 0; u < 8; ++u) {
    const float a = x[2 * u], b = x[2 * u + 1];
    uint32_t h, l;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(h) : "f"(b), "f"(a));
    const float ra = a - __uint_as_float(h << 16);
    const float rb = b - __uint_as_float(h & 0xffff0000u);
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(l) : "f"(rb), "f"(ra));
    hi[u] = h;
    lo[u] = l;
  }
}

GMF_D void store16(unsigned char* Pb, int m, int c0, const uint32_t* w) {
  *reinterpret_cast<uint4*>(Pb + kofs(m, c0, SBO_P)) = make_uint4(w[0], w[1], w[2], w[3]);
  *reinterpret_cast<uint4*>(Pb + kofs(m, c0 + 8, SBO_P)) = make_uint4(w[4], w[5], w[6], w[7]);
}

// ---------------------------------------------------------------------------
// Operand-row images (pre-pass).  A1 (GEMM1: a = [x | u | gamma | offset |
// sentinels], three bf16 splits) and A3 / A3sq (GEMM3: features 0..15 of a,
// the column side's [x | u], and their squares, hi | lo) depend on the rows
// only, so every step builds them ONCE per 64-row chunk of every row split
// (in the byte layout of the shared-memory tiles) instead of once per column
// tile; the loaders copy them with TMA.  Chunk (rs, c) of a step is ready
// when rimg_flag[rs * rimg_nch + c] reaches the step's epoch.
// ---------------------------------------------------------------------------
GMF_D void row_feats8(const Params& P, int64_t i, bool rok, int gk, float (&v)[8]) {
  const int p = P.p, q = P.q, d = P.d, KA = P.KA, Kr = P.Kr;
  const int kone = kone_of(P);
  const float* th = tptr<float>(P.th_row) + (rok ? i : 0) * Kr;
  const float* xr = tptr<float>(P.x) + (rok ? i : 0) * p;
  const float ov = P.has_off ? tptr<float>(P.off)[rok ? i : 0] : 0.f;
  #pragma unroll
  for (int e = 0; e < 8; ++e) {
    const int k = 8 * gk + e;
    // a_k: x_k (k < p), u (p <= k < p+d), gamma, offset at KA, the two
    // sentinel features, then zeros
    const int it = k < p + d ? q + (k - p) : k - p - d;
    float x = 0.f;
    if (k < p) x = xr[k];
    else if (k < KA) x = th[it];
    else if (k == KA && P.has_off) x = ov;
    if (!rok) x = 0.f;
    if (k == kone) x = 1.f;
    if (k == kone + 1) x = rok ? 0.f : kSentinel;
    v[e] = x;
  }
}

// one image task: row r of the chunk (block rows i0 + r, valid when r < rows),
// feature group gk (A1) and, for gk < 2, the A3 pieces
template <int NKA>
GMF_D void image_task(const Params& P, unsigned char* img, int64_t i0, int rows, int t) {
  constexpr int ng1 = NKA / 8;
  constexpr uint32_t sbo1 = (uint32_t)ng1 * 128u, a1h = (uint32_t)CR * NKA * 2;
  const int r = t / ng1, gk = t % ng1;
  float v[8];
  row_feats8(P, i0 + r, r < rows, gk, v);
  uint4 s0, s1, s2;
  split3_8(v, s0, s1, s2);
  *reinterpret_cast<uint4*>(img + kofs(r, 8 * gk, sbo1)) = s0;
  *reinterpret_cast<uint4*>(img + a1h + kofs(r, 8 * gk, sbo1)) = s1;
  *reinterpret_cast<uint4*>(img + 2 * a1h + kofs(r, 8 * gk, sbo1)) = s2;
  if (gk < 2) {
    unsigned char* A3b = img + 3 * a1h;
    float v2[8];
    #pragma unroll
    for (int e = 0; e < 8; ++e) v2[e] = v[e] * v[e];
    uint4 h, l;
    tc::split8(v, h, l);
    *reinterpret_cast<uint4*>(A3b + a1ofs(r, 8 * gk, 0, 512u)) = h;
    *reinterpret_cast<uint4*>(A3b + a1ofs(r, 8 * gk, 1, 512u)) = l;
    tc::split8(v2, h, l);
    *reinterpret_cast<uint4*>(A3b + 4096 + a1ofs(r, 8 * gk, 0, 512u)) = h;
    *reinterpret_cast<uint4*>(A3b + 4096 + a1ofs(r, 8 * gk, 1, 512u)) = l;
  }
}

GMF_D void st_release_u32(unsigned int* p, unsigned int v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
GMF_D unsigned int ld_acquire_u32g(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// all CTAs: the images of every chunk of row block blk (RS row splits), chunk
// q = rs * rimg_nch + c built by CTA q mod G; its flag is then set to epoch
template <int NK>
GMF_D void build_images(const Params& P, long long blk, int RS, unsigned int epoch) {
  constexpr int nka = NK <= 16 ? 16 : 32, ng1 = nka / 8;
  const int64_t r0 = P.rbp[blk], nI = P.rbp[blk + 1] - r0;
  const int64_t nq = (int64_t)RS * P.rimg_nch;
  const int64_t ib = rimg_bytes(NK);
  for (int64_t qq = blockIdx.x; qq < nq; qq += gridDim.x) {
    const int rs = (int)(qq / P.rimg_nch), c = (int)(qq % P.rimg_nch);
    const int64_t rlo = nI * rs / RS, rhi = nI * (rs + 1) / RS;
    const int64_t left = rhi - rlo - (int64_t)c * CR;
    if (left <= 0) continue;   // uniform across the CTA
    const int rows = (int)(left < CR ? left : CR);
    unsigned char* img = reinterpret_cast<unsigned char*>(P.rimg) + qq * ib;
    for (int t = threadIdx.x; t < CR * ng1; t += blockDim.x)
      image_task<nka>(P, img, r0 + rlo + (int64_t)c * CR, rows, t);
    __syncthreads();
    if (threadIdx.x == 0) {
      asm volatile("fence.proxy.async.global;" ::: "memory");   // read by TMA (async proxy)
      st_release_u32(P.rimg_flag + qq, epoch);
    }
  }
}

// ---------------------------------------------------------------------------
// K1 v2 body: every unit of this CTA.  Called by all NT threads, after
// build_images of the same step (epoch).
// ---------------------------------------------------------------------------
template <int FAM, int NK>
GMF_D void grad_units(const Params& P, long long blk, long long s, double alpha, int RS,
                      unsigned char* smem, Ctx& X, unsigned int epoch,
                      unsigned long long* kp = nullptr) {
  // optional sub-phase clocks (accumulated per CTA, 16 slots): elementwise
  // warp 0 lane 0: 0 unit prologue, 1 wait eta, 3 wait Y, 4 elementwise,
  // 5 wait P free, 6 D2 readout + P store, 7 unit drain; MMA thread: 8 wait
  // A1, 9 wait eta free, 10 issue, 11 wait P full / A3; loader lane 0:
  // 12 staging issue (incl. image-ready waits), 13 wait staged, 14 wait Y
  // free, 15 scatter
  long long kacc[16];
  #pragma unroll
  for (int i = 0; i < 16; ++i) kacc[i] = 0;
  const bool kt_ew = kp && threadIdx.x == 0;
  const bool kt_mm = kp && threadIdx.x == MMA_WARP * 32;
  const bool kt_ld = kp && threadIdx.x == LDW * 32;
  long long tk = (kt_ew || kt_ld || kt_mm) ? clock64() : 0;
  auto tick = [&](bool on, int i) {
    if (on) {
      const long long t = clock64();
      kacc[i] += t - tk;
      tk = t;
    }
  };
  // event timeline of CTA 0 (globaltimer, the last step overwrites): ev * 32 + chunk
  unsigned long long* tl = (kp && blockIdx.x == 0) ? kp - 8 + 32 * (int64_t)gridDim.x : nullptr;
  auto mark = [&](int ev, int c) {
    if (tl && c < 32) tl[ev * 32 + c] = gtimer();
  };
  __shared__ double red_scr[NT / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int Kr = P.Kr, Kc = P.Kc, p = P.p;
  const int csr = P.yfmt == GMF_Y_DENSE_I32 ? 0 : (P.yfmt == GMF_Y_CSR_PACK32 ? 2 : 1);
  const Lay L = layout(NK, Kr, p, csr, P.k1_cap, P.k1_na1);
  constexpr int nka = NK <= 16 ? 16 : 32, ng1 = nka / 8;
  constexpr uint32_t sbo1 = (uint32_t)ng1 * 128u;        // B1 / A1 splits (K-major)
  constexpr uint32_t b1sz = (uint32_t)TCC * nka * 2;
  constexpr uint32_t a1sz = (uint32_t)128 * nka * 2;
  const uint32_t sb = smem_addr(smem);
  Bars& B = *X.b;
  const int64_t r0 = P.rbp[blk], nI = P.rbp[blk + 1] - r0;
  const int64_t j0 = P.cbp[s], nJ = P.cbp[s + 1] - j0;
  const int CT = P.CT;
  const int64_t U = (int64_t)CT * RS;
  float* colpart = tptr<float>(P.colpart);
  float* rowpart = tptr<float>(P.rowpart);
  double nb_num = 0.0, nb_den = 0.0;
  // CSR through the tile-major copy (entries carry their row) when it exists
  const bool tcsr = csr && P.tent != nullptr && !P.stream_mode;
  const int64_t ib = rimg_bytes(NK);
  auto rows_of = [&](int64_t nrows, int c) {
    const int64_t left = nrows - (int64_t)c * CR;
    return (int)(left < CR ? left : CR);
  };

  for (int64_t u = blockIdx.x; u < U; u += gridDim.x) {
    const int ct = (int)(u / RS), rs = (int)(u % RS);
    const int64_t rlo = nI * rs / RS, rhi = nI * (rs + 1) / RS;
    const int64_t nrows = rhi - rlo;
    const int64_t cbase = (int64_t)ct * TCC;
    const int64_t ncv64 = nJ - cbase;
    const int ncv = ncv64 < 0 ? 0 : (ncv64 > TCC ? TCC : (int)ncv64);
    const int64_t cpb = ((int64_t)ct * RS + rs) * TCC * (2 * Kc);
    if (nrows <= 0) {   // nothing to do: zero the unit's column partials
      for (int e = tid; e < TCC * 2 * Kc; e += NT) colpart[cpb + e] = 0.f;
      continue;
    }
    const int nch = (int)((nrows + CR - 1) / CR);
    const uint32_t gc0 = X.gc;

    // ---- unit prologue: column operands R | B1 ----
    __syncthreads();   // the previous unit has fully drained (smem reuse)
    if (P.colimg_on) {   // one TMA bulk copy of the tile's image
      if (tid == 0) {
        const int64_t nb = colimg_bytes(NK);
        const unsigned char* img = reinterpret_cast<const unsigned char*>(P.colimg) + (int64_t)ct * nb;
        mbar_expect_tx(&B.cimg, (uint32_t)nb);
        bulk_g2s(smem + L.R, img, (uint32_t)nb, &B.cimg);
      }
    } else {
      const int32_t* cmap = P.col_identity ? nullptr : P.cidx + j0;
      for (int t = tid; t < colimg_tasks<NK>(); t += NT) colop_task<NK>(P, smem + L.R, cbase, ncv, t, cmap);
    }
    if (csr) for (int e = tid; e < 2 * CR * YP; e += NT) reinterpret_cast<float*>(smem + L.Y)[e] = 0.f;

    // loader (lane 0 issues): operand-row images and tile-CSR entries of a
    // chunk with TMA bulk copies
    // loader, once per unit: the tile-CSR chunk boundaries (lane l holds
    // boundaries l, l + 32, ...) and the readiness of every chunk image
    constexpr int KB = 4;   // boundary registers per lane: units of up to 127 chunks
    int64_t bnd[KB];
    bool bnd_ok = nch < 32 * KB;
    if (warp == LDW) {
      const int64_t* tp = tcsr ? P.tptr + (int64_t)ct * (P.n + 1) : nullptr;
      #pragma unroll
      for (int k = 0; k < KB; ++k) {
        const int c = lane + 32 * k;
        const int64_t row = rlo + (c < nch ? (int64_t)c * CR : nrows);
        bnd[k] = (tcsr && bnd_ok && c <= nch) ? tp[r0 + row] : 0;
      }
      const unsigned long long t0 = gtimer();
      for (;;) {   // every image of the unit built (by any CTA) this step
        bool ready = true;
        for (int c = lane; c < nch; c += 32)
          ready = ready && ld_acquire_u32g(P.rimg_flag + (int64_t)rs * P.rimg_nch + c) >= epoch;
        if (__all_sync(0xffffffffu, ready)) break;
        if (gtimer() - t0 > 4000000000ull) __trap();
      }
      asm volatile("fence.proxy.async.global;" ::: "memory");   // the TMA reads what was acquired
    }
    auto bnd_at = [&](int c) -> int64_t {   // whole warp
      int64_t v = 0;
      #pragma unroll
      for (int k = 0; k < KB; ++k) {
        const int64_t x = __shfl_sync(0xffffffffu, bnd[k], c & 31);
        if ((c >> 5) == k) v = x;
      }
      return v;
    };
    auto img_of = [&](int c) -> const unsigned char* {
      return reinterpret_cast<const unsigned char*>(P.rimg) + ((int64_t)rs * P.rimg_nch + c) * ib;
    };
    auto issue_a1 = [&](int c) {   // A1 of chunk c into slot gcc % na1 (both replicas)
      if (c >= nch || lane != 0) return;
      const uint32_t gcs = gc0 + (uint32_t)c;
      const uint32_t a1s = gcs % (uint32_t)L.na1;
      if (gcs >= (uint32_t)L.na1) mbar_wait(&B.a1_free[a1s], ((gcs / L.na1) - 1u) & 1u);
      mark(0, c);
      const unsigned char* img = img_of(c);
      uint64_t* bar = &B.a1_full[gcs & 1u];
      const uint32_t h = (uint32_t)CR * nka * 2;
      mbar_expect_tx(bar, 6u * h);
      unsigned char* dst = smem + L.A1 + a1s * 3u * a1sz;
      #pragma unroll
      for (int sp = 0; sp < 3; ++sp) {
        bulk_g2s(dst + sp * a1sz, img + sp * h, h, bar);
        bulk_g2s(dst + sp * a1sz + h, img + sp * h, h, bar);   // rows 64..127 = rows 0..63
      }
    };
    auto issue_a3 = [&](int c) {   // A3 / A3sq of chunk c into slot gcc & 1
      if (c >= nch || lane != 0) return;
      const uint32_t gcs = gc0 + (uint32_t)c;
      if (gcs >= 2) mbar_wait(&B.a3_free[gcs & 1u], ((gcs >> 1) - 1u) & 1u);
      const unsigned char* img = img_of(c);
      uint64_t* bar = &B.a3_full[gcs & 1u];
      mbar_expect_tx(bar, 8192u);
      bulk_g2s(smem + L.A3 + (gcs & 1u) * 8192u, img + 3 * CR * nka * 2, 8192u, bar);
    };
    auto issue_csr = [&](int c) {   // tile-CSR entries of chunk c into ring slot gcc % 3 (whole warp)
      if (!tcsr || c >= nch) return;
      int64_t e_lo, e_hi;
      if (bnd_ok) {
        e_lo = bnd_at(c);
        e_hi = bnd_at(c + 1);
      } else {
        const int64_t* tp = P.tptr + (int64_t)ct * (P.n + 1);
        const int64_t i0 = r0 + rlo + (int64_t)c * CR;
        e_lo = tp[i0];
        e_hi = tp[i0 + rows_of(nrows, c)];
      }
      if (lane != 0) return;
      const uint32_t gcs = gc0 + (uint32_t)c;
      const uint32_t sl = gcs % NSLOT;
      uint64_t* bar = &B.staged[sl];
      int32_t* meta = reinterpret_cast<int32_t*>(smem + L.nstage + (int64_t)sl * L.nslot_bytes);
      const int64_t ea = e_lo & ~int64_t(1), ee = (e_hi + 1) & ~int64_t(1);
      const bool fits = (ee - ea) <= L.cap;
      meta[0] = (int)(e_lo - ea);
      meta[1] = (int)(e_hi - e_lo);
      meta[2] = fits ? 1 : 0;
      *reinterpret_cast<int64_t*>(meta + 4) = e_lo;
      const uint32_t bytes = fits ? (uint32_t)((ee - ea) * 8) : 0u;
      mbar_expect_tx(bar, bytes);   // release: the metadata above
      if (bytes) bulk_g2s(meta + 8, P.tent + 2 * ea, bytes, bar);
      mark(1, c);
    };
    if (warp == LDW) {
      issue_a1(0);
      issue_csr(0);
      issue_a3(0);
      // with a single A1 buffer (shared memory short: CSR with 32-feature
      // operands) chunk 1's copy waits for GEMM1 of chunk 0, which the MMA
      // warp only issues after this prologue's barrier: it is issued in the
      // loader's role section below instead
      if (L.na1 >= 2) issue_a1(1);
      issue_csr(1);
    }
    if (P.colimg_on) mbar_wait(&B.cimg, X.nu & 1u);
    ++X.nu;
    fence_async_smem();
    __syncthreads();
    tick(kt_ew, 0);
    if (kt_ld || kt_mm) tk = clock64();
    if (tid == 0) mark(11, 0);

    if (warp < NEW) {
      // ====================== elementwise warps ======================
      const int qd = warp & 3, hf = warp >> 2, g = qd & 1;
      const int rr = 32 * g + lane;                   // chunk row of this thread
      const int cb = 64 * (qd >> 1) + 32 * hf;        // first tile column
      const uint32_t lane_base = (uint32_t)(32 * qd) << 16;
      const int vcols = ncv - cb < 0 ? 0 : (ncv - cb > 32 ? 32 : ncv - cb);
      const float rphi = (float)(1.0 / P.phi);
      const float tphi = (float)P.phi;
      const float tra = (float)(P.phi / alpha);
      unsigned char* Pg = smem + L.P + 32768 * g;
      const int mh = stack_hi(lane);
      int yv[32];
      const bool dvec = (P.m & 3) == 0 && P.col_identity;
      auto load_dense = [&](int c) {
        const int64_t rowc = rlo + (int64_t)c * CR + rr;
        const bool ok = rowc < rhi;   // rows past the unit read nothing (y = 0)
        const int64_t i = r0 + (ok ? rowc : rlo);
        if (dvec && vcols == 32) {
          const int4* src = reinterpret_cast<const int4*>(P.y + i * P.m + cbase + cb);
          #pragma unroll
          for (int v = 0; v < 8; ++v) {
            const int4 t4 = ok ? __ldcs(src + v) : make_int4(0, 0, 0, 0);
            yv[4 * v] = t4.x; yv[4 * v + 1] = t4.y; yv[4 * v + 2] = t4.z; yv[4 * v + 3] = t4.w;
          }
        } else {
          #pragma unroll
          for (int v = 0; v < 32; ++v) {
            const int64_t pos = cbase + cb + v;
            const bool okc = ok && v < vcols;
            const int64_t jj = okc ? (P.col_identity ? pos : (int64_t)P.cidx[j0 + pos]) : 0;
            yv[v] = okc ? P.y[i * P.m + jj] : 0;
          }
        }
      };
      if (!csr) load_dense(0);
      // D2 readout of chunk c (row partials): warp reads D2 of group hf
      auto readout_d2 = [&](int c) {
        const int rows_c = rows_of(nrows, c);
        uint32_t a[32];
        tmem_ld32(X.tmem + lane_base + T_D2 + 64u * hf + (qd >= 2 ? 32u : 0u), a);
        float dv[16];
        #pragma unroll
        for (int k = 0; k < 16; ++k) {
          dv[k] = __uint_as_float(a[k]) + __uint_as_float(a[16 + k]);
          dv[k] += __shfl_xor_sync(0xffffffffu, dv[k], 8);
        }
        const int r = 32 * hf + 16 * (qd & 1) + 8 * (lane >> 4) + (lane & 7);
        if (!(lane & 8) && r < rows_c) {
          float* outp = rowpart + ((int64_t)ct * P.nstar_max + rlo + (int64_t)c * CR + r) * (2 * Kr) +
                        (qd < 2 ? 0 : Kr);
          #pragma unroll
          for (int k = 0; k < 16; ++k)
            if (k < Kr) outp[k] = dv[k];
        }
      };
      for (int c = 0; c < nch; ++c) {
        const uint32_t gcc = gc0 + (uint32_t)c;
        const int slot = (int)(gcc & 1u);
        // ---- eta and counts of this chunk ----
        mbar_wait(&B.eta_full[slot], (gcc >> 1) & 1u);
        fence_after();
        tick(kt_ew, 1);
        if (tid == 0) mark(6, c);
        float4* yrow;
        if (csr) {
          mbar_wait(&B.y_full[slot], (gcc >> 1) & 1u);
          yrow = reinterpret_cast<float4*>(reinterpret_cast<float*>(smem + L.Y) + (slot * CR + rr) * YP + cb);
        } else {   // dense: this thread's counts through its private stretch of the Y scratch
          yrow = reinterpret_cast<float4*>(reinterpret_cast<float*>(smem + L.Y) + rr * YP + cb);
          #pragma unroll
          for (int v = 0; v < 8; ++v)
            yrow[v] = make_float4((float)yv[4 * v], (float)yv[4 * v + 1], (float)yv[4 * v + 2],
                                  (float)yv[4 * v + 3]);
          if (c + 1 < nch) load_dense(c + 1);   // next chunk's counts in flight
        }
        tick(kt_ew, 3);
        // ---- dotD / ddotD, 16 entries at a time (a compact loop body keeps the
        // instruction cache warm for the other roles) ----
        float cn = 0.f, cdn = 0.f;
        #pragma unroll 1
        for (int half = 0; half < 2; ++half) {
          uint32_t ev[16];
          tc::tmem_ld16(X.tmem + lane_base + (uint32_t)(128 * slot) + (uint32_t)(cb + 16 * half), ev);
          float yf[16];
          #pragma unroll
          for (int v = 0; v < 4; ++v) {
            const float4 t4 = yrow[4 * half + v];
            yf[4 * v] = t4.x; yf[4 * v + 1] = t4.y; yf[4 * v + 2] = t4.z; yf[4 * v + 3] = t4.w;
          }
          if (csr) {
            const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
            #pragma unroll
            for (int v = 0; v < 4; ++v) yrow[4 * half + v] = z4;
          }
          float dd[16], hh[16];
          #pragma unroll
          for (int i = 0; i < 16; ++i) {
            // entries outside the block have eta = -1000 (sentinel features)
            // and y = 0: mu, dotD, ddotD and the moment terms vanish
            const float mu = exp_pre(__uint_as_float(ev[i]));
            const float r = yf[i] - mu;
            if (FAM == 0) {
              dd[i] = -rphi * r;
              hh[i] = rphi * mu;
            } else {
              const float rc = rcp_fast(fmaf(mu, tra, tphi));
              dd[i] = -r * rc;
              hh[i] = mu * rc;
              cn = fmaf(mu, mu, cn);
              cdn += fmaf(r, r, -mu);
            }
          }
          uint32_t dh[8], dl[8], hh_[8], hl[8];
          split16_alu(dd, dh, dl);
          split16_alu(hh, hh_, hl);
          if (half == 0) {
            tick(kt_ew, 4);
            if (tid == 0) mark(7, c);
            // P is free once GEMM2/3 of the previous chunk completed; that
            // chunk's row side is then in D2
            if (gcc > 0) {
              mbar_wait(&B.p_free, (gcc - 1u) & 1u);
              fence_after();
            }
            tick(kt_ew, 5);
            if (tid == 0) mark(8, c);
            if (c > 0) readout_d2(c - 1);
          }
          const int c0 = cb + 16 * half;
          store16(Pg, mh, c0, dh);
          store16(Pg, mh + 8, c0, dl);
          store16(Pg, 64 + mh, c0, hh_);
          store16(Pg, 64 + mh + 8, c0, hl);
        }
        nb_num += (double)cn;
        nb_den += (double)cdn;
        fence_before();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&B.eta_free[slot]);
          if (csr) mbar_arrive(&B.y_free[slot]);
        }
        fence_async_smem();
        fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&B.p_full);
        tick(kt_ew, 6);
        if (tid == 0) mark(9, c);
      }
      // ---- unit drain: last chunk's row side, then the column side ----
      const uint32_t gl = gc0 + (uint32_t)nch - 1u;
      mbar_wait(&B.p_free, gl & 1u);
      fence_after();
      readout_d2(nch - 1);
      {
        // lane = tile column; D3 columns = a-features [x | u | gamma], whose
        // first Kc are the column side's [x | u]
        uint32_t a[32];
        tmem_ld32(X.tmem + lane_base + T_D3 + (hf ? 32u : 0u), a);
        const int c = 32 * qd + lane;
        float* outp = colpart + cpb + (int64_t)c * (2 * Kc) + (hf ? Kc : 0);
        #pragma unroll
        for (int f = 0; f < 16; ++f)
          if (f < Kc) outp[f] = __uint_as_float(a[f]) + __uint_as_float(a[16 + f]);
      }
      fence_before();
      tick(kt_ew, 7);
      if (tid == 0) mark(12, 0);
    } else if (warp == MMA_WARP) {
      // ====================== MMA issuer ======================
      if (lane == 0) {
        const uint32_t tm = X.tmem;
        constexpr uint32_t ID1 = idesc(128, 128, 0, 0);
        constexpr uint32_t ID2 = idesc(128, 64, 0, 0);
        constexpr uint32_t ID3 = idesc(128, 32, 1, 1);
        // A single thread issues every MMA, so its instruction stream is a
        // dependent chain: the shared-memory descriptors are unit invariants
        // (base + a small start-address increment per K step; the 14-bit
        // address field never carries), built once here, and umma_nc carries
        // no memory clobber (volatile asm keeps the MMA / commit / wait order),
        // so the increments are hoisted and overlapped instead of re-derived
        // between issues.
        const uint64_t dR = sdesc(sb + (uint32_t)L.R, 128, SBO_P);
        const uint64_t dB1_0 = sdesc(sb + (uint32_t)L.B1, 128, sbo1);
        const uint64_t dB1_1 = sdesc(sb + (uint32_t)L.B1 + b1sz, 128, sbo1);
        const uint64_t dB1_2 = sdesc(sb + (uint32_t)L.B1 + 2 * b1sz, 128, sbo1);
        const uint64_t dA1 = sdesc(sb + (uint32_t)L.A1, 128, sbo1);   // slot 0, split 0
        const uint64_t dP2_0 = sdesc(sb + (uint32_t)L.P, 128, SBO_P);           // GEMM2, group 0
        const uint64_t dP3_0 = sdesc(sb + (uint32_t)L.P, 2048, 128);            // GEMM3 dd, group 0
        const uint64_t dA3 = sdesc(sb + (uint32_t)L.A3, 0, 128);                // A3 slot 0
        auto adv = [](uint64_t d, uint32_t bytes) { return d + (uint64_t)(bytes >> 4); };
        auto umma_nc = [](uint32_t d, uint64_t a, uint64_t bb, uint32_t id, uint32_t acc) {
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
              "l"(a), "l"(bb), "r"(id), "r"(acc));
        };
        // GEMM1 runs one chunk ahead of the elementwise warps' demand: in the
        // in-order tensor pipe GEMM1(c+1) precedes GEMM2/3(c-1)
        auto gemm1 = [&](int c) {
          if (c >= nch) return;
          const uint32_t gcc = gc0 + (uint32_t)c;
          const int slot = (int)(gcc & 1u);
          mbar_wait(&B.a1_full[slot], (gcc >> 1) & 1u);
          tick(kt_mm, 8);
          if (gcc >= 2) mbar_wait(&B.eta_free[slot], ((gcc >> 1) - 1u) & 1u);
          tick(kt_mm, 9);
          mark(4, c);
          fence_after();
          const uint32_t d = tm + (uint32_t)(128 * slot);
          const uint32_t a1s = gcc % (uint32_t)L.na1;
          const uint64_t a0b = adv(dA1, a1s * 3u * a1sz);
          #pragma unroll
          for (int kt = 0; kt < nka / 16; ++kt) {
            const uint32_t kb = (uint32_t)kt * 256u;
            const uint64_t a0 = adv(a0b, kb), a1 = adv(a0b, a1sz + kb), a2 = adv(a0b, 2 * a1sz + kb);
            const uint64_t b0 = adv(dB1_0, kb), b1 = adv(dB1_1, kb), b2 = adv(dB1_2, kb);
            umma_nc(d, a0, b0, ID1, kt > 0 ? 1u : 0u);
            umma_nc(d, a0, b1, ID1, 1u);
            umma_nc(d, a1, b0, ID1, 1u);
            umma_nc(d, a0, b2, ID1, 1u);
            umma_nc(d, a1, b1, ID1, 1u);
            umma_nc(d, a2, b0, ID1, 1u);
          }
          umma_commit(&B.eta_full[slot]);
          umma_commit(&B.a1_free[a1s]);
          tick(kt_mm, 10);
          mark(15, c);
        };
        gemm1(0);
        for (int c = 0; c < nch; ++c) {
          gemm1(c + 1);
          {
            const uint32_t gp = gc0 + (uint32_t)c;
            const uint64_t a3 = adv(dA3, (gp & 1u) * 8192u);
            mbar_wait(&B.p_full, gp & 1u);
            mbar_wait(&B.a3_full[gp & 1u], (gp >> 1) & 1u);
            tick(kt_mm, 11);
            mark(5, c);
            fence_after();
            #pragma unroll
            for (int gg = 0; gg < 2; ++gg) {
              const uint64_t p2 = adv(dP2_0, 32768u * gg), p3 = adv(dP3_0, 32768u * gg);
              #pragma unroll
              for (int kt = 0; kt < TCC / 16; ++kt)
                umma_nc(tm + T_D2 + 64u * gg, adv(p2, 256u * kt), adv(dR, 256u * kt), ID2,
                        kt > 0 ? 1u : 0u);
              // D3[col][f] += P^T . [a_hi | a_lo] (dd) and P^T . [a2_hi | a2_lo] (hh);
              // K-step u = stacked rows 16u..16u+15 = group rows 8u..8u+7 hi then
              // lo, paired with feature rows 8u..8u+7 twice (LBO 0)
              #pragma unroll
              for (int uu = 0; uu < 4; ++uu) {
                const uint32_t acc0 = (c == 0 && gg == 0 && uu == 0) ? 0u : 1u;
                const uint32_t rg = 512u * (uint32_t)(4 * gg + uu);
                umma_nc(tm + T_D3, adv(p3, 4096u * uu), adv(a3, rg), ID3, acc0);
                umma_nc(tm + T_D3 + 32, adv(p3, 16384u + 4096u * uu), adv(a3, 4096u + rg), ID3, acc0);
              }
            }
            umma_commit(&B.p_free);
            umma_commit(&B.a3_free[gp & 1u]);
            tick(kt_mm, 10);
          }
        }
      }
      __syncwarp();
    } else if (warp == LDW) {
      // ====================== loader ======================
      // scatters chunk c+1's tile nonzeros into its Y tile (lane-parallel:
      // every tile-CSR entry carries its row) while the elementwise warps work
      // on chunk c, and stages A1 and entries of c+2 and A3 of c+1 (whose
      // slot frees when GEMM3 of c-1 completes)
      if (kt_ld) tk = clock64();
      auto scatter = [&](int c) {
        if (c >= nch) return;
        const uint32_t gcc = gc0 + (uint32_t)c;
        const uint32_t sl = gcc % NSLOT, ys = gcc & 1u;
        if (tcsr) mbar_wait(&B.staged[sl], (gcc / NSLOT) & 1u);
        tick(kt_ld, 13);
        if (gcc >= 2) mbar_wait(&B.y_free[ys], ((gcc >> 1) - 1u) & 1u);
        tick(kt_ld, 14);
        if (lane == 0) mark(2, c);
        float* Y = reinterpret_cast<float*>(smem + L.Y) + ys * CR * YP;
        const int64_t i0 = r0 + rlo + (int64_t)c * CR;
        const int rows = rows_of(nrows, c);
        if (tcsr) {
          const int32_t* meta = reinterpret_cast<const int32_t*>(smem + L.nstage + (int64_t)sl * L.nslot_bytes);
          const int n_e = meta[1];
          if (meta[2]) {
            const int2* ent = reinterpret_cast<const int2*>(meta + 8) + meta[0];
            #pragma unroll 4
            for (int e = lane; e < n_e; e += 32) {
              const int2 w = ent[e];
              Y[(int)(w.x - i0) * YP + (w.y & 255)] = (float)(w.y >> 8);
            }
          } else {   // more nonzeros than a staging slot holds: straight from memory
            const int64_t elo = *reinterpret_cast<const int64_t*>(meta + 4);
            #pragma unroll 4
            for (int e = lane; e < n_e; e += 32) {
              const int2 w = reinterpret_cast<const int2*>(P.tent)[elo + e];
              Y[(int)(w.x - i0) * YP + (w.y & 255)] = (float)(w.y >> 8);
            }
          }
        } else {   // no tile-CSR (streamed blocks, general J): each lane walks rows
          for (int r = lane; r < rows; r += 32) {
            const int64_t i = i0 + r;
            for (int64_t k = P.rp[i]; k < P.rp[i + 1]; ++k) {
              const int col = csr_col_at(P, k);
              const int64_t pp = P.col_identity ? col : ((P.cbof[col] == s) ? (int64_t)P.cpos[col] : -1);
              const int64_t cl = pp - cbase;
              if (pp >= 0 && cl >= 0 && cl < TCC) Y[r * YP + cl] = (float)csr_val_at(P, k);
            }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&B.y_full[ys]);
        tick(kt_ld, 15);
      };
      if (L.na1 < 2) issue_a1(1);
      if (csr) scatter(0);
      for (int c = 0; c < nch; ++c) {
        issue_a1(c + 2);
        issue_csr(c + 2);
        tick(kt_ld, 12);
        if (csr) {
          scatter(c + 1);
        } else if (nka == 32 && c + 2 < nch && (P.m & 3) == 0 && P.col_identity && ncv > 0) {
          // dense: the chunk after next into L2 (one bulk prefetch per row).
          // Only with the 32-feature operands, whose longer GEMM1 leaves this
          // warp slack: with 16 features the prefetches took half the loader's
          // time and delayed the operand copies that gate GEMM1 (deep dense
          // cell K1 1.17 -> 0.92 ms without them), and the elementwise warps
          // already load the counts a whole chunk ahead
          const int rows2 = rows_of(nrows, c + 2);
          for (int r = lane; r < rows2; r += 32) {
            const int64_t i = r0 + rlo + (int64_t)(c + 2) * CR + r;
            prefetch_l2(P.y + i * P.m + cbase, (uint32_t)(ncv * 4));
          }
        }
        issue_a3(c + 1);
        tick(kt_ld, 12);
        __syncwarp();
      }
    }
    X.gc = gc0 + (uint32_t)nch;
  }
  if (kt_ew || kt_mm || kt_ld)
    for (int i = 0; i < 16; ++i)
      if (kacc[i]) atomicAdd(kp + i, (unsigned long long)kacc[i]);
  // per-CTA NB moment sums (fixed order: threads, then warps)
  __syncthreads();
  const double bn = block_sum<NT>(nb_num, red_scr);
  const double bd = block_sum<NT>(nb_den, red_scr);
  if (tid == 0) {
    P.nbpart[2 * blockIdx.x] = bn;
    P.nbpart[2 * blockIdx.x + 1] = bd;
  }
}

}  // namespace tc2
}  // namespace gmf
