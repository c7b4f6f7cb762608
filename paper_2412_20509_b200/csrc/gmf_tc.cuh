// K1 on the 5th-generation tensor cores (fp32 path): tcgen05.mma with
// operands in shared memory, accumulators in TMEM.
//
// Same contract as grad_cta (gmf_kern.cuh): one CTA owns column tile `ct`
// (128 columns of block J) and a balanced contiguous row range of block I,
// and writes rowpart / colpart / nbpart identically.  Per 32-row chunk:
//
//   GEMM1  eta[128 x 128]  = A1 . B1^T        rows x columns, K = p+q+d
//          (A1 = a_i = [x|u|gamma] of the 32 rows, replicated into the four
//          TMEM lane quarters so all 8 warps read eta; B1 = [b|v|z] * log2 e)
//   elementwise (CUDA cores, thread = row, 16 columns):
//          mu = 2^eta, dotD / ddotD (NB or Poisson, log link), NB moments,
//          written as the stacked bf16 tile P (dd rows, then hh rows; hi and
//          lo split rows interleaved by 8, see stack_hi)
//   GEMM2  D2[128 x 64]    = P . R           row side, K = tile columns
//          (R = [Rd_hi | Rd_lo | Rd2_hi | Rd2_lo], Rd = [z_j | v_j])
//   GEMM3  D3[128 x 64]   += P^T . [A1 | A1^2]   column side, K = chunk rows
//          (P and the chunk's A1 rows both read MN-major; [x|u] = first Kc of a)
//
// fp32 accuracy from bf16 operands: every operand is split x = hi + lo
// (hi = bf16(x), lo = bf16(x - hi)); the column side of GEMM1 also carries a
// third split x3 = bf16(x - hi - lo), so GEMM1 sums hi.hi + hi.lo + lo.hi +
// hi.x3 (the intercept and offset features are exact in bf16, so large
// intercepts b_j enter eta to ~2^-24); GEMM2/3 sum all four products,
// accumulation in fp32 (TMEM).
// Shared-memory operands use the canonical no-swizzle core-matrix layout
// (8 rows x 16 bytes): K-major tiles for GEMM1/GEMM2 and the same P and A1
// tiles read MN-major by GEMM3 (verified layouts: tools/umma_test.cu).
// TMEM: 256 columns per CTA (two CTAs per SM): eta [0,128), D2 [128,192),
// D3 [192,256).  One thread issues the MMAs (19 per chunk: tiny MMAs cost
// ~47 cycles each on the tensor pipe, tools/umma_bench.cu); completion is
// tracked with tcgen05.commit -> mbarrier.
#pragma once
#include <cuda_bf16.h>

#include <type_traits>

#include "gmf_kern.cuh"

namespace gmf {
namespace tc {

static_assert(kThreads == 256, "tensor-core K1 assumes 8 warps: 4 TMEM lane quarters x 2 column halves");
constexpr int TCC = 128;              // tile columns (GEMM1 N, GEMM3 M)
constexpr int TRC = 32;               // rows per chunk (x4 replicas = UMMA M 128)
constexpr int YP = 132;               // Y tile pitch (int32): conflict-free 16-byte row reads
constexpr uint32_t kCols = 256;       // TMEM columns per CTA
constexpr uint32_t T_ETA = 0, T_D2 = 128, T_D3 = 192;
constexpr uint32_t SBO_P = 2048;      // P / R: 16 column cores x 128 B

struct Smem {
  int64_t P, R, B1h, B1l, B1x, A1, As, Y, stage, araw, off, rp, total;
  int nka;
};

GMF_HD Smem smem_layout(int NK) {
  Smem s;
  int64_t o = 0;
  auto al = [](int64_t v) { return (v + 127) & ~int64_t(127); };
  s.nka = NK <= 16 ? 16 : 32;
  s.P = o; o = al(o + 128 * TCC * 2);
  s.R = o; o = al(o + 64 * TCC * 2);
  s.B1h = o; o = al(o + TCC * s.nka * 2);
  s.B1l = o; o = al(o + TCC * s.nka * 2);
  s.B1x = o; o = al(o + TCC * s.nka * 2);   // third split of the column operand
  s.A1 = o; o = al(o + 128 * s.nka * 2 * 2);   // hi | lo interleaved per 16 features
  s.As = o; o = al(o + TRC * 16 * 2 * 2);       // squares of features 0..15, hi | lo
  s.Y = o; o = al(o + TRC * YP * 4);
  s.stage = o; o = al(o + (int64_t)kStageCap * 8);   // == TRC * TCC * 4 (dense); CSR col | val
  s.araw = o; o = al(o + (TRC * NK + 16) * 4);
  s.off = o; o = al(o + (TRC + 8) * 4);
  s.rp = o; o = al(o + (kRpMax + 1) * 8);
  s.total = o;
  return s;
}

// byte offset of bf16 element (mn, k) in a K-major no-swizzle tile:
// core matrices of 8 (mn) rows x 8 k-elements, next k core +128 B,
// next 8-row group +sbo
GMF_HD uint32_t kofs(int mn, int k, uint32_t sbo) {
  return (uint32_t)(mn >> 3) * sbo + (uint32_t)(k >> 3) * 128u + (uint32_t)(mn & 7) * 16u +
         (uint32_t)(k & 7) * 2u;
}

// A1 (row features, K-major) with hi and lo interleaved per 16 features:
// row group of 8 rows = per K-step [hi core 0 | hi core 1 | lo core 0 | lo core 1];
// GEMM1 reads hi or lo (LBO 128), GEMM3 reads hi|lo of features 0..15 as one
// MN-major N=32 operand.  sboc = (nka / 16) * 512.
GMF_HD uint32_t a1ofs(int row, int k, int lo, uint32_t sboc) {
  return (uint32_t)(row >> 3) * sboc + (uint32_t)((k >> 4) * 4 + lo * 2 + ((k >> 3) & 1)) * 128u +
         (uint32_t)(row & 7) * 16u + (uint32_t)(k & 7) * 2u;
}

// stacked P rows: dd rows in lane quarters 0-1, hh rows in 2-3; within a
// quarter, chunk rows 8g..8g+7 as hi (8 rows) then lo (8 rows), so a hi row
// and its lo row sit 8 lanes apart in one warp and GEMM3 pairs them with the
// same 8 feature rows (LBO 0)
GMF_HD int stack_hi(int r) { return 32 * (r >> 4) + 16 * ((r >> 3) & 1) + (r & 7); }

GMF_D uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// shared-memory matrix descriptor (no swizzle, Blackwell version bit)
GMF_D uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}

// instruction descriptor: bf16 x bf16 -> fp32, M x N, operand majors
constexpr uint32_t idesc(int M, int N, int a_mn, int b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

GMF_D void umma(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(id), "r"(acc)
      : "memory");
}

GMF_D void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_addr(bar))
               : "memory");
}

GMF_D void mbar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(bar)) : "memory");
}

GMF_D void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(done)
        : "r"(smem_addr(bar)), "r"(parity)
        : "memory");
  } while (!done);
}

GMF_D void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
GMF_D void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
GMF_D void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

GMF_D void tmem_alloc(uint32_t* dst) {   // whole warp
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(dst)),
               "n"(kCols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
GMF_D void tmem_dealloc(uint32_t base) {   // whole warp
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(base), "n"(kCols)
               : "memory");
}

// 32 lanes x 16 consecutive TMEM columns -> 16 registers per thread; the
// wait carries the registers so no use is scheduled before the data lands
GMF_D void tmem_ld16(uint32_t addr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15])
      : "r"(addr)
      : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]),
                 "+r"(v[6]), "+r"(v[7]), "+r"(v[8]), "+r"(v[9]), "+r"(v[10]), "+r"(v[11]),
                 "+r"(v[12]), "+r"(v[13]), "+r"(v[14]), "+r"(v[15])
               :
               : "memory");
}

// per-CTA tensor state, persistent across calls (mbarrier phases)
struct Ctx {
  uint32_t tmem;
  uint64_t* bar;   // [0] GEMM1 done, [1] GEMM2+3 done
  uint32_t n1, n23;
};

// CTA prologue / epilogue (all threads)
GMF_D void ctx_open(Ctx& X, uint32_t* s_tmem, uint64_t* s_bar) {
  if (threadIdx.x < 32) tmem_alloc(s_tmem);
  if (threadIdx.x == 0) {
    mbar_init(&s_bar[0]);
    mbar_init(&s_bar[1]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  fence_before();
  __syncthreads();
  fence_after();
  X.tmem = *s_tmem;
  X.bar = s_bar;
  X.n1 = 0;
  X.n23 = 0;
}
GMF_D void ctx_close(const Ctx& X) {
  fence_before();
  __syncthreads();
  fence_after();
  if (threadIdx.x < 32) tmem_dealloc(X.tmem);
}

GMF_D void split_bf16(float x, __nv_bfloat16& hi, __nv_bfloat16& lo) {
  hi = __float2bfloat16_rn(x);
  lo = __float2bfloat16_rn(x - __bfloat162float(hi));
}

// 16 consecutive fp32 values -> bf16 hi at stacked row m_hi and lo at m_lo
// of the P tile, columns c0..c0+15 (two 16-byte core rows each)
GMF_D void put_split16(const float (&x)[16], unsigned char* Pb, int m_hi, int m_lo, int c0) {
  uint32_t hi[8], lo[8];
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
  *reinterpret_cast<uint4*>(Pb + kofs(m_hi, c0, SBO_P)) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
  *reinterpret_cast<uint4*>(Pb + kofs(m_hi, c0 + 8, SBO_P)) = make_uint4(hi[4], hi[5], hi[6], hi[7]);
  *reinterpret_cast<uint4*>(Pb + kofs(m_lo, c0, SBO_P)) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
  *reinterpret_cast<uint4*>(Pb + kofs(m_lo, c0 + 8, SBO_P)) = make_uint4(lo[4], lo[5], lo[6], lo[7]);
}

GMF_D void cp_async16(void* sdst, const void* gsrc) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gsrc) : "memory");
}

// Stage elements [begin, end) of a 4-byte array of `total` elements into
// shared memory (block-cooperative): whole 16-byte quads inside the array by
// 16-byte cp.async, the array's ragged tail by 4-byte copies.  The quad
// containing `begin` starts at dst, so element `begin` lands at dst[begin % 4];
// returns that offset.
GMF_D int stage_range4(void* dst, const void* src, int64_t begin, int64_t end, int64_t total) {
  const int64_t b4 = begin & ~int64_t(3);
  const int64_t nq = (end - b4 + 3) >> 2;
  const int64_t full = total >> 2;
  for (int64_t qi = threadIdx.x; qi < nq; qi += kThreads) {
    const int64_t qg = (b4 >> 2) + qi;
    char* d = reinterpret_cast<char*>(dst) + qi * 16;
    const char* sp = reinterpret_cast<const char*>(src);
    if (qg < full) {
      cp_async16(d, sp + qg * 16);
    } else {
      #pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t e = qg * 4 + u;
        cp_async<4>(d + 4 * u, sp + (e < total ? e : 0) * 4, e < total);
      }
    }
  }
  return (int)(begin - b4);
}

// 8 fp32 values -> packed bf16 hi (4 words) and lo = bf16(x - hi) (4 words)
GMF_D void split8(const float (&x)[8], uint4& hi, uint4& lo) {
  uint32_t h[4], l[4];
  #pragma unroll
  for (int u = 0; u < 4; ++u) {
    const float a = x[2 * u], b = x[2 * u + 1];
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(h[u]) : "f"(b), "f"(a));
    const float ra = a - __uint_as_float(h[u] << 16);
    const float rb = b - __uint_as_float(h[u] & 0xffff0000u);
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(l[u]) : "f"(rb), "f"(ra));
  }
  hi = make_uint4(h[0], h[1], h[2], h[3]);
  lo = make_uint4(l[0], l[1], l[2], l[3]);
}

// 8 fp32 values -> three bf16 splits x = s0 + s1 + s2 (error ~2^-24 |x|)
GMF_D void split3_8(const float (&x)[8], uint4& s0, uint4& s1, uint4& s2) {
  uint32_t a[4], b[4], c[4];
  #pragma unroll
  for (int u = 0; u < 4; ++u) {
    const float x0 = x[2 * u], x1 = x[2 * u + 1];
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(a[u]) : "f"(x1), "f"(x0));
    const float r0 = x0 - __uint_as_float(a[u] << 16);
    const float r1 = x1 - __uint_as_float(a[u] & 0xffff0000u);
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(b[u]) : "f"(r1), "f"(r0));
    const float q0 = r0 - __uint_as_float(b[u] << 16);
    const float q1 = r1 - __uint_as_float(b[u] & 0xffff0000u);
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(c[u]) : "f"(q1), "f"(q0));
  }
  s0 = make_uint4(a[0], a[1], a[2], a[3]);
  s1 = make_uint4(b[0], b[1], b[2], b[3]);
  s2 = make_uint4(c[0], c[1], c[2], c[3]);
}

GMF_D void split3_bf16(float x, __nv_bfloat16& a, __nv_bfloat16& b, __nv_bfloat16& c) {
  a = __float2bfloat16_rn(x);
  const float r = x - __bfloat162float(a);
  b = __float2bfloat16_rn(r);
  c = __float2bfloat16_rn(r - __bfloat162float(b));
}

// ---- column-operand images (persistent kernel, all columns every step) ----
GMF_HD int64_t colimg_bytes(int NK) {
  const Smem L = smem_layout(NK);
  return L.B1x + (L.B1l - L.B1h) - L.R;   // R | B1h | B1l | B1x, contiguous in smem
}

// task t of column tile ct: R rows (feature k, 8 columns) then B1 rows
// (column, 8 features), written into the tile's image exactly as K1 would
// build them in shared memory
template <int NK>
GMF_D void colimg_task(const Params& P, int ct, int t) {
  const Smem L = smem_layout(NK);
  const int nka = L.nka, ng1 = nka / 8;
  const uint32_t sbo1 = (uint32_t)(nka / 8) * 128u;
  unsigned char* img = reinterpret_cast<unsigned char*>(P.colimg) + (int64_t)ct * colimg_bytes(NK);
  unsigned char* Rb = img, *B1h = img + (L.B1h - L.R), *B1l = img + (L.B1l - L.R),
                *B1x = img + (L.B1x - L.R);
  const float* th_col = tptr<float>(P.th_col);
  const float* zg = tptr<float>(P.z);
  const int Kr = P.Kr, Kc = P.Kc, KA = P.KA, p = P.p, q = P.q;
  const int64_t cbase = (int64_t)ct * TCC;
  const int ncv = (int)(P.m - cbase < TCC ? P.m - cbase : TCC);
  if (t < 16 * (TCC / 8)) {
    const int rk = t / (TCC / 8), rcg = t % (TCC / 8);
    float v[8], v2[8];
    #pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int c = 8 * rcg + u;
      const bool ok = c < ncv && rk < Kr;
      const int64_t j = cbase + c;
      v[u] = !ok ? 0.f : (rk < q ? zg[j * q + rk] : th_col[j * Kc + p + (rk - q)]);
      v2[u] = v[u] * v[u];
    }
    uint4 h, l, h2, l2;
    split8(v, h, l);
    split8(v2, h2, l2);
    *reinterpret_cast<uint4*>(Rb + kofs(rk, 8 * rcg, SBO_P)) = h;
    *reinterpret_cast<uint4*>(Rb + kofs(16 + rk, 8 * rcg, SBO_P)) = l;
    *reinterpret_cast<uint4*>(Rb + kofs(32 + rk, 8 * rcg, SBO_P)) = h2;
    *reinterpret_cast<uint4*>(Rb + kofs(48 + rk, 8 * rcg, SBO_P)) = l2;
    return;
  }
  t -= 16 * (TCC / 8);
  if (t >= TCC * ng1) return;
  const int c = t / ng1, g = t % ng1;
  const bool ok = c < ncv;
  const int64_t j = cbase + c;
  float v[8];
  #pragma unroll
  for (int u = 0; u < 8; ++u) {
    const int k = 8 * g + u;
    float x = 0.f;
    if (ok && k < Kc) x = th_col[j * Kc + k];
    else if (ok && k < KA) x = zg[j * q + (k - Kc)];
    v[u] = x * 1.4426950408889634f;
  }
  uint4 h, l, x;
  split3_8(v, h, l, x);
  *reinterpret_cast<uint4*>(B1h + kofs(c, 8 * g, sbo1)) = h;
  *reinterpret_cast<uint4*>(B1l + kofs(c, 8 * g, sbo1)) = l;
  *reinterpret_cast<uint4*>(B1x + kofs(c, 8 * g, sbo1)) = x;
}

template <int NK>
GMF_HD int colimg_tasks() { return 16 * (TCC / 8) + TCC * ((NK <= 16 ? 16 : 32) / 8); }

// column j's coordinate k (of [b | v]) changed to v: its B1 and R entries
template <int NK>
GMF_D void colimg_write(const Params& P, int64_t j, int k, float v) {
  const Smem L = smem_layout(NK);
  const uint32_t sbo1 = (uint32_t)(L.nka / 8) * 128u;
  const int ct = (int)(j / TCC), c = (int)(j % TCC);
  unsigned char* img = reinterpret_cast<unsigned char*>(P.colimg) + (int64_t)ct * colimg_bytes(NK);
  __nv_bfloat16 h, l, x;
  split3_bf16(v * 1.4426950408889634f, h, l, x);
  *reinterpret_cast<__nv_bfloat16*>(img + (L.B1h - L.R) + kofs(c, k, sbo1)) = h;
  *reinterpret_cast<__nv_bfloat16*>(img + (L.B1l - L.R) + kofs(c, k, sbo1)) = l;
  *reinterpret_cast<__nv_bfloat16*>(img + (L.B1x - L.R) + kofs(c, k, sbo1)) = x;
  if (k >= P.p) {
    const int kr = P.q + (k - P.p);
    __nv_bfloat16 h2, l2;
    split_bf16(v, h, l);
    split_bf16(v * v, h2, l2);
    *reinterpret_cast<__nv_bfloat16*>(img + kofs(kr, c, SBO_P)) = h;
    *reinterpret_cast<__nv_bfloat16*>(img + kofs(16 + kr, c, SBO_P)) = l;
    *reinterpret_cast<__nv_bfloat16*>(img + kofs(32 + kr, c, SBO_P)) = h2;
    *reinterpret_cast<__nv_bfloat16*>(img + kofs(48 + kr, c, SBO_P)) = l2;
  }
}

template <int FAM, int NK>
GMF_D void grad_cta(const Params& P, long long blk, long long s, double alpha, int rs, int ct, int RS,
                    unsigned char* smem, Ctx& X, unsigned long long* kp) {
  // optional sub-phase clocks (thread 0, accumulated): 0 column operands,
  // 1 staging wait + GEMM2/3(c-1) wait, 2 Y + A1, 3 next staging + GEMM1
  // issue, 4 D2 readout, 5 elementwise, 6 GEMM2/3 issue, 7 drain
  long long tk = (kp && threadIdx.x == 0) ? clock64() : 0;
  long long kacc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  auto tick = [&](int i) {
    if (kp && threadIdx.x == 0) {
      const long long t = clock64();
      kacc[i] += t - tk;
      tk = t;
    }
  };
  using T = float;
  __shared__ double red_scr[kThreads / 32];
  __shared__ int stage_n;
  __shared__ int s_oth, s_ox, s_oo, s_ocsr;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int qd = warp & 3, hf = warp >> 2;
  const int Kr = P.Kr, Kc = P.Kc, KA = P.KA, p = P.p, q = P.q;
  const int64_t r0 = P.rbp[blk], nI = P.rbp[blk + 1] - r0;
  const int64_t j0 = P.cbp[s], nJ = P.cbp[s + 1] - j0;
  const int64_t rlo = nI * rs / RS, rhi = nI * (rs + 1) / RS;
  const int64_t nrows = rhi - rlo;
  const bool csr = P.yfmt != GMF_Y_DENSE_I32;
  const bool rp_staged = csr && nrows <= kRpMax;
  const int64_t cbase = (int64_t)ct * TCC;
  const int64_t ncv64 = nJ - cbase;
  const int ncv = ncv64 < 0 ? 0 : (ncv64 > TCC ? TCC : (int)ncv64);   // valid tile columns
  const Smem L = smem_layout(NK);
  const int nka = L.nka;
  const uint32_t sbo1 = (uint32_t)(nka / 8) * 128u;   // B1
  const uint32_t sboc = (uint32_t)(nka / 16) * 512u;  // A1 (hi | lo)
  const uint32_t sb = smem_addr(smem);

  unsigned char* Pb = smem + L.P;
  unsigned char* Rb = smem + L.R;
  unsigned char* B1h = smem + L.B1h;
  unsigned char* B1l = smem + L.B1l;
  unsigned char* B1x = smem + L.B1x;
  unsigned char* A1b = smem + L.A1;
  unsigned char* Asb = smem + L.As;
  int32_t* Y = reinterpret_cast<int32_t*>(smem + L.Y);
  unsigned char* st = smem + L.stage;
  T* araw = reinterpret_cast<T*>(smem + L.araw);
  T* off_s = reinterpret_cast<T*>(smem + L.off);
  int64_t* rp_s = reinterpret_cast<int64_t*>(smem + L.rp);

  const T* th_row = tptr<T>(P.th_row);
  const T* th_col = tptr<T>(P.th_col);
  const T* xg = tptr<T>(P.x);
  const T* zg = tptr<T>(P.z);
  const T* offg = tptr<T>(P.off);
  const T pre = 1.4426950408889634f;
  T* colpart = tptr<T>(P.colpart);
  const int64_t cpb = ((int64_t)ct * RS + rs) * TCC * (2 * Kc);

  __syncthreads();   // shared memory reuse across calls (persistent kernel)
  if (nrows <= 0) {   // nothing to do: zero column partials and NB sums
    for (int e = tid; e < TCC * 2 * Kc; e += kThreads) colpart[cpb + e] = T(0);
    if (tid == 0) {
      P.nbpart[2 * ((int64_t)ct * RS + rs)] = 0.0;
      P.nbpart[2 * ((int64_t)ct * RS + rs) + 1] = 0.0;
    }
    return;
  }

  // ---- asynchronous staging of one chunk: its rows are contiguous in the
  // block-major layout, so theta_row, x, offsets and the CSR range are four
  // contiguous ranges (16-byte cp.async) ----
  T* thr_s = araw;                          // rows x Kr (+ alignment slack)
  T* xr_s = araw + TRC * Kr + 8;            // rows x p
  auto issue = [&](int64_t rowbase) {
    const int rows = (int)((rhi - rowbase) < TRC ? (rhi - rowbase) : TRC);
    const int64_t i0 = r0 + rowbase;
    const int oth = stage_range4(thr_s, th_row, i0 * Kr, (i0 + rows) * Kr, P.n * Kr);
    const int ox = p ? stage_range4(xr_s, xg, i0 * p, (i0 + rows) * p, P.n * p) : 0;
    const int oo = P.has_off ? stage_range4(off_s, offg, i0, i0 + rows, P.n) : 0;
    int ocsr = 0;
    if (!csr) {
      int32_t* y_b = reinterpret_cast<int32_t*>(st);
      for (int e = tid; e < TRC * TCC; e += kThreads) {
        const int rr = e / TCC, cc = e % TCC;
        const bool ok = rr < rows && cc < ncv;
        const int64_t pos = cbase + cc;
        const int64_t jj = ok ? (P.col_identity ? pos : (int64_t)P.cidx[j0 + pos]) : 0;
        cp_async<4>(y_b + e, ok ? P.y + (i0 + rr) * P.m + jj : P.y, ok);
      }
    } else if (rp_staged) {
      const int64_t lo = rp_s[rowbase - rlo], hi = rp_s[rowbase - rlo + rows];
      if (hi - lo + 6 <= kStageCap) {
        int32_t* col_b = reinterpret_cast<int32_t*>(st);
        int32_t* val_b = col_b + kStageCap;
        ocsr = stage_range4(col_b, P.ci, lo, hi, P.nnz);
        if (P.yfmt != GMF_Y_CSR_PACK32) stage_range4(val_b, P.cv, lo, hi, P.nnz);
        if (tid == 0) stage_n = (int)(hi - lo);
      } else if (tid == 0) {
        stage_n = -1;
      }
    } else if (tid == 0) {
      stage_n = -1;
    }
    if (tid == 0) { s_oth = oth; s_ox = ox; s_oo = oo; s_ocsr = ocsr; }
    cp_async_commit();
  };

  // ---- column operands of the tile (once per call); global loads first ----
  // feature order a = [x | u | gamma], c = [b | v | z]
  // B1: thread per (column, 8 features); R: thread per (feature, 8 columns).
  // In the persistent kernel with all columns every step, the column updates
  // keep a byte image of R | B1h | B1l per tile: one 16-byte cp.async copy.
  const int ng1 = nka / 8;
  const bool use_img = P.colimg_on != 0;
  if (use_img) {
    const int64_t nb = colimg_bytes(NK);
    const unsigned char* img = reinterpret_cast<const unsigned char*>(P.colimg) + (int64_t)ct * nb;
    for (int64_t o = (int64_t)tid * 16; o < nb; o += (int64_t)kThreads * 16)
      cp_async16(Rb + o, img + o);
  }
  float b1v[8], rv[8];
  int b1c = 0, b1g = 0, rk = 0, rcg = 0;
  const bool b1_task = !use_img;
  if (!use_img) {
    const int t = tid;
    b1c = t / ng1; b1g = t % ng1;
    const int64_t pos = cbase + b1c;
    const bool ok = b1c < ncv;
    const int64_t j = ok ? (P.col_identity ? pos : (int64_t)P.cidx[j0 + pos]) : 0;
    #pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int k = 8 * b1g + u;
      const bool in_c = ok && k < Kc, in_z = ok && k >= Kc && k < KA;
      const float* src = in_c ? th_col + j * Kc + k : (in_z ? zg + j * q + (k - Kc) : th_col);
      const float x = *src;
      b1v[u] = (in_c || in_z) ? x * pre : 0.f;
    }
    rk = t / (TCC / 8); rcg = t % (TCC / 8);
    #pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int c = 8 * rcg + u;
      const bool okr = c < ncv && rk < Kr;
      const int64_t posr = cbase + c;
      const int64_t jr = okr ? (P.col_identity ? posr : (int64_t)P.cidx[j0 + posr]) : 0;
      const float* src = !okr ? th_col : (rk < q ? zg + jr * q + rk : th_col + jr * Kc + p + (rk - q));
      const float x = *src;
      rv[u] = okr ? x : 0.f;
    }
  }
  if (rp_staged)
    for (int64_t e = tid; e <= nrows; e += kThreads) rp_s[e] = P.rp[r0 + rlo + e];
  for (int e = tid; e < TRC * YP; e += kThreads) Y[e] = 0;
  __syncthreads();   // rp staged
  issue(rlo);   // (commits the image copy with the first chunk's staging)
  if (!use_img) {
    uint4 h, l;
    if (b1_task) {
      uint4 x;
      split3_8(b1v, h, l, x);
      *reinterpret_cast<uint4*>(B1h + kofs(b1c, 8 * b1g, sbo1)) = h;
      *reinterpret_cast<uint4*>(B1l + kofs(b1c, 8 * b1g, sbo1)) = l;
      *reinterpret_cast<uint4*>(B1x + kofs(b1c, 8 * b1g, sbo1)) = x;
    }
    float r2[8];
    #pragma unroll
    for (int u = 0; u < 8; ++u) r2[u] = rv[u] * rv[u];
    uint4 h2, l2;
    split8(rv, h, l);
    split8(r2, h2, l2);
    *reinterpret_cast<uint4*>(Rb + kofs(rk, 8 * rcg, SBO_P)) = h;
    *reinterpret_cast<uint4*>(Rb + kofs(16 + rk, 8 * rcg, SBO_P)) = l;
    *reinterpret_cast<uint4*>(Rb + kofs(32 + rk, 8 * rcg, SBO_P)) = h2;
    *reinterpret_cast<uint4*>(Rb + kofs(48 + rk, 8 * rcg, SBO_P)) = l2;
  }
  if (ng1 == 4 && !use_img) {   // K = 32: the second half of the B1 tasks
    const int t = tid + kThreads;
    const int c = t / ng1, g = t % ng1;
    const int64_t pos = cbase + c;
    const bool ok = c < ncv;
    const int64_t j = ok ? (P.col_identity ? pos : (int64_t)P.cidx[j0 + pos]) : 0;
    float v[8];
    #pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int k = 8 * g + u;
      const bool in_c = ok && k < Kc, in_z = ok && k >= Kc && k < KA;
      const float* src = in_c ? th_col + j * Kc + k : (in_z ? zg + j * q + (k - Kc) : th_col);
      const float x = *src;
      v[u] = (in_c || in_z) ? x * pre : 0.f;
    }
    uint4 h, l, x;
    split3_8(v, h, l, x);
    *reinterpret_cast<uint4*>(B1h + kofs(c, 8 * g, sbo1)) = h;
    *reinterpret_cast<uint4*>(B1l + kofs(c, 8 * g, sbo1)) = l;
    *reinterpret_cast<uint4*>(B1x + kofs(c, 8 * g, sbo1)) = x;
  }
  tick(0);

  const T rphi = T(1.0 / P.phi);
  const T ralpha = T(1.0 / alpha);
  const T tphi = T(P.phi);
  const T tra = tphi * ralpha;
  const uint32_t tm = X.tmem;
  constexpr uint32_t ID1 = idesc(128, 128, 0, 0);
  constexpr uint32_t ID2 = idesc(128, 64, 0, 0);
  constexpr uint32_t ID3 = idesc(128, 32, 1, 1);
  const int c0 = 32 * qd + 16 * hf;                 // this thread's first tile column
  const int vcols = ncv - c0 < 0 ? 0 : (ncv - c0 > 16 ? 16 : ncv - c0);
  const uint32_t lane_base = (uint32_t)(32 * qd) << 16;
  double nb_num = 0.0, nb_den = 0.0;
  T* rowpart = tptr<T>(P.rowpart);
  const int rkk = 2 * Kr;
  // A1 task of this thread: (replica, row, 8-feature group)
  const int a_rep = tid / (TRC * 2), a_rr = (tid / 2) % TRC, a_g2 = tid & 1;

  // D2 readout (warps 0-3): quarters 0-1 hold dd rows, 2-3 hh rows (stack_hi);
  // each lane adds its Rd_hi and Rd_lo halves, then its hi/lo partner 8
  // lanes away; the hi lane writes the row's Kr values
  auto readout_d2 = [&](int64_t rowbase, int rows) {
    float dv[16];
    uint32_t a[16], b[16];
    const uint32_t col = tm + lane_base + T_D2 + (qd >= 2 ? 32u : 0u);
    tmem_ld16(col, a);
    tmem_ld16(col + 16, b);
    #pragma unroll
    for (int k = 0; k < 16; ++k) {
      dv[k] = __uint_as_float(a[k]) + __uint_as_float(b[k]);
      dv[k] += __shfl_xor_sync(0xffffffffu, dv[k], 8);
    }
    const int r = 16 * (qd & 1) + 8 * (lane >> 4) + (lane & 7);
    if (!(lane & 8) && r < rows) {
      T* outp = rowpart + ((int64_t)ct * P.nstar_max + rowbase + r) * rkk + (qd < 2 ? 0 : Kr);
      #pragma unroll
      for (int k = 0; k < 16; ++k)
        if (k < Kr) outp[k] = dv[k];
    }
  };

  int64_t prev_rowbase = -1;
  int prev_rows = 0;
  bool first3 = true;
  for (int64_t rowbase = rlo; rowbase < rhi; rowbase += TRC) {
    const int rows = (int)((rhi - rowbase) < TRC ? (rhi - rowbase) : TRC);
    const int64_t i0 = r0 + rowbase;
    // ---- S1: chunk staged; GEMM2/3 of the previous chunk done (frees P, A1, D2) ----
    cp_async_wait0();
    if (prev_rowbase >= 0) {
      mbar_wait(&X.bar[1], X.n23 & 1u);
      ++X.n23;
    }
    fence_after();
    __syncthreads();
    tick(1);
    // ---- S2: Y tile and A1 = a_i (hi/lo, four replicas) + a_i^2 (hi/lo) ----
    if (!csr) {
      const int32_t* y_b = reinterpret_cast<const int32_t*>(st);
      for (int e = tid; e < TRC * TCC; e += kThreads) Y[(e / TCC) * YP + (e % TCC)] = y_b[e];
    } else {
      const int n_st = stage_n;
      if (n_st >= 0) {
        const int32_t* col_b = reinterpret_cast<const int32_t*>(st);
        const int32_t* val_b = col_b + kStageCap;
        const int64_t* rpc = rp_s + (rowbase - rlo);
        const int lo = (int)rpc[0] - s_ocsr;
        for (int rr = warp; rr < rows; rr += kThreads / 32) {
          const int a = (int)rpc[rr] - lo, bnd = (int)rpc[rr + 1] - lo;
          const int pack = P.yfmt == GMF_Y_CSR_PACK32;
          for (int e = a + lane; e < bnd; e += 32) {
            const int32_t w = col_b[e];
            const int col = stg_col(pack, w);
            const int pp = P.col_identity ? col : ((P.cbof[col] == s) ? P.cpos[col] : -1);
            const int cl = pp - (int)cbase;
            if (pp >= 0 && cl >= 0 && cl < TCC) Y[rr * YP + cl] = stg_val(pack, w, pack ? 0 : val_b[e]);
          }
        }
      } else {   // too many nonzeros to stage: direct loads, this tile's range only
        const bool tix = P.tidx != nullptr && !P.stream_mode;
        for (int rr = warp; rr < rows; rr += kThreads / 32) {
          const int64_t i = i0 + rr;
          int64_t k0 = P.rp[i], k1 = P.rp[i + 1];
          if (tix) {
            const int32_t* tr = P.tidx + i * (P.CT + 1) + ct;
            k1 = k0 + tr[1];
            k0 += tr[0];
          }
          for (int64_t k = k0 + lane; k < k1; k += 32) {
            const int col = csr_col_at(P, k);
            const int64_t pp = P.col_identity ? col : ((P.cbof[col] == s) ? (int64_t)P.cpos[col] : -1);
            const int64_t cl = pp - cbase;
            if (pp >= 0 && cl >= 0 && cl < TCC) Y[rr * YP + cl] = csr_val_at(P, k);
          }
        }
      }
    }
    {
      const T* thr = thr_s + s_oth + a_rr * Kr;
      const T* xr = xr_s + s_ox + a_rr * p;
      const bool rok = a_rr < rows;
      for (int g = a_g2; g < ng1; g += 2) {
        float v[8], v2[8];
        #pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int k = 8 * g + u;
          // a_k: x_k (k < p), else theta_row[(k - p + q) mod Kr] = u then gamma
          int kt = k - p + q;
          kt = kt >= Kr ? kt - Kr : kt;
          kt = (k >= p && k < KA) ? kt : 0;
          const int kx = k < p ? k : 0;
          const float tv = thr[kt], xv = xr[kx];
          v[u] = !rok ? 0.f : (k < p ? xv : (k < KA ? tv : 0.f));
          v2[u] = v[u] * v[u];
        }
        uint4 h, l;
        split8(v, h, l);
        *reinterpret_cast<uint4*>(A1b + a1ofs(32 * a_rep + a_rr, 8 * g, 0, sboc)) = h;
        *reinterpret_cast<uint4*>(A1b + a1ofs(32 * a_rep + a_rr, 8 * g, 1, sboc)) = l;
        if (a_rep == 0 && g < 2) {   // squares of features 0..15 (the column side's [x | u])
          split8(v2, h, l);
          *reinterpret_cast<uint4*>(Asb + a1ofs(a_rr, 8 * g, 0, 512u)) = h;
          *reinterpret_cast<uint4*>(Asb + a1ofs(a_rr, 8 * g, 1, 512u)) = l;
        }
      }
    }
    const T offr = (lane < rows && P.has_off) ? off_s[s_oo + lane] * pre : T(0);
    fence_async_smem();
    __syncthreads();   // Y, A1 written; staging consumed
    tick(2);
    // ---- S3: prefetch the next chunk, GEMM1 eta = A1 . B1^T ----
    if (rowbase + TRC < rhi) issue(rowbase + TRC);
    if (tid == 0) {
      fence_after();
      for (int kt = 0; kt < nka / 16; ++kt) {
        const uint32_t ko = (uint32_t)kt * 256u;
        const uint64_t ah = sdesc(sb + (uint32_t)L.A1 + (uint32_t)kt * 512u, 128, sboc);
        const uint64_t al = sdesc(sb + (uint32_t)L.A1 + (uint32_t)kt * 512u + 256u, 128, sboc);
        const uint64_t bh = sdesc(sb + (uint32_t)L.B1h + ko, 128, sbo1);
        const uint64_t bl = sdesc(sb + (uint32_t)L.B1l + ko, 128, sbo1);
        const uint64_t bx = sdesc(sb + (uint32_t)L.B1x + ko, 128, sbo1);
        umma(tm + T_ETA, ah, bh, ID1, kt > 0 ? 1u : 0u);
        umma(tm + T_ETA, ah, bl, ID1, 1u);
        umma(tm + T_ETA, al, bh, ID1, 1u);
        umma(tm + T_ETA, ah, bx, ID1, 1u);   // the column side's third split (intercepts)
      }
      umma_commit(&X.bar[0]);
    }
    tick(3);
    // ---- S4: previous chunk's row side (warps 0-3) ----
    if (prev_rowbase >= 0 && hf == 0) readout_d2(prev_rowbase, prev_rows);
    tick(4);
    // ---- S5: elementwise, thread = chunk row `lane`, columns c0..c0+15 ----
    mbar_wait(&X.bar[0], X.n1 & 1u);
    ++X.n1;
    fence_after();
    uint32_t ev[16];
    tmem_ld16(tm + lane_base + T_ETA + (uint32_t)c0, ev);
    int4* yrow = reinterpret_cast<int4*>(Y + lane * YP + c0);
    int yv[16];
    #pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int4 t4 = yrow[u];
      yv[4 * u] = t4.x; yv[4 * u + 1] = t4.y; yv[4 * u + 2] = t4.z; yv[4 * u + 3] = t4.w;
    }
    const bool row_ok = lane < rows;
    float dd[16], hh[16];
    float cn = 0.f, cdn = 0.f;
    // a full row of 16 valid columns (the common case) skips the masking
    auto entries = [&](auto masked) {
      #pragma unroll
      for (int i = 0; i < 16; ++i) {
        const float w = masked ? ((row_ok && i < vcols) ? 1.f : 0.f) : 1.f;
        const float mu = exp_pre(__uint_as_float(ev[i]) + offr);
        const float r = (float)yv[i] - mu;
        if (FAM == 0) {
          const float ws = masked ? w * rphi : rphi;
          dd[i] = -ws * r;
          hh[i] = ws * mu;
        } else {
          const float rc = rcp_fast(fmaf(mu, tra, tphi));
          const float inv = masked ? w * rc : rc;
          dd[i] = -r * inv;
          hh[i] = mu * inv;
          cn = fmaf(masked ? w * mu : mu, mu, cn);
          cdn = masked ? fmaf(w, fmaf(r, r, -mu), cdn) : cdn + fmaf(r, r, -mu);
        }
      }
    };
    if (row_ok && vcols == 16) entries(std::false_type{});
    else entries(std::true_type{});
    nb_num += (double)cn;
    nb_den += (double)cdn;
    put_split16(dd, Pb, stack_hi(lane), stack_hi(lane) + 8, c0);
    put_split16(hh, Pb, 64 + stack_hi(lane), 64 + stack_hi(lane) + 8, c0);
    if (csr) {
      const int4 z4 = make_int4(0, 0, 0, 0);
      #pragma unroll
      for (int u = 0; u < 4; ++u) yrow[u] = z4;
    }
    fence_async_smem();
    fence_before();
    __syncthreads();
    tick(5);
    // ---- S6: GEMM2 (row side) and GEMM3 (column side) ----
    if (tid == 0) {
      fence_after();
      #pragma unroll
      for (int kt = 0; kt < TCC / 16; ++kt) {
        const uint32_t ko = (uint32_t)kt * 256u;
        umma(tm + T_D2, sdesc(sb + (uint32_t)L.P + ko, 128, SBO_P),
             sdesc(sb + (uint32_t)L.R + ko, 128, SBO_P), ID2, kt > 0 ? 1u : 0u);
      }
      // D3[col][f] += P^T . [a_hi | a_lo] (dd) and P^T . [a2_hi | a2_lo] (hh),
      // features 0..15; K-step u = stacked rows 16u..16u+15 = chunk rows
      // 8u..8u+7 hi then lo, paired with feature rows 8u..8u+7 twice (LBO 0).
      // P read MN-major (column chunks +128 B, 8-row K groups +2048 B).
      #pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t acc0 = (first3 && u == 0) ? 0u : 1u;
        umma(tm + T_D3, sdesc(sb + (uint32_t)L.P + 4096u * u, 2048, 128),
             sdesc(sb + (uint32_t)L.A1 + sboc * u, 0, 128), ID3, acc0);
        umma(tm + T_D3 + 32, sdesc(sb + (uint32_t)L.P + 16384u + 4096u * u, 2048, 128),
             sdesc(sb + (uint32_t)L.As + 512u * u, 0, 128), ID3, acc0);
      }
      umma_commit(&X.bar[1]);
    }
    first3 = false;
    tick(6);
    prev_rowbase = rowbase;   // block-relative row index of the chunk
    prev_rows = rows;
  }
  cp_async_wait0();
  // ---- drain: last chunk's row side, then the column side ----
  mbar_wait(&X.bar[1], X.n23 & 1u);
  ++X.n23;
  fence_after();
  if (hf == 0) readout_d2(prev_rowbase, prev_rows);
  {
    // lane = tile column; D3 columns = a-features [x | u | gamma], whose first
    // Kc are the column side's [x | u]
    uint32_t a[16], b[16];
    const uint32_t col = tm + lane_base + T_D3 + (hf ? 32u : 0u);
    const int c = 32 * qd + lane;
    T* outp = colpart + cpb + (int64_t)c * (2 * Kc) + (hf ? Kc : 0);
    tmem_ld16(col, a);
    tmem_ld16(col + 16, b);
    #pragma unroll
    for (int f = 0; f < 16; ++f)
      if (f < Kc) outp[f] = __uint_as_float(a[f]) + __uint_as_float(b[f]);
  }
  fence_before();
  const double bn = block_sum<kThreads>(nb_num, red_scr);
  const double bd = block_sum<kThreads>(nb_den, red_scr);
  if (tid == 0) {
    P.nbpart[2 * ((int64_t)ct * RS + rs)] = bn;
    P.nbpart[2 * ((int64_t)ct * RS + rs) + 1] = bd;
  }
  tick(7);
  if (kp && tid == 0)
    for (int i = 0; i < 8; ++i) atomicAdd(kp + i, (unsigned long long)kacc[i]);   // no read-back
}

}  // namespace tc
}  // namespace gmf
