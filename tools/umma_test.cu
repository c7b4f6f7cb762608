// Standalone tcgen05 (UMMA) probe: one MMA D[M x N] = A[M x K] B[N x K]^T with
// K = 32 bytes of operand (8 tf32 or 16 bf16), operands in shared memory in the
// canonical no-swizzle / 128B-swizzle layouts (K-major or MN-major),
// accumulator in TMEM, read back with tcgen05.ld.  Inputs are small integers
// (exact in tf32 and bf16), so results must match the CPU bitwise.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o umma_test umma_test.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// es = element bytes, epc = elements per 16-byte chunk
// K-major no swizzle: core = 8 MN rows x 16 B of K; LBO = next K core, SBO = next 8 MN rows
__host__ __device__ int off_k_none(int r, int k, int es, int lbo, int sbo) {
  const int epc = 16 / es;
  return (r / 8) * sbo + (k / epc) * lbo + (r % 8) * 16 + (k % epc) * es;
}
// MN-major no swizzle: core = 8 K rows x 16 B of MN; SBO = next MN chunk, LBO = next 8 K rows
__host__ __device__ int off_mn_none(int mn, int k, int es, int lbo, int sbo) {
  const int epc = 16 / es;
  return (mn / epc) * sbo + (k / 8) * lbo + (k % 8) * 16 + (mn % epc) * es;
}
// MN-major 128B swizzle: atom = 128 B of MN x 8 K rows; LBO = next MN atom, SBO = next 8 K rows
__host__ __device__ int off_mn_sw128(int mn, int k, int es, int lbo, int sbo) {
  const int epa = 128 / es, epc = 16 / es;
  const int row = k % 8, chunk = (mn % epa) / epc;
  return (mn / epa) * lbo + (k / 8) * sbo + row * 128 + ((chunk ^ row) * 16) + (mn % epc) * es;
}
// K-major 128B swizzle: atom = 8 MN rows x 128 B of K; SBO = next 8 MN rows
__host__ __device__ int off_k_sw128(int r, int k, int es, int sbo) {
  const int epa = 128 / es, epc = 16 / es;
  const int row = r % 8, chunk = (k % epa) / epc;
  return (r / 8) * sbo + row * 128 + ((chunk ^ row) * 16) + (k % epc) * es;
}

__device__ __forceinline__ uint64_t make_desc(uint32_t addr, int lbo, int sbo, int layout) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;                 // version (Blackwell)
  d |= (uint64_t)layout << 61;            // 0 none, 2 = 128B swizzle
  return d;
}

struct Opnd {
  int mn;        // 1 = MN-major
  int sw;        // 0 none, 2 = 128B swizzle
  int lbo, sbo;
};
struct Case {
  int M, N, bf;  // bf: 1 = bf16 (kind::f16), 0 = tf32
  Opnd a, b;
};

__host__ __device__ int off(const Opnd& o, int mn, int k, int es) {
  if (o.sw) return o.mn ? off_mn_sw128(mn, k, es, o.lbo, o.sbo) : off_k_sw128(mn, k, es, o.sbo);
  return o.mn ? off_mn_none(mn, k, es, o.lbo, o.sbo) : off_k_none(mn, k, es, o.lbo, o.sbo);
}

__device__ void put(unsigned char* base, int o, float v, int bf) {
  if (bf) *reinterpret_cast<__nv_bfloat16*>(base + o) = __float2bfloat16(v);
  else *reinterpret_cast<float*>(base + o) = v;
}

__global__ void k_umma(Case cs, const float* A, const float* B, float* D) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t mbar;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int es = cs.bf ? 2 : 4, K = 32 / es;
  unsigned char* sa = smem;
  unsigned char* sb = smem + 64 * 1024;
  for (int e = tid; e < 128 * 1024 / 4; e += blockDim.x) reinterpret_cast<float*>(smem)[e] = 0.f;
  __syncthreads();
  for (int e = tid; e < cs.M * K; e += blockDim.x) put(sa, off(cs.a, e / K, e % K, es), A[e], cs.bf);
  for (int e = tid; e < cs.N * K; e += blockDim.x) put(sb, off(cs.b, e / K, e % K, es), B[e], cs.bf);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tmem_base;
  if (tid == 0) {
    const uint64_t da = make_desc(smem_u32(sa), cs.a.lbo, cs.a.sbo, cs.a.sw);
    const uint64_t db = make_desc(smem_u32(sb), cs.b.lbo, cs.b.sbo, cs.b.sw);
    uint32_t idesc = 0;
    idesc |= 1u << 4;                                   // D = F32
    idesc |= (cs.bf ? 1u : 2u) << 7;                    // A = BF16 / TF32
    idesc |= (cs.bf ? 1u : 2u) << 10;                   // B = BF16 / TF32
    idesc |= (uint32_t)cs.a.mn << 15;
    idesc |= (uint32_t)cs.b.mn << 16;
    idesc |= (uint32_t)(cs.N >> 3) << 17;
    idesc |= (uint32_t)(cs.M >> 4) << 24;
    if (cs.bf)
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tm),
          "l"(da), "l"(db), "r"(idesc), "r"(0));
    else
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tm),
          "l"(da), "l"(db), "r"(idesc), "r"(0));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&mbar)));
  }
  {
    uint32_t done = 0;
    while (!done) {
      asm volatile(
          "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
          "selp.u32 %0, 1, 0, p;\n\t}\n" : "=r"(done) : "r"(smem_u32(&mbar)), "r"(0));
    }
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp < 4) {
    const int row = 32 * warp + (tid & 31);
    for (int c0 = 0; c0 < cs.N; c0 += 8) {
      uint32_t v[8];
      const uint32_t addr = tm + ((uint32_t)(32 * warp) << 16) + c0;
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
                     "=r"(v[6]), "=r"(v[7])
                   : "r"(addr));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      if (row < cs.M)
        for (int i = 0; i < 8; ++i) D[row * cs.N + c0 + i] = __uint_as_float(v[i]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(256));
}

int main() {
  const int M = 128, N = 64, KMAX = 16;
  static float hA[M * KMAX], hB[N * KMAX], ref[M * N], out[M * N];
  float *dA, *dB, *dD;
  cudaMalloc(&dA, sizeof(hA));
  cudaMalloc(&dB, sizeof(hB));
  cudaMalloc(&dD, sizeof(out));
  cudaFuncSetAttribute(k_umma, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 1024);
  Case cases[] = {
      {M, N, 0, {0, 0, 128, 256}, {0, 0, 128, 256}},        // tf32 K-major both (known good)
      {M, N, 0, {0, 2, 16, 1024}, {0, 2, 16, 1024}},        // tf32 K-major SW128 (known good)
      {M, N, 0, {1, 0, 4096, 128}, {0, 0, 128, 256}},       // tf32 A MN-major none
      {M, N, 0, {0, 0, 128, 256}, {1, 0, 2048, 128}},       // tf32 B MN-major none
      {M, N, 0, {1, 2, 1024, 4096}, {0, 0, 128, 256}},      // tf32 A MN-major SW128
      {M, N, 1, {0, 0, 128, 256}, {0, 0, 128, 256}},        // bf16 K-major both
      {M, N, 1, {1, 0, 2048, 128}, {0, 0, 128, 256}},       // bf16 A MN-major none
      {M, N, 1, {0, 0, 128, 256}, {1, 0, 1024, 128}},       // bf16 B MN-major none
      {M, N, 1, {1, 2, 1024, 2048}, {0, 0, 128, 256}},      // bf16 A MN-major SW128
      {M, N, 1, {1, 0, 128, 2048}, {0, 0, 128, 256}},       // bf16 A MN-major none, swapped
      {M, N, 1, {1, 0, 2048, 128}, {1, 0, 0, 128}},         // bf16 B MN-major, LBO 0 (K groups alias)
  };
  for (auto& cs : cases) {
    const int K = cs.bf ? 16 : 8;
    for (int r = 0; r < M; ++r)
      for (int k = 0; k < K; ++k) hA[r * K + k] = (float)((r * 7 + k * 3) % 17 - 8);
    for (int n = 0; n < N; ++n)
      for (int k = 0; k < K; ++k) hB[n * K + k] = (float)((n * 5 + k * 11) % 13 - 6);
    if (cs.b.mn && cs.b.lbo == 0)   // aliased K groups: B[n][k] == B[n][k % 8]
      for (int n = 0; n < N; ++n)
        for (int k = 8; k < K; ++k) hB[n * K + k] = hB[n * K + k - 8];
    for (int r = 0; r < M; ++r)
      for (int n = 0; n < N; ++n) {
        float s = 0;
        for (int k = 0; k < K; ++k) s += hA[r * K + k] * hB[n * K + k];
        ref[r * N + n] = s;
      }
    cudaMemcpy(dA, hA, sizeof(hA), cudaMemcpyHostToDevice);
    cudaMemcpy(dB, hB, sizeof(hB), cudaMemcpyHostToDevice);
    cudaMemset(dD, 0, sizeof(out));
    k_umma<<<1, 128, 128 * 1024>>>(cs, dA, dB, dD);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(out, dD, sizeof(out), cudaMemcpyDeviceToHost);
    int bad = 0;
    double maxerr = 0;
    for (int i = 0; i < M * N; ++i) {
      double d = fabs(out[i] - ref[i]);
      if (d > 0) ++bad;
      if (d > maxerr) maxerr = d;
    }
    printf("%s A(mn=%d sw=%d lbo=%d sbo=%d) B(mn=%d sw=%d lbo=%d sbo=%d): %s, mismatches %d/%d, "
           "max err %g, D[0..3]=%g %g %g %g ref %g %g %g %g\n",
           cs.bf ? "bf16" : "tf32", cs.a.mn, cs.a.sw, cs.a.lbo, cs.a.sbo, cs.b.mn, cs.b.sw, cs.b.lbo,
           cs.b.sbo, cudaGetErrorString(e), bad, M * N, maxerr, out[0], out[1], out[2], out[3],
           ref[0], ref[1], ref[2], ref[3]);
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
