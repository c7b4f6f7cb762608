// Standalone tcgen05 (UMMA) probe: one kind::tf32 MMA D[M x N] = A[M x 8] B[N x 8]^T
// with operands in shared memory (no-swizzle canonical layouts, K-major or
// MN-major), accumulator in TMEM, read back with tcgen05.ld.  Inputs are
// small integers (exact in tf32), so results must match the CPU bitwise.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o umma_test umma_test.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// byte offset of element (row, k) in a K-major no-swizzle tile
__host__ __device__ int off_kmajor(int r, int k, int sbo, int lbo) {
  return (r / 8) * sbo + (k / 4) * lbo + (r % 8) * 16 + (k % 4) * 4;
}
// byte offset of element (mn, k) in an MN-major no-swizzle tile
__host__ __device__ int off_mnmajor(int mn, int k, int sbo, int lbo) {
  return (mn / 4) * sbo + (k / 8) * lbo + (k % 8) * 16 + (mn % 4) * 4;
}
// MN-major, 128B swizzle: atom = 32 MN x 8 K (1 KB), 16B chunk ^= K row
__host__ __device__ int off_mn_sw128(int mn, int k, int lbo, int sbo) {
  const int row = k % 8, chunk = (mn % 32) / 4;
  return (mn / 32) * lbo + (k / 8) * sbo + row * 128 + ((chunk ^ row) * 16) + (mn % 4) * 4;
}
// K-major, 128B swizzle: atom = 8 rows x 32 K (1 KB)
__host__ __device__ int off_k_sw128(int r, int k, int sbo) {
  const int row = r % 8, chunk = (k % 32) / 4;
  return (r / 8) * sbo + row * 128 + ((chunk ^ row) * 16) + (k % 4) * 4;
}

__device__ __forceinline__ uint64_t make_desc(uint32_t addr, int lbo, int sbo, int layout = 0) {
  uint64_t d = 0;
  d |= (uint64_t)layout << 61;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;   // version (Blackwell)
  return d;                 // base offset 0, lbo mode 0, layout SWIZZLE_NONE
}

struct Case {
  int M, N, a_mn, b_mn;
  int a_sbo, a_lbo, b_sbo, b_lbo;
  int a_sw, b_sw;   // 0 none, 2 = 128B swizzle
};

__global__ void k_umma(Case cs, const float* A, const float* B, float* D) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t mbar;
  const int tid = threadIdx.x, warp = tid >> 5;
  unsigned char* sa = smem;
  unsigned char* sb = smem + 64 * 1024;
  // stage operands
  for (int e = tid; e < cs.M * 8; e += blockDim.x) {
    const int r = e / 8, k = e % 8;
    const int o = cs.a_sw ? (cs.a_mn ? off_mn_sw128(r, k, cs.a_lbo, cs.a_sbo) : off_k_sw128(r, k, cs.a_sbo))
                          : (cs.a_mn ? off_mnmajor(r, k, cs.a_sbo, cs.a_lbo) : off_kmajor(r, k, cs.a_sbo, cs.a_lbo));
    *reinterpret_cast<float*>(sa + o) = A[r * 8 + k];
  }
  for (int e = tid; e < cs.N * 8; e += blockDim.x) {
    const int n = e / 8, k = e % 8;
    const int o = cs.b_sw ? (cs.b_mn ? off_mn_sw128(n, k, cs.b_lbo, cs.b_sbo) : off_k_sw128(n, k, cs.b_sbo))
                          : (cs.b_mn ? off_mnmajor(n, k, cs.b_sbo, cs.b_lbo) : off_kmajor(n, k, cs.b_sbo, cs.b_lbo));
    *reinterpret_cast<float*>(sb + o) = B[n * 8 + k];
  }
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
    const uint64_t da = make_desc(smem_u32(sa), cs.a_lbo, cs.a_sbo, cs.a_sw);
    const uint64_t db = make_desc(smem_u32(sb), cs.b_lbo, cs.b_sbo, cs.b_sw);
    uint32_t idesc = 0;
    idesc |= 1u << 4;                       // D = F32
    idesc |= 2u << 7;                       // A = TF32
    idesc |= 2u << 10;                      // B = TF32
    idesc |= (uint32_t)cs.a_mn << 15;
    idesc |= (uint32_t)cs.b_mn << 16;
    idesc |= (uint32_t)(cs.N >> 3) << 17;
    idesc |= (uint32_t)(cs.M >> 4) << 24;
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tm),
        "l"(da), "l"(db), "r"(idesc), "r"(0));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&mbar)));
  }
  // wait for the MMA
  {
    uint32_t done = 0;
    while (!done) {
      asm volatile(
          "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
          "selp.u32 %0, 1, 0, p;\n\t}\n" : "=r"(done) : "r"(smem_u32(&mbar)), "r"(0));
    }
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  // thread (warp w, lane l) reads TMEM lane 32w + l: row 32w + l, N columns
  if (warp < 4 && 32 * warp < cs.M) {
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
  const int M = 128, N = 64;
  float hA[M * 8], hB[N * 8], ref[M * N], out[M * N];
  for (int r = 0; r < M; ++r)
    for (int k = 0; k < 8; ++k) hA[r * 8 + k] = (float)((r * 7 + k * 3) % 17 - 8);
  for (int n = 0; n < N; ++n)
    for (int k = 0; k < 8; ++k) hB[n * 8 + k] = (float)((n * 5 + k * 11) % 13 - 6);
  for (int r = 0; r < M; ++r)
    for (int n = 0; n < N; ++n) {
      float s = 0;
      for (int k = 0; k < 8; ++k) s += hA[r * 8 + k] * hB[n * 8 + k];
      ref[r * N + n] = s;
    }
  float *dA, *dB, *dD;
  cudaMalloc(&dA, sizeof(hA));
  cudaMalloc(&dB, sizeof(hB));
  cudaMalloc(&dD, sizeof(out));
  cudaMemcpy(dA, hA, sizeof(hA), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, sizeof(hB), cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k_umma, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 1024);
  Case cases[] = {
      // K-major A & B: core 8 rows x 16 B, LBO = next K core (128), SBO = next 8-row group (256)
      {M, N, 0, 0, 256, 128, 256, 128, 0, 0},
      // K-major with 128B swizzle (SBO = next 8-row atom = 1024)
      {M, N, 0, 0, 1024, 16, 1024, 16, 2, 2},
      // MN-major 128B swizzle A: LBO = next 32-MN atom (1024), SBO = next K group
      {M, N, 1, 0, 4096, 1024, 256, 128, 2, 0},
      {M, N, 1, 0, 1024, 4096, 256, 128, 2, 0},
      // MN-major 128B swizzle B
      {M, N, 0, 1, 256, 128, 2048, 1024, 0, 2},
      {M, N, 0, 1, 256, 128, 1024, 2048, 0, 2},
      // MN-major no swizzle, more LBO/SBO guesses
      {M, N, 1, 0, 128, 128, 256, 128, 0, 0},
      {M, N, 1, 0, 4096, 4096, 256, 128, 0, 0},
  };
  for (auto& cs : cases) {
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
    printf("sw=%d/%d a_mn=%d b_mn=%d a(sbo=%d,lbo=%d) b(sbo=%d,lbo=%d): %s, mismatches %d / %d, max err %g, D[0..3]=%g %g %g %g ref %g %g %g %g\n",
           cs.a_sw, cs.b_sw, cs.a_mn, cs.b_mn, cs.a_sbo, cs.a_lbo, cs.b_sbo, cs.b_lbo, cudaGetErrorString(e), bad,
           M * N, maxerr, out[0], out[1], out[2], out[3], ref[0], ref[1], ref[2], ref[3]);
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
