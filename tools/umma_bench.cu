// tcgen05 kind::f16 (bf16) MMA issue/throughput microbenchmark: one CTA per
// SM (or two) issues R back-to-back MMAs of shape M x N x 16 from shared
// memory (no-swizzle K-major operands, or the MN-major A used by GEMM3) into
// TMEM and waits for the commit; reports cycles per MMA.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o umma_bench umma_bench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46) | ((uint64_t)layout << 61);
}
__device__ __forceinline__ uint32_t idesc(int M, int N, int amn, int bmn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)amn << 15) | ((uint32_t)bmn << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

struct Cfg { int N, amn, swz, reps, ncols; };

__global__ void k_bench(Cfg c, long long* out) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x;
  for (int e = tid; e < 96 * 1024 / 4; e += blockDim.x) reinterpret_cast<uint32_t*>(smem)[e] = 0x3f803f80u;
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tmem_base;
  if (tid == 0) {
    const uint32_t sa = smem_u32(smem), sbm = smem_u32(smem + 48 * 1024);
    // K-major A: M=128 rows, LBO 128 (next K core), SBO 2048 (16 K cores per row group)
    // MN-major A: MN chunks +128, K groups +2048.  SW128 K-major: SBO 1024
    const uint64_t da = c.swz ? sdesc(sa, 16, 1024, 2) : (c.amn ? sdesc(sa, 2048, 128, 0) : sdesc(sa, 128, 2048, 0));
    const uint64_t db = c.swz ? sdesc(sbm, 16, 1024, 2) : sdesc(sbm, 128, 2048, 0);
    const uint32_t id = idesc(128, c.N, c.amn, 0);
    const long long t0 = clock64();
    #pragma unroll 8
    for (int r = 0; r < c.reps; ++r) {
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tm),
                   "l"(da), "l"(db), "r"(id), "r"(1));
    }
    const long long t1 = clock64();
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    uint32_t done = 0;
    while (!done)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
                   : "=r"(done) : "r"(smem_u32(&bar)));
    const long long t2 = clock64();
    out[2 * blockIdx.x] = t1 - t0;
    out[2 * blockIdx.x + 1] = t2 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tm));
}

int main() {
  long long* d;
  cudaMalloc(&d, 2 * 296 * sizeof(long long));
  cudaFuncSetAttribute(k_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  Cfg cases[] = {
      {16, 0, 0, 512, 128}, {32, 0, 0, 512, 128}, {64, 0, 0, 512, 128}, {128, 0, 0, 512, 128},
      {16, 1, 0, 512, 128}, {32, 1, 0, 512, 128}, {64, 1, 0, 512, 128},
      {16, 0, 1, 512, 128}, {64, 0, 1, 512, 128}, {128, 0, 1, 512, 128},
  };
  for (int grid : {148, 296}) {
    for (auto& c : cases) {
      k_bench<<<grid, 128, 100 * 1024>>>(c, d);   // warm
      k_bench<<<grid, 128, 100 * 1024>>>(c, d);
      cudaError_t e = cudaDeviceSynchronize();
      long long h[2 * 296];
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      double issue = 0, total = 0;
      for (int b = 0; b < grid; ++b) { issue += h[2 * b]; total += h[2 * b + 1]; }
      printf("grid %3d N=%3d A %s%s: issue %.1f cyc/mma, complete %.1f cyc/mma  (%s)\n", grid, c.N,
             c.amn ? "MN-major" : "K-major", c.swz ? " SW128" : "", issue / grid / c.reps,
             total / grid / c.reps, cudaGetErrorString(e));
    }
  }
  return 0;
}
