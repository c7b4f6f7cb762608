// Microbenchmarks backing the persistent-kernel design:
// grid-wide barrier cost, dependent L2/HBM load latency, globaltimer
// resolution.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb microbench.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>

namespace cg = cooperative_groups;

__device__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__global__ void k_barrier(int iters, unsigned long long* out) {
  cg::grid_group g = cg::this_grid();
  unsigned long long t0 = gt();
  for (int i = 0; i < iters; ++i) g.sync();
  unsigned long long t1 = gt();
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = t1 - t0;
}

// pointer chase: dependent loads
__global__ void k_chase(const unsigned* next, int steps, unsigned long long* out, unsigned* sink) {
  unsigned p = 0;
  unsigned long long t0 = gt();
  long long c0 = clock64();
  for (int i = 0; i < steps; ++i) p = __ldcg(next + p);
  long long c1 = clock64();
  unsigned long long t1 = gt();
  out[0] = t1 - t0;
  out[1] = c1 - c0;
  *sink = p;
}

__global__ void k_timer(unsigned long long* out) {
  unsigned long long a = gt(), b = a;
  int n = 0;
  while (n < 20) {
    unsigned long long c = gt();
    if (c != b) { out[n++] = c - b; b = c; }
  }
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 64 * 8);
  unsigned long long h[64];
  int dev = 0, nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  for (int bps : {1, 2}) {
    int grid = nsm * bps, iters = 2000;
    void* args[] = {&iters, &d};
    cudaLaunchCooperativeKernel((void*)k_barrier, grid, 256, args, 0, 0);
    cudaLaunchCooperativeKernel((void*)k_barrier, grid, 256, args, 0, 0);
    cudaDeviceSynchronize();
    cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
    printf("grid.sync: %d CTAs x 256 threads: %.3f us per barrier (%s)\n", grid,
           h[0] / 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
  }
  for (size_t mb : {4, 64, 1024}) {
    size_t n = mb * 1024 * 1024 / 4;
    unsigned* hp = new unsigned[n];
    // random cyclic permutation with a large stride
    size_t stride = 4099 * 16 + 7;
    for (size_t i = 0; i < n; ++i) hp[i] = (unsigned)((i + stride) % n);
    unsigned* dp;
    unsigned* sink;
    cudaMalloc(&dp, n * 4);
    cudaMalloc(&sink, 4);
    cudaMemcpy(dp, hp, n * 4, cudaMemcpyHostToDevice);
    int steps = 20000;
    k_chase<<<1, 1>>>(dp, 1000, d, sink);
    k_chase<<<1, 1>>>(dp, steps, d, sink);
    cudaDeviceSynchronize();
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("dependent __ldcg, %zu MiB footprint: %.1f ns, %.0f cycles per load\n", mb,
           h[0] / (double)steps, h[1] / (double)steps);
    cudaFree(dp);
    cudaFree(sink);
    delete[] hp;
  }
  k_timer<<<1, 1>>>(d);
  cudaDeviceSynchronize();
  cudaMemcpy(h, d, 20 * 8, cudaMemcpyDeviceToHost);
  printf("globaltimer increments (ns):");
  for (int i = 0; i < 20; ++i) printf(" %llu", h[i]);
  printf("\n");
  return 0;
}
