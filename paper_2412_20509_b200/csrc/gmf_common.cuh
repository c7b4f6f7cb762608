// Shared device helpers for the aSGD hot path (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <math.h>

#include "gmf_asgd.h"

#define GMF_HD __host__ __device__ __forceinline__
#define GMF_D __device__ __forceinline__

namespace gmf {

void set_error(const char* fmt, ...);
int cuda_fail(cudaError_t e, const char* where);

#define GMF_CUDA(call)                                                   \
  do {                                                                   \
    cudaError_t e_ = (call);                                             \
    if (e_ != cudaSuccess) return ::gmf::cuda_fail(e_, #call);           \
  } while (0)

#define GMF_LAUNCH_CHECK(where)                                          \
  do {                                                                   \
    cudaError_t e_ = cudaGetLastError();                                 \
    if (e_ != cudaSuccess) return ::gmf::cuda_fail(e_, where);           \
  } while (0)

constexpr int kThreads = 256;
constexpr int kSMs = 148;

// ---------------------------------------------------------------------------
// fast exp: fp32 via ex2.approx (MUFU), fp64 via libdevice exp (1 ulp)
// ---------------------------------------------------------------------------
GMF_D float exp_t(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x * 1.4426950408889634f));
  return y;
}
GMF_D double exp_t(double x) { return exp(x); }

GMF_D float rcp_t(float x) { return __frcp_rn(x); }
GMF_D double rcp_t(double x) { return 1.0 / x; }

// ---------------------------------------------------------------------------
// deterministic block reduction of doubles (fixed tree order)
// ---------------------------------------------------------------------------
template <int NT>
GMF_D double block_sum(double v, double* scratch /* >= NT/32 */) {
  #pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) scratch[wid] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0) {
    #pragma unroll
    for (int w = 0; w < NT / 32; ++w) s += scratch[w];
  }
  return s;   // valid in thread 0
}

// "last CTA done" ticket: returns true in every thread of the last CTA to
// arrive; that CTA then reads every other CTA's published partials.
GMF_D bool last_block_ticket(unsigned int* counter, unsigned int expected) {
  __shared__ bool is_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int prev = atomicAdd(counter, 1u);
    is_last = (prev == expected - 1);
  }
  __syncthreads();
  if (is_last) __threadfence();
  return is_last;
}

GMF_D double ld_cg(const double* p) { return __ldcg(p); }

// ---------------------------------------------------------------------------
// per-entry family algebra (gmfkit/kernels/_ref.py, _core.pyx)
// ---------------------------------------------------------------------------
template <typename T>
GMF_D T mean_of_eta_t(int lcode, T eta) {
  switch (lcode) {
    case GMF_IDENTITY: return eta;
    case GMF_LOG: return (T)exp((double)eta) ;
    case GMF_LOGIT: return (T)(1.0 / (1.0 + exp(-(double)eta)));
    case GMF_INVERSE: return (T)(1.0 / (double)eta);
    default: return (T)(1.0 / sqrt((double)eta));
  }
}

// xlogy(y, y/mu) with 0 log 0 = 0 (scipy.special.xlogy)
GMF_HD double xlogy_ratio(double y, double mu) { return y == 0.0 ? 0.0 : y * log(y / mu); }

// fp32 unit deviance for the fp32 path's tracked objective (Poisson / NB);
// callers accumulate in fp64
GMF_D float unit_deviance_f(int fcode, float y, float mu, float alpha) {
  const float xl = y == 0.f ? 0.f : y * __logf(y / mu);
  if (fcode == GMF_POISSON) return 2.f * (xl - (y - mu));
  return 2.f * (xl - (y + alpha) * log1pf((y - mu) / (mu + alpha)));
}

GMF_HD double unit_deviance(int fcode, double y, double mu, double alpha) {
  switch (fcode) {
    case GMF_POISSON: return 2.0 * (xlogy_ratio(y, mu) - (y - mu));
    case GMF_NEG_BINOMIAL:
      return 2.0 * (xlogy_ratio(y, mu) - (y + alpha) * log1p((y - mu) / (mu + alpha)));
    case GMF_GAUSSIAN: return (y - mu) * (y - mu);
    case GMF_GAMMA: return 2.0 * ((y - mu) / mu - log(y / mu));
    case GMF_INV_GAUSSIAN: return (y - mu) * (y - mu) / (y * mu * mu);
    default: {  // Bernoulli, clipped mean (families.py:389-391)
      double m = fmin(fmax(mu, 1e-10), 1.0 - 1e-10);
      return 2.0 * (xlogy_ratio(y, m) + xlogy_ratio(1.0 - y, 1.0 - m));
    }
  }
}

}  // namespace gmf
