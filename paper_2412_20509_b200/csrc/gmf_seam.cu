// Level 1: the elementwise backend seam of gmfkit/kernels (mean_of_eta,
// derivs_from_mu, deviance_from_mu) as sm_100a kernels, plus the error and
// version plumbing of the C ABI.
#include <stdarg.h>
#include <stdio.h>

#include "gmf_common.cuh"

namespace gmf {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int cuda_fail(cudaError_t e, const char* where) {
  set_error("CUDA error %s (%s) at %s", cudaGetErrorName(e), cudaGetErrorString(e), where);
  return GMF_ERR_CUDA;
}

// kernels/_ref.py:21-32
template <typename T>
__global__ void k_mean_of_eta(int lcode, const T* __restrict__ eta, T* __restrict__ mu, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    mu[i] = mean_of_eta_t<T>(lcode, eta[i]);
}

GMF_D double variance_of(int fcode, double mu, double alpha) {  // _core.pyx:28-40
  switch (fcode) {
    case GMF_GAUSSIAN: return 1.0;
    case GMF_GAMMA: return mu * mu;
    case GMF_INV_GAUSSIAN: return mu * mu * mu;
    case GMF_POISSON: return mu;
    case GMF_BERNOULLI: return mu * (1.0 - mu);
    default: return mu * (1.0 + mu / alpha);
  }
}

GMF_D double link_d1(int lcode, double mu) {  // _core.pyx:43-53
  switch (lcode) {
    case GMF_IDENTITY: return 1.0;
    case GMF_LOG: return 1.0 / mu;
    case GMF_LOGIT: return 1.0 / (mu * (1.0 - mu));
    case GMF_INVERSE: return -1.0 / (mu * mu);
    default: return -2.0 / (mu * mu * mu);
  }
}

// kernels/_core.pyx:58-111 (canonical shortcuts 79-103, generic 104-110)
template <typename T>
__global__ void k_derivs(int fcode, int lcode, const T* __restrict__ y, const T* __restrict__ mu,
                         const T* __restrict__ w, int64_t n, double phi, double alpha,
                         T* __restrict__ dotd, T* __restrict__ ddotd) {
  const bool canon = (fcode == GMF_POISSON && lcode == GMF_LOG) ||
                     (fcode == GMF_BERNOULLI && lcode == GMF_LOGIT) ||
                     (fcode == GMF_GAUSSIAN && lcode == GMF_IDENTITY) ||
                     (fcode == GMF_GAMMA && lcode == GMF_INVERSE) ||
                     (fcode == GMF_INV_GAUSSIAN && lcode == GMF_INVERSE_SQUARED) ||
                     (fcode == GMF_NEG_BINOMIAL && lcode == GMF_LOG);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double m = (double)mu[i];
    const double wi = w ? (double)w[i] : 1.0;
    const double r = (double)y[i] - m;
    double a, b;
    if (canon) {
      switch (fcode) {
        case GMF_POISSON: a = -wi * r / phi; b = wi * m / phi; break;
        case GMF_BERNOULLI: a = -wi * r / phi; b = wi * m * (1.0 - m) / phi; break;
        case GMF_GAUSSIAN: a = -wi * r / phi; b = wi / phi; break;
        case GMF_GAMMA: a = wi * r / phi; b = wi * m * m / phi; break;
        case GMF_INV_GAUSSIAN: a = wi * r / (2.0 * phi); b = wi * m * m * m / (4.0 * phi); break;
        default: {
          const double den = 1.0 + m / alpha;
          a = -wi * r / (phi * den);
          b = wi * m / (phi * den);
        }
      }
    } else {
      const double nu = variance_of(fcode, m, alpha);
      const double g1 = link_d1(lcode, m);
      a = -wi * r / (phi * nu * g1);
      b = wi / (phi * nu * g1 * g1);
    }
    dotd[i] = (T)a;
    ddotd[i] = (T)b;
  }
}

constexpr int kSeamBlocks = 2 * kSMs;

template <typename T>
__global__ void k_deviance(int fcode, const T* __restrict__ y, const T* __restrict__ mu,
                           const T* __restrict__ w, int64_t n, double alpha, double* part,
                           unsigned int* ticket, double* out) {
  __shared__ double scratch[kThreads / 32];
  double s = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double wi = w ? (double)w[i] : 1.0;
    s += wi * unit_deviance(fcode, (double)y[i], (double)mu[i], alpha);
  }
  s = block_sum<kThreads>(s, scratch);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
  if (last_block_ticket(ticket, gridDim.x)) {
    if (threadIdx.x == 0) {
      double tot = 0.0;
      for (unsigned int b = 0; b < gridDim.x; ++b) tot += ld_cg(part + b);
      *out = tot;
      *ticket = 0u;
    }
  }
}

// metrics.py:35-55 (rel_log_rmse, rel_deviance) on device arrays: out =
// [sum D(y, mu), sum D(y, ybar), sum log^2((1+y)/(1+mu)), sum log^2((1+y)/(1+ybar))]
template <typename T>
__global__ void k_score_pairs(int fcode, const T* __restrict__ y, const T* __restrict__ mu,
                              int64_t n, double ybar, double alpha, double* part,
                              unsigned int* ticket, double* out) {
  __shared__ double scratch[kThreads / 32];
  double s[4] = {0.0, 0.0, 0.0, 0.0};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double yi = (double)y[i], mi = (double)mu[i];
    s[0] += unit_deviance(fcode, yi, mi, alpha);
    s[1] += unit_deviance(fcode, yi, ybar, alpha);
    const double a = log((1.0 + yi) / (1.0 + mi)), b = log((1.0 + yi) / (1.0 + ybar));
    s[2] += a * a;
    s[3] += b * b;
  }
  for (int c = 0; c < 4; ++c) {
    const double t = block_sum<kThreads>(s[c], scratch);
    if (threadIdx.x == 0) part[c * gridDim.x + blockIdx.x] = t;
  }
  if (last_block_ticket(ticket, gridDim.x)) {
    if (threadIdx.x < 4) {
      double tot = 0.0;
      for (unsigned int b = 0; b < gridDim.x; ++b) tot += ld_cg(part + threadIdx.x * gridDim.x + b);
      out[threadIdx.x] = tot;
    }
    __syncthreads();
    if (threadIdx.x == 0) *ticket = 0u;
  }
}

static int blocks_for(int64_t n) {
  int64_t b = (n + kThreads - 1) / kThreads;
  if (b < 1) b = 1;
  if (b > 8 * kSMs) b = 8 * kSMs;
  return (int)b;
}

static bool dtype_ok(int dtype) {
  if (dtype == GMF_F32 || dtype == GMF_F64) return true;
  set_error("unknown dtype code %d", dtype);
  return false;
}

}  // namespace gmf

using namespace gmf;

extern "C" {

const char* gmf_last_error(void) { return g_err; }
const char* gmf_version(void) { return "gmf_asgd 0.1.0 sm_100a"; }

int gmf_mean_of_eta(int lcode, int dtype, const void* eta, void* mu, int64_t n, void* stream) {
  if (lcode < 0 || lcode > GMF_INVERSE_SQUARED) { set_error("unknown link code %d", lcode); return GMF_ERR_DOMAIN; }
  if (!dtype_ok(dtype)) return GMF_ERR_CONFIG;
  if (n <= 0) return GMF_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == GMF_F64)
    k_mean_of_eta<double><<<blocks_for(n), kThreads, 0, s>>>(lcode, (const double*)eta, (double*)mu, n);
  else
    k_mean_of_eta<float><<<blocks_for(n), kThreads, 0, s>>>(lcode, (const float*)eta, (float*)mu, n);
  GMF_LAUNCH_CHECK("gmf_mean_of_eta");
  return GMF_OK;
}

int gmf_derivs_from_mu(int fcode, int lcode, int dtype, const void* y, const void* mu,
                       const void* w, int64_t n, double phi, double alpha, void* dotd,
                       void* ddotd, void* stream) {
  if (fcode < 0 || fcode > GMF_NEG_BINOMIAL) { set_error("unknown family code %d", fcode); return GMF_ERR_DOMAIN; }
  if (lcode < 0 || lcode > GMF_INVERSE_SQUARED) { set_error("unknown link code %d", lcode); return GMF_ERR_DOMAIN; }
  if (!dtype_ok(dtype)) return GMF_ERR_CONFIG;
  if (n <= 0) return GMF_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == GMF_F64)
    k_derivs<double><<<blocks_for(n), kThreads, 0, s>>>(fcode, lcode, (const double*)y,
        (const double*)mu, (const double*)w, n, phi, alpha, (double*)dotd, (double*)ddotd);
  else
    k_derivs<float><<<blocks_for(n), kThreads, 0, s>>>(fcode, lcode, (const float*)y,
        (const float*)mu, (const float*)w, n, phi, alpha, (float*)dotd, (float*)ddotd);
  GMF_LAUNCH_CHECK("gmf_derivs_from_mu");
  return GMF_OK;
}

int64_t gmf_reduce_work_bytes(int64_t n) {
  (void)n;
  return (int64_t)kSeamBlocks * 8 + 64;
}

int gmf_deviance_from_mu(int fcode, int dtype, const void* y, const void* mu, const void* w,
                         int64_t n, double alpha, double* dev_sum, void* work, void* stream) {
  if (fcode < 0 || fcode > GMF_NEG_BINOMIAL) { set_error("unknown family code %d", fcode); return GMF_ERR_DOMAIN; }
  if (!dtype_ok(dtype)) return GMF_ERR_CONFIG;
  if (!work || !dev_sum) { set_error("deviance: null work/out"); return GMF_ERR_CONFIG; }
  cudaStream_t s = (cudaStream_t)stream;
  double* part = (double*)work;
  unsigned int* ticket = (unsigned int*)((char*)work + (int64_t)kSeamBlocks * 8);
  GMF_CUDA(cudaMemsetAsync(ticket, 0, sizeof(unsigned int), s));
  int nb = blocks_for(n);
  if (nb > kSeamBlocks) nb = kSeamBlocks;
  if (dtype == GMF_F64)
    k_deviance<double><<<nb, kThreads, 0, s>>>(fcode, (const double*)y, (const double*)mu,
        (const double*)w, n, alpha, part, ticket, dev_sum);
  else
    k_deviance<float><<<nb, kThreads, 0, s>>>(fcode, (const float*)y, (const float*)mu,
        (const float*)w, n, alpha, part, ticket, dev_sum);
  GMF_LAUNCH_CHECK("gmf_deviance_from_mu");
  return GMF_OK;
}

int64_t gmf_score_work_bytes(void) { return (int64_t)4 * kSeamBlocks * 8 + 64; }

int gmf_score_pairs(int fcode, int dtype, const void* y, const void* mu, int64_t n, double ybar,
                    double alpha, double* sums4, void* work, void* stream) {
  if (fcode < 0 || fcode > GMF_NEG_BINOMIAL) { set_error("unknown family code %d", fcode); return GMF_ERR_DOMAIN; }
  if (!dtype_ok(dtype)) return GMF_ERR_CONFIG;
  if (!work || !sums4) { set_error("score_pairs: null work/out"); return GMF_ERR_CONFIG; }
  cudaStream_t s = (cudaStream_t)stream;
  double* part = (double*)work;
  unsigned int* ticket = (unsigned int*)((char*)work + (int64_t)4 * kSeamBlocks * 8);
  GMF_CUDA(cudaMemsetAsync(ticket, 0, sizeof(unsigned int), s));
  int nb = blocks_for(n);
  if (nb > kSeamBlocks) nb = kSeamBlocks;
  if (dtype == GMF_F64)
    k_score_pairs<double><<<nb, kThreads, 0, s>>>(fcode, (const double*)y, (const double*)mu, n,
                                                  ybar, alpha, part, ticket, sums4);
  else
    k_score_pairs<float><<<nb, kThreads, 0, s>>>(fcode, (const float*)y, (const float*)mu, n,
                                                 ybar, alpha, part, ticket, sums4);
  GMF_LAUNCH_CHECK("gmf_score_pairs");
  return GMF_OK;
}

}  // extern "C"
