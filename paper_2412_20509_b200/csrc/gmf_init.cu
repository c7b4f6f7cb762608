// OLS-SVD initialization on the GPU (gmfkit/initialization.py:143-169,
// randomized_svd 62-82) without materialising the n x m residual.
//
// With a fully observed count matrix Y and the log link, the transformed
// response is log(Y + eps) = log(eps) 1 1' + S, where S is as sparse as Y
// (s_ij = log(y_ij + eps) - log(eps), zero where y_ij = 0).  Every product
// the initialization needs (X' Y_eps, Z' Y_eps', and the randomized range
// finder's A P and A' Q with A = Y_eps - X B' - Gamma Z') is therefore a
// sparse product with S plus rank-(1+p+q) corrections done on the host side
// of the ABI.  The kernels here are the sparse parts and the NB moment pass:
//
//   gmf_csr_spmm    out = S P over a CSR (or, given the CSC, S' Q): warp per
//                   (row, nonzero segment), lanes over P's columns; segment
//                   partials summed in fixed order (deterministic).
//   gmf_init_moments  sums over ALL n x m entries of mu0 = exp(clip(eta0)),
//                   eta0 = X B' + Gamma Z': [sum mu0^2, sum ((y - mu0)^2 - mu0)]
//                   for _nb_shape_moment (initialization.py:93-100); zeros
//                   handled over the dense grid, nonzeros corrected from CSR.
#include "gmf_common.cuh"

namespace gmf {

constexpr int kSeg = 2048;          // nonzeros per warp task
constexpr int kInitThreads = 256;

// partial[s][i][c] (or out[i][c] when nseg == 1) = sum over row i's nonzeros
// in segment s of s(val) * P[col][c]
__global__ void __launch_bounds__(kInitThreads) k_spmm(int64_t nrows, const int64_t* __restrict__ ptr,
                                                       const int32_t* __restrict__ col,
                                                       const int32_t* __restrict__ val, double eps,
                                                       const double* __restrict__ P, int r,
                                                       int64_t nseg, double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t task = ((int64_t)blockIdx.x * kInitThreads + threadIdx.x) >> 5;
  if (task >= nrows * nseg) return;
  const int64_t i = task / nseg, s = task - i * nseg;
  const int64_t lo = ptr[i] + s * kSeg;
  const int64_t hi = min(ptr[i + 1], lo + kSeg);
  const double leps = log(eps);
  for (int c0 = 0; c0 < r; c0 += 32) {
    const int c = c0 + lane;
    double acc = 0.0;
    for (int64_t k0 = lo; k0 < hi; k0 += 32) {
      const int64_t k = k0 + lane;
      int32_t j = 0;
      double sv = 0.0;
      if (k < hi) {
        j = col[k];
        sv = log((double)val[k] + eps) - leps;
      }
      const int cnt = (int)min((int64_t)32, hi - k0);
      for (int t = 0; t < cnt; ++t) {
        const int32_t jt = __shfl_sync(0xffffffffu, j, t);
        const double st = __shfl_sync(0xffffffffu, sv, t);
        if (c < r) acc = fma(st, P[(int64_t)jt * r + c], acc);
      }
    }
    if (c < r) out[(s * nrows + i) * r + c] = acc;
  }
}

__global__ void __launch_bounds__(kInitThreads) k_seg_sum(int64_t total, int64_t nseg,
                                                          const double* __restrict__ part,
                                                          double* __restrict__ out) {
  for (int64_t g = (int64_t)blockIdx.x * kInitThreads + threadIdx.x; g < total;
       g += (int64_t)gridDim.x * kInitThreads) {
    double s = 0.0;
    for (int64_t t = 0; t < nseg; ++t) s += part[t * total + g];
    out[g] = s;
  }
}

// eta0_ij = x_i . b_j + gamma_i . z_j, clipped to [lo, hi] (initialization.py:217-225)
GMF_D double eta0_at(int64_t i, int64_t j, const double* x, const double* b, int p,
                     const double* g, const double* z, int q, double lo, double hi) {
  double e = 0.0;
  for (int k = 0; k < p; ++k) e += x[i * p + k] * b[j * p + k];
  for (int k = 0; k < q; ++k) e += g[i * q + k] * z[j * q + k];
  return fmin(fmax(e, lo), hi);
}

__global__ void __launch_bounds__(kInitThreads) k_moments(int64_t n, int64_t m,
                                                          const int64_t* __restrict__ ptr,
                                                          const int32_t* __restrict__ col,
                                                          const int32_t* __restrict__ val,
                                                          const double* x, const double* b, int p,
                                                          const double* g, const double* z, int q,
                                                          double lo, double hi, double* part,
                                                          unsigned int* ticket, double* out) {
  __shared__ double scr[kInitThreads / 32];
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * kInitThreads + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * kInitThreads) >> 5;
  double num = 0.0, den = 0.0;
  for (int64_t i = gw; i < n; i += nw) {
    // every entry as a zero: mu^2 and (0 - mu)^2 - mu
    for (int64_t j = lane; j < m; j += 32) {
      const double mu = exp(eta0_at(i, j, x, b, p, g, z, q, lo, hi));
      num += mu * mu;
      den += mu * mu - mu;
    }
    // nonzeros: (y - mu)^2 - mu minus the zero term = y^2 - 2 y mu
    for (int64_t k = ptr[i] + lane; k < ptr[i + 1]; k += 32) {
      const double mu = exp(eta0_at(i, col[k], x, b, p, g, z, q, lo, hi));
      const double y = (double)val[k];
      den += y * y - 2.0 * y * mu;
    }
  }
  num = block_sum<kInitThreads>(num, scr);
  if (threadIdx.x == 0) part[blockIdx.x] = num;
  den = block_sum<kInitThreads>(den, scr);
  if (threadIdx.x == 0) part[gridDim.x + blockIdx.x] = den;
  if (last_block_ticket(ticket, gridDim.x)) {
    if (threadIdx.x < 2) {
      double t = 0.0;
      for (unsigned int k = 0; k < gridDim.x; ++k) t += ld_cg(part + threadIdx.x * gridDim.x + k);
      out[threadIdx.x] = t;
    }
    __syncthreads();
    if (threadIdx.x == 0) *ticket = 0u;
  }
}

constexpr int kMomentBlocks = 4 * kSMs;

}  // namespace gmf

using namespace gmf;

extern "C" {

int64_t gmf_spmm_work_bytes(int64_t nrows, int64_t max_row_nnz, int32_t r) {
  const int64_t nseg = max_row_nnz > kSeg ? (max_row_nnz + kSeg - 1) / kSeg : 1;
  return nseg > 1 ? nseg * nrows * r * 8 : 0;
}

int gmf_csr_spmm(int64_t nrows, const int64_t* ptr, const int32_t* col, const int32_t* val,
                 int64_t max_row_nnz, double eps, const double* P, int32_t r, double* out,
                 void* work, void* stream) {
  if (nrows < 0 || r < 0 || !(eps > 0.0)) { set_error("spmm: bad sizes or eps"); return GMF_ERR_CONFIG; }
  if (nrows == 0 || r == 0) return GMF_OK;
  if (!ptr || !out || (max_row_nnz > 0 && (!col || !val || !P))) {
    set_error("spmm: null pointer");
    return GMF_ERR_CONFIG;
  }
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t nseg = max_row_nnz > kSeg ? (max_row_nnz + kSeg - 1) / kSeg : 1;
  if (nseg > 1 && !work) { set_error("spmm: long rows need work (gmf_spmm_work_bytes)"); return GMF_ERR_CONFIG; }
  const int64_t warps = nrows * nseg;
  const int64_t blocks = (warps * 32 + kInitThreads - 1) / kInitThreads;
  double* dst = nseg > 1 ? (double*)work : out;
  k_spmm<<<(unsigned)blocks, kInitThreads, 0, st>>>(nrows, ptr, col, val, eps, P, r, nseg, dst);
  GMF_LAUNCH_CHECK("k_spmm");
  if (nseg > 1) {
    const int64_t total = nrows * r;
    int64_t b = (total + kInitThreads - 1) / kInitThreads;
    if (b > 8 * kSMs) b = 8 * kSMs;
    k_seg_sum<<<(unsigned)b, kInitThreads, 0, st>>>(total, nseg, dst, out);
    GMF_LAUNCH_CHECK("k_seg_sum");
  }
  return GMF_OK;
}

int64_t gmf_moments_work_bytes(void) { return (int64_t)2 * kMomentBlocks * 8 + 64; }

int gmf_init_moments(int64_t n, int64_t m, const int64_t* ptr, const int32_t* col,
                     const int32_t* val, const double* x, const double* b, int32_t p,
                     const double* gamma, const double* z, int32_t q, double eta_lo,
                     double eta_hi, double* out2, void* work, void* stream) {
  if (n <= 0 || m <= 0 || p < 0 || q < 0) { set_error("moments: bad sizes"); return GMF_ERR_CONFIG; }
  if (!ptr || !out2 || !work) { set_error("moments: null pointer"); return GMF_ERR_CONFIG; }
  cudaStream_t st = (cudaStream_t)stream;
  double* part = (double*)work;
  unsigned int* ticket = (unsigned int*)((char*)work + (int64_t)2 * kMomentBlocks * 8);
  GMF_CUDA(cudaMemsetAsync(ticket, 0, sizeof(unsigned int), st));
  k_moments<<<kMomentBlocks, kInitThreads, 0, st>>>(n, m, ptr, col, val, x, b, p, gamma, z, q,
                                                     eta_lo, eta_hi, part, ticket, out2);
  GMF_LAUNCH_CHECK("k_moments");
  return GMF_OK;
}

}  // extern "C"
