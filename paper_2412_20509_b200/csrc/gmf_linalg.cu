// Level 3: row-reduction primitives of the (A)+(B1) identifiability
// projection (identify.py:29-110).  The O(n d^2) work -- Gram matrices,
// design cross products, and applying small transforms to every row -- runs
// here; only d x d / p x p factorizations happen on the host, as in the
// reference's d x d SVD (identify.py:40-45).
#include "gmf_common.cuh"

namespace gmf {

constexpr int kCrossCtas = kSMs;
constexpr int kCrossRows = 64;

template <typename T>
__global__ void __launch_bounds__(kThreads)
k_cross(int64_t rows, const T* __restrict__ A, int64_t lda, int a0, int a, const T* __restrict__ B,
        int64_t ldb, int b0, int b, int tr, double* part, unsigned int* ticket, double* out) {
  extern __shared__ double sm[];
  double* As = sm;                       // [tr][a]  (tr <= kCrossRows rows per tile)
  double* Bs = sm + tr * a;              // [tr][b]
  const int nout = a * b;
  const int64_t per = (rows + gridDim.x - 1) / gridDim.x;
  const int64_t lo = blockIdx.x * per;
  const int64_t hi = lo + per < rows ? lo + per : rows;
  double acc[16];
  #pragma unroll
  for (int k = 0; k < 16; ++k) acc[k] = 0.0;
  for (int64_t r0 = lo; r0 < hi; r0 += tr) {
    const int nr = (int)(hi - r0 < tr ? hi - r0 : tr);
    __syncthreads();
    for (int e = threadIdx.x; e < nr * a; e += kThreads)
      As[e] = (double)A[(r0 + e / a) * lda + a0 + e % a];
    for (int e = threadIdx.x; e < nr * b; e += kThreads)
      Bs[e] = (double)B[(r0 + e / b) * ldb + b0 + e % b];
    __syncthreads();
    #pragma unroll
    for (int k = 0; k < 16; ++k) {
      const int o = threadIdx.x + k * kThreads;
      if (o < nout) {
        const int ia = o / b, ib = o % b;
        double s = acc[k];
        for (int r = 0; r < nr; ++r) s += As[r * a + ia] * Bs[r * b + ib];
        acc[k] = s;
      }
    }
  }
  #pragma unroll
  for (int k = 0; k < 16; ++k) {
    const int o = threadIdx.x + k * kThreads;
    if (o < nout) part[(int64_t)blockIdx.x * nout + o] = acc[k];
  }
  if (last_block_ticket(ticket, gridDim.x)) {
    for (int o = threadIdx.x; o < nout; o += kThreads) {
      double s = 0.0;
      for (unsigned int g = 0; g < gridDim.x; ++g) s += __ldcg(part + (int64_t)g * nout + o);
      out[o] = s;
    }
    if (threadIdx.x == 0) *ticket = 0u;
  }
}

constexpr int kAffThreads = 128;

template <typename T>
__global__ void __launch_bounds__(kAffThreads)
k_affine(int64_t rows, T* Y, int64_t ldy, int y0, int c, double beta, const T* A, int64_t lda,
         int a0, int a, const double* __restrict__ M) {
  extern __shared__ double sm[];
  double* Ms = sm;                                  // [a][c]
  double* rb = sm + a * c + threadIdx.x * (a + c);  // this thread's A row, then outputs
  for (int e = threadIdx.x; e < a * c; e += kAffThreads) Ms[e] = M[e];
  __syncthreads();
  const int64_t r = blockIdx.x * (int64_t)kAffThreads + threadIdx.x;
  if (r >= rows) return;
  for (int k = 0; k < a; ++k) rb[k] = (double)A[r * lda + a0 + k];
  double* ob = rb + a;
  for (int jc = 0; jc < c; ++jc) {
    double s = beta == 0.0 ? 0.0 : beta * (double)Y[r * ldy + y0 + jc];
    for (int k = 0; k < a; ++k) s += rb[k] * Ms[k * c + jc];
    ob[jc] = s;
  }
  for (int jc = 0; jc < c; ++jc) Y[r * ldy + y0 + jc] = (T)ob[jc];
}

}  // namespace gmf

using namespace gmf;

extern "C" {

int64_t gmf_cross_work_bytes(int32_t a, int32_t b) {
  return (int64_t)kCrossCtas * a * b * 8 + 256;
}

int gmf_cross_rows(int dtype, int64_t rows, const void* A, int64_t lda, int32_t a0, int32_t a,
                   const void* B, int64_t ldb, int32_t b0, int32_t b, double* out, void* work,
                   void* stream) {
  if (a < 1 || b < 1 || a * b > 16 * kThreads) { set_error("cross_rows: a*b out of range"); return GMF_ERR_UNSUPPORTED; }
  if (dtype != GMF_F32 && dtype != GMF_F64) { set_error("bad dtype"); return GMF_ERR_CONFIG; }
  cudaStream_t st = (cudaStream_t)stream;
  double* part = (double*)work;
  unsigned int* ticket = (unsigned int*)((char*)work + (int64_t)kCrossCtas * a * b * 8);
  GMF_CUDA(cudaMemsetAsync(ticket, 0, 4, st));
  // rows per shared-memory tile: up to kCrossRows within the 48 KB default
  int tr = (48 * 1024) / ((a + b) * 8);
  tr = tr > kCrossRows ? kCrossRows : tr;
  if (tr < 1) { set_error("cross_rows: too wide"); return GMF_ERR_UNSUPPORTED; }
  const size_t sm = (size_t)tr * (a + b) * 8;
  if (dtype == GMF_F64)
    k_cross<double><<<kCrossCtas, kThreads, sm, st>>>(rows, (const double*)A, lda, a0, a,
        (const double*)B, ldb, b0, b, tr, part, ticket, out);
  else
    k_cross<float><<<kCrossCtas, kThreads, sm, st>>>(rows, (const float*)A, lda, a0, a,
        (const float*)B, ldb, b0, b, tr, part, ticket, out);
  GMF_LAUNCH_CHECK("k_cross");
  return GMF_OK;
}

int gmf_rows_affine(int dtype, int64_t rows, void* Y, int64_t ldy, int32_t y0, int32_t c,
                    double beta, const void* A, int64_t lda, int32_t a0, int32_t a,
                    const double* M, void* stream) {
  if (rows <= 0 || c <= 0) return GMF_OK;
  if (a < 0 || a > 64 || c > 64) { set_error("rows_affine: a, c must be <= 64"); return GMF_ERR_UNSUPPORTED; }
  if (dtype != GMF_F32 && dtype != GMF_F64) { set_error("bad dtype"); return GMF_ERR_CONFIG; }
  cudaStream_t st = (cudaStream_t)stream;
  const size_t sm = (size_t)(a * c + kAffThreads * (a + c)) * 8;
  const int grid = (int)((rows + kAffThreads - 1) / kAffThreads);
  if (dtype == GMF_F64) {
    GMF_CUDA(cudaFuncSetAttribute(k_affine<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    k_affine<double><<<grid, kAffThreads, sm, st>>>(rows, (double*)Y, ldy, y0, c, beta,
        (const double*)A, lda, a0, a, M);
  } else {
    GMF_CUDA(cudaFuncSetAttribute(k_affine<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    k_affine<float><<<grid, kAffThreads, sm, st>>>(rows, (float*)Y, ldy, y0, c, beta,
        (const float*)A, lda, a0, a, M);
  }
  GMF_LAUNCH_CHECK("k_affine");
  return GMF_OK;
}

}  // extern "C"
