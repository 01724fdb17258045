// norm.cu -- iterated mode epilogue (BJ.configs[5]): nu = ||y||_2 from a fixed
// chunking of the rows (partials in chunk order, every rank sums the gathered
// partials in rank order => identical nu everywhere), then x = y / nu.
#include "common.cuh"
#include "internal.h"

namespace spmv {

__global__ void __launch_bounds__(kNT) norm_partials_kernel(const double* __restrict__ y, int64_t m,
                                                            double* __restrict__ partials) {
  const int64_t b = blockIdx.x;
  const int64_t r0 = b * m / kNormPartials, r1 = (b + 1) * m / kNormPartials;
  double a0 = 0.0, a1 = 0.0;
  int64_t i = r0 + threadIdx.x;
  for (; i + kNT < r1; i += 2 * kNT) {
    const double v0 = ld_stream(y + i), v1 = ld_stream(y + i + kNT);
    a0 = fma(v0, v0, a0);
    a1 = fma(v1, v1, a1);
  }
  if (i < r1) {
    const double v = ld_stream(y + i);
    a0 = fma(v, v, a0);
  }
  const double t = warp_sum(a0 + a1);
  __shared__ double ws[kNT / 32];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = t;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < kNT / 32; ++w) s += ws[w];
    partials[b] = s;
  }
}

__global__ void __launch_bounds__(kNT) normalize_kernel(const double* __restrict__ y, int64_t m,
                                                        const double* __restrict__ partials, int count,
                                                        double* __restrict__ x_out, double* __restrict__ nu_dev) {
  __shared__ double nu_s;
  if (threadIdx.x == 0) {
    double ss = 0.0;
    for (int q = 0; q < count; ++q) ss += partials[q];
    nu_s = sqrt(ss);
    if (blockIdx.x == 0 && nu_dev) *nu_dev = nu_s;
  }
  __syncthreads();
  const double nu = nu_s;
  const int64_t stride = (int64_t)gridDim.x * kNT;
  for (int64_t i = (int64_t)blockIdx.x * kNT + threadIdx.x; i < m; i += stride) x_out[i] = y[i] / nu;
}

int launch_norm_partials(const double* y, int64_t m, double* partials, cudaStream_t s) {
  norm_partials_kernel<<<kNormPartials, kNT, 0, s>>>(y, m, partials);
  return 1;
}

int launch_normalize(const double* y, int64_t m, const double* partials, int count, double* x_out, double* nu_dev,
                     cudaStream_t s) {
  int64_t grid = (m + kNT - 1) / kNT;
  if (grid > 148 * 8) grid = 148 * 8;
  if (grid < 1) grid = 1;
  normalize_kernel<<<(int)grid, kNT, 0, s>>>(y, m, partials, count, x_out, nu_dev);
  return 1;
}

}  // namespace spmv
