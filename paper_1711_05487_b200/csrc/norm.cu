// norm.cu -- iterated mode epilogue (BJ.configs[5]): nu = ||y||_2 from a fixed
// chunking of the rows (partials in chunk order, every rank sums the gathered
// partials in rank order => identical nu everywhere), then x = y / nu.
//
// Deferred normalisation (reading 25): the iterate runs on the
// unnormalised vectors yh_k = A yh_{k-1} (yh_{-1} = x_0), written by the SpMV
// straight into the other x replica, so no per-iteration x = y / nu pass:
// x_k = yh_{k-1} / ||yh_{k-1}|| and nu_k = ||A x_k|| = ||yh_k|| / ||yh_{k-1}||.
// The running norm lives on the device (nn[0]); when it leaves [2^-256,
// 2^256] the block is rescaled by an exact power of two (nn[1]), so the
// magnitudes never overflow and no rounding is added.
#include "common.cuh"
#include "internal.h"
#include "iterfuse.cuh"

namespace spmv {

template <bool SQ>
__global__ void __launch_bounds__(kNT) norm_partials_kernel(const double* __restrict__ y, int64_t m,
                                                            double* __restrict__ partials) {
  pdl_trigger();  // the next kernel in the stream may launch (it waits before reading)
  pdl_wait();
  const int64_t b = blockIdx.x;
  const int64_t r0 = b * m / kNormPartials, r1 = (b + 1) * m / kNormPartials;
  // 8 independent accumulators per thread (8 loads in flight: with 2 the
  // 512-chunk pass over a C5 block was latency-bound), fixed combine order
  double a[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  int64_t i = r0 + threadIdx.x;
  for (; i + 7 * kNT < r1; i += 8 * kNT) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = __ldcg(y + i + u * kNT);  // written by the previous kernel: L2-coherent
#pragma unroll
    for (int u = 0; u < 8; ++u) a[u] = SQ ? fma(v[u], v[u], a[u]) : a[u] + v[u];
  }
#pragma unroll
  for (int u = 0; u < 8; ++u)
    if (i + u * kNT < r1) {
      const double v = __ldcg(y + i + u * kNT);
      a[u] = SQ ? fma(v, v, a[u]) : a[u] + v;
    }
  const double t = warp_sum(((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7])));
  __shared__ double ws[kNT / 32];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = t;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < kNT / 32; ++w) s += ws[w];
    partials[b] = s;
  }
}

// sum of partials[0..count) by one CTA in a fixed order (thread t: q = t,
// t+kNT, ... ascending; butterflies; warps ascending) -- identical on every
// rank; one thread walking the partials waited one L2 round trip per few
// partials (~30 us for 512, the iterated mode's largest overhead on C5)
__device__ __forceinline__ double block_sum_fixed(const double* __restrict__ partials, int count) {
  double a = 0.0;
  for (int q = threadIdx.x; q < count; q += kNT) a += __ldcg(partials + q);
  a = warp_sum(a);
  __shared__ double ws[kNT / 32];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = a;
  __syncthreads();
  double ss = 0.0;
  for (int w = 0; w < kNT / 32; ++w) ss += ws[w];
  return ss;
}

__global__ void __launch_bounds__(kNT) normalize_kernel(const double* __restrict__ y, int64_t m,
                                                        const double* __restrict__ partials, int count,
                                                        double* __restrict__ x_out, double* __restrict__ nu_dev) {
  __shared__ double nu_s;
  const double ss = block_sum_fixed(partials, count);
  if (threadIdx.x == 0) {
    nu_s = sqrt(ss);
    if (blockIdx.x == 0 && nu_dev) *nu_dev = nu_s;
  }
  __syncthreads();
  const double nu = nu_s;
  const int64_t stride = (int64_t)gridDim.x * kNT;
  for (int64_t i = (int64_t)blockIdx.x * kNT + threadIdx.x; i < m; i += stride) x_out[i] = y[i] / nu;
}

// the norm step on gathered partials, one CTA (norm_step_scalar in
// iterfuse.cuh): *nu_k = ||yh_k|| / nn[0] (||yh_k|| at k = 0), nn[0] =
// ||yh_k|| brought into [2^-256, 2^256] by an exact power of two, nn[1] =
// that pending factor -- the block itself is not touched: the next SpMV
// multiplies its output by nn[1] (or spmv_unit the final x)
__global__ void __launch_bounds__(kNT) norm_step_kernel(const double* __restrict__ partials, int count,
                                                        double* __restrict__ nn, double* __restrict__ nu_k) {
  pdl_trigger();  // the next kernel in the stream may launch (it waits before reading)
  pdl_wait();
  const double ss = block_sum_fixed(partials, count);
  if (threadIdx.x == 0) norm_step_scalar(ss, nn, nu_k);
}

// Non-fused variants' iteration epilogue: y *= s (the pending factor nn[1]
// of the previous step; nothing written when s is 1) and the kNormPartials
// fixed-chunk partials of y^2 -- one pass over y
__global__ void __launch_bounds__(kNT) scale_partials_kernel(double* __restrict__ y, int64_t m,
                                                             const double* __restrict__ nn,
                                                             double* __restrict__ partials) {
  pdl_trigger();
  pdl_wait();
  const double f0 = nn ? __ldcg(nn + 1) : 1.0;
  const double f = f0 != 0.0 ? f0 : 1.0;
  const int64_t b = blockIdx.x;
  const int64_t r0 = b * m / kNormPartials, r1 = (b + 1) * m / kNormPartials;
  double a = 0.0;
  for (int64_t i = r0 + threadIdx.x; i < r1; i += kNT) {
    double v = __ldcg(y + i);
    if (f != 1.0) {
      v *= f;
      y[i] = v;
    }
    a = fma(v, v, a);
  }
  const double t = warp_sum(a);
  __shared__ double ws[kNT / 32];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = t;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < kNT / 32; ++w) s += ws[w];
    partials[b] = s;
  }
}

// x_out = yh * nn[1] / nn[0] (the pending factor applied, exact)
__global__ void __launch_bounds__(kNT) unit_kernel(const double* __restrict__ y, int64_t m,
                                                   const double* __restrict__ nn, double* __restrict__ x_out) {
  pdl_trigger();  // the next kernel in the stream may launch (it waits before reading)
  pdl_wait();
  const double nu = __ldcg(nn), f1 = __ldcg(nn + 1);
  const double f = f1 != 0.0 ? f1 : 1.0;
  const int64_t stride = (int64_t)gridDim.x * kNT;
  for (int64_t i = (int64_t)blockIdx.x * kNT + threadIdx.x; i < m; i += stride) x_out[i] = (__ldcg(y + i) * f) / nu;
}

// lagged iteration's last step: x_out = y / n with n = ||y|| from the
// fixed-order fold of the last launch's per-CTA sums (every CTA folds the
// same way); CTA 0 writes the last nu = n / (st[1] st[0]) (n at the first step)
__global__ void __launch_bounds__(kNT) unit_fold_kernel(const double* __restrict__ y, int64_t m,
                                                        const double* __restrict__ cta_part, int grid,
                                                        const double* __restrict__ st, double* __restrict__ nu_last,
                                                        double* __restrict__ x_out) {
  pdl_trigger();
  pdl_wait();
  __shared__ double n_s;
  const double ss = block_sum_fixed(cta_part, grid);
  if (threadIdx.x == 0) {
    const double n = sqrt(ss);
    n_s = n;
    if (blockIdx.x == 0) {
      const double Np = __ldcg(st), F1 = __ldcg(st + 1);
      *nu_last = Np > 0.0 ? n / ((F1 != 0.0 ? F1 : 1.0) * Np) : n;
    }
  }
  __syncthreads();
  const double n = n_s;
  const int64_t stride = (int64_t)gridDim.x * kNT;
  for (int64_t i = (int64_t)blockIdx.x * kNT + threadIdx.x; i < m; i += stride) x_out[i] = __ldcg(y + i) / n;
}

static int grid_for(int64_t m) {
  int64_t g = (m + kNT - 1) / kNT;
  if (g > dev_sm_count() * 8) g = dev_sm_count() * 8;
  return (int)(g < 1 ? 1 : g);
}

int launch_norm_step(const double* partials, int count, double* nn, double* nu_k, cudaStream_t s) {
  launch_pdl(norm_step_kernel, dim3(1), dim3(kNT), 0, s, partials, count, nn, nu_k);
  return 1;
}

int launch_scale_partials(double* y, int64_t m, const double* nn, double* partials, cudaStream_t s) {
  launch_pdl(scale_partials_kernel, dim3(kNormPartials), dim3(kNT), 0, s, y, m, nn, partials);
  return 1;
}

int launch_unit_fold(const double* y, int64_t m, const double* cta_part, int grid, const double* st, double* nu_last,
                     double* x_out, cudaStream_t s) {
  launch_pdl(unit_fold_kernel, dim3(grid_for(m)), dim3(kNT), 0, s, y, m, cta_part, grid, st, nu_last, x_out);
  return 1;
}

int launch_unit(const double* y, int64_t m, const double* nn, double* x_out, cudaStream_t s) {
  launch_pdl(unit_kernel, dim3(grid_for(m)), dim3(kNT), 0, s, y, m, nn, x_out);
  return 1;
}

int launch_norm_partials(const double* y, int64_t m, double* partials, cudaStream_t s) {
  launch_pdl(norm_partials_kernel<true>, dim3(kNormPartials), dim3(kNT), 0, s, y, m, partials);
  return 1;
}

int launch_sum_partials(const double* v, int64_t n, double* partials, cudaStream_t s) {
  launch_pdl(norm_partials_kernel<false>, dim3(kNormPartials), dim3(kNT), 0, s, v, n, partials);
  return 1;
}

int launch_normalize(const double* y, int64_t m, const double* partials, int count, double* x_out, double* nu_dev,
                     cudaStream_t s) {
  int64_t grid = (m + kNT - 1) / kNT;
  if (grid > dev_sm_count() * 8) grid = dev_sm_count() * 8;
  if (grid < 1) grid = 1;
  normalize_kernel<<<(int)grid, kNT, 0, s>>>(y, m, partials, count, x_out, nu_dev);
  return 1;
}

}  // namespace spmv
