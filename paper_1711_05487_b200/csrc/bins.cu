// bins.cu -- plan-time decomposition of A by row length for long_row_split
// (IMB class; Fig. 6 layout read through SPEC S:120-125):
//
//   short  rows (len <= T_s):        a compacted CSR in which every other row
//                                    is EMPTY (rowptr_s[i] + offset[i] equals
//                                    the original rowptr[i]), run by the
//                                    cta_stream kernel (which writes y = 0 for
//                                    the emptied rows);
//   medium rows (T_s < len <= L):    ordered row list, one warp per row,
//                                    straight from the original arrays;
//   long   rows (len > L):           ordered row list + chunk table (inspect.cu).
//
// All passes are deterministic (integer scans, ordered compaction).
#include "common.cuh"
#include "internal.h"

namespace spmv {

template <typename RP>
__device__ __forceinline__ int64_t row_len(const RP* rp, int64_t i) {
  return (int64_t)rp[i + 1] - (int64_t)rp[i];
}

// ---- multi-block exclusive scan of f(i), i < n, into out[0..n] ---------------
constexpr int kScanItems = kNT * 8;  // items per CTA

template <typename F>
__device__ __forceinline__ int64_t block_sum_items(int64_t base, int64_t n, F f) {
  int64_t s = 0;
  for (int q = 0; q < 8; ++q) {
    const int64_t i = base + (int64_t)q * kNT + threadIdx.x;
    if (i < n) s += f(i);
  }
  s = warp_sum(s);
  __shared__ int64_t ws[kNT / 32];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
  __syncthreads();
  int64_t t = 0;
  if (threadIdx.x == 0)
    for (int w = 0; w < kNT / 32; ++w) t += ws[w];
  __syncthreads();
  return t;  // valid in thread 0
}

template <typename RP>
__global__ void __launch_bounds__(kNT) filt_sum_kernel(const RP* __restrict__ rp, int64_t m, int64_t lo, int64_t hi,
                                                       int64_t* __restrict__ bsum) {
  const int64_t base = (int64_t)blockIdx.x * kScanItems;
  const int64_t t = block_sum_items(base, m, [&](int64_t i) {
    const int64_t l = row_len(rp, i);
    return (l >= lo && l <= hi) ? l : (int64_t)0;
  });
  if (threadIdx.x == 0) bsum[blockIdx.x] = t;
}

// single CTA: exclusive scan of nb block sums (in place, out[nb] = total)
__global__ void __launch_bounds__(kNT) scan_blocks_kernel(int64_t* __restrict__ v, int64_t nb) {
  __shared__ int64_t wsum[kNT / 32];
  __shared__ int64_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int64_t b = 0; b < nb; b += kNT) {
    const int64_t i = b + threadIdx.x;
    const int64_t x = i < nb ? v[i] : 0;
    int64_t inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    if (lane == 31) wsum[w] = inc;
    __syncthreads();
    int64_t pre = 0;
    for (int q = 0; q < w; ++q) pre += wsum[q];
    const int64_t c = carry;
    __syncthreads();
    if (i < nb) v[i] = c + pre + inc - x;
    if (threadIdx.x == kNT - 1) carry = c + pre + inc;
    __syncthreads();
  }
  if (threadIdx.x == 0) v[nb] = carry;
}

// out_rp[i] = sum_{r < i} len_r [lo <= len_r <= hi], i = 0..m
template <typename RP>
__global__ void __launch_bounds__(kNT) filt_rowptr_kernel(const RP* __restrict__ rp, int64_t m, int64_t lo,
                                                          int64_t hi, const int64_t* __restrict__ boff,
                                                          RP* __restrict__ out) {
  __shared__ int64_t wsum[kNT / 32];
  __shared__ int64_t carry;
  const int64_t base = (int64_t)blockIdx.x * kScanItems;
  if (threadIdx.x == 0) carry = boff[blockIdx.x];
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int q = 0; q < 8; ++q) {
    const int64_t i = base + (int64_t)q * kNT + threadIdx.x;
    int64_t x = 0;
    if (i < m) {
      const int64_t l = row_len(rp, i);
      x = (l >= lo && l <= hi) ? l : 0;
    }
    int64_t inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    if (lane == 31) wsum[w] = inc;
    __syncthreads();
    int64_t pre = 0;
    for (int u = 0; u < w; ++u) pre += wsum[u];
    const int64_t c = carry;
    __syncthreads();
    if (i < m) out[i] = (RP)(c + pre + inc - x);
    if (threadIdx.x == kNT - 1) carry = c + pre + inc;
    __syncthreads();
  }
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) out[m] = (RP)carry;
}

// copy the nonzeros of rows with lo <= len <= hi to their compacted position
template <typename RP>
__global__ void __launch_bounds__(kNT) filt_copy_kernel(const RP* __restrict__ rp, const int32_t* __restrict__ col,
                                                        const double* __restrict__ val, int64_t m, int64_t lo,
                                                        int64_t hi, const RP* __restrict__ rps,
                                                        int32_t* __restrict__ cols, double* __restrict__ vals) {
  // one warp per 32 rows; lanes stride inside each row
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * kNT + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * kNT) >> 5;
  for (int64_t r0 = warp * 32; r0 < m; r0 += nwarps * 32) {
    const int64_t r1 = r0 + 32 < m ? r0 + 32 : m;
    for (int64_t r = r0; r < r1; ++r) {
      const int64_t a = rp[r], l = (int64_t)rp[r + 1] - a;
      if (l < lo || l > hi) continue;
      const int64_t d = rps[r];
      for (int64_t t = lane; t < l; t += 32) {
        if (cols) cols[d + t] = col[a + t];  // (null: a values refresh, spmv_plan_update_values)
        vals[d + t] = val[a + t];
      }
    }
  }
}

// ---- ordered row lists: rows with lo <= len <= hi ----------------------------
template <typename RP>
__global__ void __launch_bounds__(kNT) rows_count_kernel(const RP* __restrict__ rp, int64_t m, int64_t lo,
                                                         int64_t hi, int64_t* __restrict__ bsum) {
  const int64_t base = (int64_t)blockIdx.x * kScanItems;
  const int64_t t = block_sum_items(base, m, [&](int64_t i) {
    const int64_t l = row_len(rp, i);
    return (l >= lo && l <= hi) ? (int64_t)1 : (int64_t)0;
  });
  if (threadIdx.x == 0) bsum[blockIdx.x] = t;
}

template <typename RP>
__global__ void __launch_bounds__(kNT) rows_write_kernel(const RP* __restrict__ rp, int64_t m, int64_t lo, int64_t hi,
                                                         const int64_t* __restrict__ boff, int32_t* __restrict__ out) {
  __shared__ int wcnt[kNT / 32];
  __shared__ int64_t base_s;
  const int64_t base = (int64_t)blockIdx.x * kScanItems;
  if (threadIdx.x == 0) base_s = boff[blockIdx.x];
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int q = 0; q < 8; ++q) {
    const int64_t i = base + (int64_t)q * kNT + threadIdx.x;
    bool f = false;
    if (i < m) {
      const int64_t l = row_len(rp, i);
      f = l >= lo && l <= hi;
    }
    const unsigned bal = __ballot_sync(0xffffffffu, f);
    if (lane == 0) wcnt[w] = __popc(bal);
    __syncthreads();
    int pre = 0;
    for (int u = 0; u < w; ++u) pre += wcnt[u];
    if (f) out[base_s + pre + __popc(bal & ((1u << lane) - 1))] = (int32_t)i;
    __syncthreads();
    if (threadIdx.x == 0) {
      int t = 0;
      for (int u = 0; u < kNT / 32; ++u) t += wcnt[u];
      base_s += t;
    }
    __syncthreads();
  }
}

int64_t scan_blocks(int64_t m) { return (m + kScanItems - 1) / kScanItems; }

template <typename RP>
static void filtered_csr_t(const MatView& A, int64_t lo, int64_t hi, void* out_rp, int32_t* out_col,
                           double* out_val, int64_t* scratch, cudaStream_t s) {
  const RP* rp = (const RP*)A.rowptr;
  const int64_t nb = scan_blocks(A.m);
  if (A.m == 0) {
    cudaMemsetAsync(out_rp, 0, sizeof(RP), s);
    return;
  }
  filt_sum_kernel<RP><<<(int)nb, kNT, 0, s>>>(rp, A.m, lo, hi, scratch);
  scan_blocks_kernel<<<1, kNT, 0, s>>>(scratch, nb);
  filt_rowptr_kernel<RP><<<(int)nb, kNT, 0, s>>>(rp, A.m, lo, hi, scratch, (RP*)out_rp);
  if (out_col) {
    int64_t g = (A.m + 32 * 8 - 1) / (32 * 8);
    if (g > dev_sm_count() * 16) g = dev_sm_count() * 16;
    filt_copy_kernel<RP><<<(int)g, kNT, 0, s>>>(rp, A.col, A.val, A.m, lo, hi, (const RP*)out_rp, out_col, out_val);
  }
}

// values of the filtered sub-matrix again (its rowptr out_rp from
// launch_filtered_csr): the bin's colind, possibly re-encoded since, is kept
void launch_filtered_vals(const MatView& A, int64_t lo, int64_t hi, const void* out_rp, double* out_val,
                          cudaStream_t s) {
  if (A.m == 0) return;
  int64_t g = (A.m + 32 * 8 - 1) / (32 * 8);
  if (g > dev_sm_count() * 16) g = dev_sm_count() * 16;
  if (A.rp_bytes == 8)
    filt_copy_kernel<int64_t><<<(int)g, kNT, 0, s>>>((const int64_t*)A.rowptr, A.col, A.val, A.m, lo, hi,
                                                     (const int64_t*)out_rp, nullptr, out_val);
  else
    filt_copy_kernel<int32_t><<<(int)g, kNT, 0, s>>>((const int32_t*)A.rowptr, A.col, A.val, A.m, lo, hi,
                                                     (const int32_t*)out_rp, nullptr, out_val);
}

// rowptr (and, when out_col != null, colind/values) of the sub-matrix made of
// the rows with lo <= len <= hi, every other row empty. scratch: scan_blocks(m)+1.
void launch_filtered_csr(const MatView& A, int64_t lo, int64_t hi, void* out_rp, int32_t* out_col, double* out_val,
                         int64_t* scratch, cudaStream_t s) {
  if (A.rp_bytes == 8) filtered_csr_t<int64_t>(A, lo, hi, out_rp, out_col, out_val, scratch, s);
  else filtered_csr_t<int32_t>(A, lo, hi, out_rp, out_col, out_val, scratch, s);
}

template <typename RP>
static void row_list_t(const MatView& A, int64_t lo, int64_t hi, int32_t* out, int64_t* scratch, cudaStream_t s) {
  const RP* rp = (const RP*)A.rowptr;
  const int64_t nb = scan_blocks(A.m);
  if (A.m == 0) {
    cudaMemsetAsync(scratch, 0, 16, s);
    return;
  }
  rows_count_kernel<RP><<<(int)nb, kNT, 0, s>>>(rp, A.m, lo, hi, scratch);
  scan_blocks_kernel<<<1, kNT, 0, s>>>(scratch, nb);
  if (out) rows_write_kernel<RP><<<(int)nb, kNT, 0, s>>>(rp, A.m, lo, hi, scratch, out);
}

// ordered list of the rows with lo <= len <= hi; scratch: scan_blocks(m)+1
void launch_row_list(const MatView& A, int64_t lo, int64_t hi, int32_t* out, int64_t* scratch, cudaStream_t s) {
  if (A.rp_bytes == 8) row_list_t<int64_t>(A, lo, hi, out, scratch, s);
  else row_list_t<int32_t>(A, lo, hi, out, scratch, s);
}

// ---- first nonzero of each row-aligned STREAM tile ---------------------------------
template <typename RP>
__global__ void tile_nz_kernel(const RP* __restrict__ rp, const int32_t* __restrict__ tile_row, int64_t T,
                               int64_t* __restrict__ out) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k <= T) out[k] = (int64_t)rp[tile_row[k]];
}

void launch_tile_nz(const MatView& A, const int32_t* tile_row, int64_t T, int64_t* tile_nz, cudaStream_t s) {
  const int g = (int)((T + 1 + kNT - 1) / kNT);
  if (A.rp_bytes == 8) tile_nz_kernel<int64_t><<<g, kNT, 0, s>>>((const int64_t*)A.rowptr, tile_row, T, tile_nz);
  else tile_nz_kernel<int32_t><<<g, kNT, 0, s>>>((const int32_t*)A.rowptr, tile_row, T, tile_nz);
}

// ---- compacted rowptr of a bin ---------------------------------------------------
template <typename RP>
__global__ void gather_rowptr_kernel(const RP* __restrict__ frp, const int32_t* __restrict__ rows, int64_t n,
                                     int64_t m, RP* __restrict__ out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q <= n; q += stride)
    out[q] = q < n ? frp[rows[q]] : frp[m];
}

void launch_gather_rowptr(const void* frp, int rp_bytes, const int32_t* rows, int64_t n, int64_t m, void* out,
                          cudaStream_t s) {
  int64_t g = (n + 1 + kNT - 1) / kNT;
  if (g > dev_sm_count() * 16) g = dev_sm_count() * 16;
  if (rp_bytes == 8)
    gather_rowptr_kernel<int64_t><<<(int)g, kNT, 0, s>>>((const int64_t*)frp, rows, n, m, (int64_t*)out);
  else
    gather_rowptr_kernel<int32_t><<<(int)g, kNT, 0, s>>>((const int32_t*)frp, rows, n, m, (int32_t*)out);
}

// ---- medium rows: one VS-lane group per listed row ----------------------------
template <int VS, typename RP>
__global__ void __launch_bounds__(kNT) rowlist_kernel(const RP* __restrict__ rp, const int32_t* __restrict__ col,
                                                      const double* __restrict__ val, const double* __restrict__ x,
                                                      double* __restrict__ y, const int32_t* __restrict__ rows,
                                                      int64_t nrows) {
  const int lane = threadIdx.x % VS;
  const int gi = (threadIdx.x & 31) / VS;
  const int64_t ngroups = (int64_t)gridDim.x * (kNT / VS);
  const int64_t wfirst = ((int64_t)blockIdx.x * kNT + (threadIdx.x & ~31)) / VS;
  for (int64_t qb = wfirst; qb < nrows; qb += ngroups) {
    const int64_t q = qb + gi;
    const bool active = q < nrows;
    int64_t r = 0, a = 0, b = 0;
    if (active) {
      r = ld_ro(rows + q);
      a = (int64_t)ld_ro(rp + r);
      b = (int64_t)ld_ro(rp + r + 1);
    }
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    int64_t j = a + lane;
    for (; j + 3 * VS < b; j += 4 * VS) {
      const int c0 = ld_stream(col + j), c1 = ld_stream(col + j + VS), c2 = ld_stream(col + j + 2 * VS),
                c3 = ld_stream(col + j + 3 * VS);
      const double v0 = ld_stream(val + j), v1 = ld_stream(val + j + VS), v2 = ld_stream(val + j + 2 * VS),
                   v3 = ld_stream(val + j + 3 * VS);
      a0 = fma(v0, ld_x(x + c0), a0);
      a1 = fma(v1, ld_x(x + c1), a1);
      a2 = fma(v2, ld_x(x + c2), a2);
      a3 = fma(v3, ld_x(x + c3), a3);
    }
    for (; j < b; j += VS) a0 = fma(ld_stream(val + j), ld_x(x + ld_stream(col + j)), a0);
    const double s = group_sum<VS>((a0 + a1) + (a2 + a3));
    if (active && lane == 0) y[r] = s;
  }
}

void launch_rowlist(const ExecArgs& a, const int32_t* rows, int64_t nrows, cudaStream_t s) {
  if (nrows == 0) return;
  int64_t grid = (nrows * 32 + kNT - 1) / kNT;
  const int64_t cap = (int64_t)a.sm_count * 8;
  if (grid > cap) grid = cap;
  if (a.A.rp_bytes == 8)
    rowlist_kernel<32, int64_t><<<(int)grid, kNT, 0, s>>>((const int64_t*)a.A.rowptr, a.A.col, a.A.val, a.x, a.y,
                                                          rows, nrows);
  else
    rowlist_kernel<32, int32_t><<<(int)grid, kNT, 0, s>>>((const int32_t*)a.A.rowptr, a.A.col, a.A.val, a.x, a.y,
                                                          rows, nrows);
}

}  // namespace spmv
