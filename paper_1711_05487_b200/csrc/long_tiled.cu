// long_tiled.cu -- column-tiled long rows for long_row_split (IMB
// decomposition): "every row is computed by all threads and a
// reduction of partial results follows", re-designed for sm_100a
// so the x gather of dense-ish long rows is served from shared memory.
//
// CTA b stages the x block [b*XB, (b+1)*XB) in smem (coalesced, 16 KB) and
// streams, warp by warp, the segment of every long row whose columns fall in
// that block (segment bounds precomputed at plan time by binary search inside
// each sorted row). Each (row, block) partial goes to partial[q][b]; a second
// kernel sums each row's partials in block order (deterministic) into y.
// Chosen when the long rows are dense enough that a block segment averages
// >= 64 nonzeros; otherwise the nonzero-chunk kernel is used.
#include "common.cuh"
#include "internal.h"

namespace spmv {

// seg[q*(nblk+1) + b] = first nonzero of long row q with column >= b*XB
template <typename RP>
__global__ void long_seg_kernel(const RP* __restrict__ rp, const int32_t* __restrict__ col,
                                const int32_t* __restrict__ long_rows, int64_t n_long, int64_t nblk,
                                int64_t* __restrict__ seg) {
  const int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= n_long * (nblk + 1)) return;
  const int64_t q = id / (nblk + 1), b = id % (nblk + 1);
  const int64_t r = long_rows[q];
  int64_t lo = (int64_t)rp[r], hi = (int64_t)rp[r + 1];
  const int64_t key = b * kLongXB;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if ((int64_t)col[mid] < key) lo = mid + 1; else hi = mid;
  }
  seg[id] = lo;
}

void launch_long_seg(const MatView& A, const int32_t* long_rows, int64_t n_long, int64_t nblk, int64_t* seg,
                     cudaStream_t s) {
  const int64_t n = n_long * (nblk + 1);
  const int g = (int)((n + kNT - 1) / kNT);
  if (A.rp_bytes == 8)
    long_seg_kernel<int64_t><<<g, kNT, 0, s>>>((const int64_t*)A.rowptr, A.col, long_rows, n_long, nblk, seg);
  else
    long_seg_kernel<int32_t><<<g, kNT, 0, s>>>((const int32_t*)A.rowptr, A.col, long_rows, n_long, nblk, seg);
}

__global__ void __launch_bounds__(kNT) long_tiled_kernel(const int32_t* __restrict__ col,
                                                         const double* __restrict__ val, const double* __restrict__ x,
                                                         int64_t n_long, int64_t n_cols, const int64_t* __restrict__ seg,
                                                         int64_t nblk, double* __restrict__ partial) {
  __shared__ double xs[kLongXB];
  const int64_t b = blockIdx.x;
  const int64_t c0 = b * kLongXB;
  const int cw = (int)((n_cols - c0) < kLongXB ? (n_cols - c0) : kLongXB);
  for (int i = threadIdx.x; i < cw; i += kNT) xs[i] = ld_x(x + c0 + i);
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int64_t q = w; q < n_long; q += kNT / 32) {
    const int64_t s0 = ld_ro(seg + q * (nblk + 1) + b), s1 = ld_ro(seg + q * (nblk + 1) + b + 1);
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    int64_t j = s0 + lane;
    for (; j + 96 < s1; j += 128) {
      const int k0 = ld_stream(col + j) - (int)c0, k1 = ld_stream(col + j + 32) - (int)c0,
                k2 = ld_stream(col + j + 64) - (int)c0, k3 = ld_stream(col + j + 96) - (int)c0;
      a0 = fma(ld_stream(val + j), xs[k0], a0);
      a1 = fma(ld_stream(val + j + 32), xs[k1], a1);
      a2 = fma(ld_stream(val + j + 64), xs[k2], a2);
      a3 = fma(ld_stream(val + j + 96), xs[k3], a3);
    }
    for (; j < s1; j += 32) a0 = fma(ld_stream(val + j), xs[ld_stream(col + j) - (int)c0], a0);
    const double t = warp_sum((a0 + a1) + (a2 + a3));
    if (lane == 0) partial[q * nblk + b] = t;
  }
}

// y[long_rows[q]] = sum_b partial[q][b] (lane-strided, butterfly: fixed order)
__global__ void __launch_bounds__(kNT) long_reduce_kernel(const double* __restrict__ partial, int64_t n_long,
                                                          int64_t nblk, const int32_t* __restrict__ long_rows,
                                                          double* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  const int64_t q = ((int64_t)blockIdx.x * kNT + threadIdx.x) >> 5;
  if (q >= n_long) return;
  double a = 0.0;
  for (int64_t b = lane; b < nblk; b += 32) a += partial[q * nblk + b];
  a = warp_sum(a);
  if (lane == 0) y[long_rows[q]] = a;
}

// part 1: the column-tiled partials; part 2: the ordered per-row reduction
void launch_long_tiled(const ExecArgs& a, int part, cudaStream_t s) {
  if (a.n_long == 0) return;
  if (part == 1)
    long_tiled_kernel<<<(int)a.nblk, kNT, 0, s>>>(a.A.col, a.A.val, a.x, a.n_long, a.A.n_cols, a.long_seg, a.nblk,
                                                  a.long_partial);
  else
    long_reduce_kernel<<<(int)((a.n_long * 32 + kNT - 1) / kNT), kNT, 0, s>>>(a.long_partial, a.n_long, a.nblk,
                                                                             a.long_rows, a.y);
}

}  // namespace spmv
