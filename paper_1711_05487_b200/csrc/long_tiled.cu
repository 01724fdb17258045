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

constexpr int kLongRG = 2;  // row groups per x block (CTAs per block)

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

__device__ __forceinline__ void lt_ld256_s32(const int32_t* p, int (&c)[8]) {
  asm volatile("ld.global.nc.L1::no_allocate.v8.s32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(c[0]), "=r"(c[1]), "=r"(c[2]), "=r"(c[3]), "=r"(c[4]), "=r"(c[5]), "=r"(c[6]), "=r"(c[7])
               : "l"(p));
}
__device__ __forceinline__ void lt_ld256_f64(const double* p, double* v) {
  asm volatile("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
               : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3])
               : "l"(p));
}

// CTA (b, g): x block b staged in smem, long rows q = g, g + RG, ... of it.
// A warp streams a segment [s0, s1) in 8-aligned groups of 8 nonzeros per
// lane (one 256-bit colind load + two 256-bit value loads, 16 nonzeros per
// lane in flight), masking the group edges outside the segment.
__global__ void __launch_bounds__(kNT) long_tiled_kernel(const int32_t* __restrict__ col,
                                                         const double* __restrict__ val, const double* __restrict__ x,
                                                         int64_t n_long, int64_t n_cols, const int64_t* __restrict__ seg,
                                                         int64_t nblk, int rg, double* __restrict__ partial) {
  __shared__ double xs[kLongXB];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  // persistent: work item (b, g) = it / rg, it % rg, round-robin over CTAs
  for (int64_t it = blockIdx.x; it < nblk * rg; it += gridDim.x) {
  const int64_t b = it / rg, g = it % rg;
  const int64_t c0 = b * kLongXB;
  const int cw = (int)((n_cols - c0) < kLongXB ? (n_cols - c0) : kLongXB);
  __syncthreads();  // previous item's readers are done with xs
  for (int i = threadIdx.x; i < cw; i += kNT) xs[i] = ld_x(x + c0 + i);
  __syncthreads();
  for (int64_t q = g + (int64_t)rg * w; q < n_long; q += (int64_t)rg * (kNT / 32)) {
    const int64_t s0 = ld_ro(seg + q * (nblk + 1) + b), s1 = ld_ro(seg + q * (nblk + 1) + b + 1);
    double a0 = 0.0, a1 = 0.0;
    for (int64_t base = s0 & ~7ll; base < s1; base += 512) {
      int c[2][8];
      double v[2][8];
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int64_t e = base + 256 * r + 8 * lane;
        if (e < s1) {
          lt_ld256_s32(col + e, c[r]);
          lt_ld256_f64(val + e, v[r]);
          lt_ld256_f64(val + e + 4, v[r] + 4);
        } else {
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            c[r][i] = (int)c0;
            v[r][i] = 0.0;
          }
        }
      }
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int64_t e = base + 256 * r + 8 * lane;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const bool in = e + i >= s0 && e + i < s1;
          const double t = v[r][i] * xs[in ? c[r][i] - (int)c0 : 0];
          if (i & 1) a1 += in ? t : 0.0;
          else a0 += in ? t : 0.0;
        }
      }
    }
    const double t = warp_sum(a0 + a1);
    if (lane == 0) partial[q * nblk + b] = t;
  }
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
// persistent grid: per_sm CTAs per SM (<= 0: one CTA per work item)
int long_tiled_grid(int64_t nblk, int sm_count, int per_sm) {
  const int64_t items = nblk * kLongRG;
  if (per_sm <= 0) return (int)items;
  const int64_t g = (int64_t)sm_count * per_sm;
  return (int)(g < items ? g : items);
}

void launch_long_tiled(const ExecArgs& a, int part, cudaStream_t s) {
  if (a.n_long == 0) return;
  if (part == 1)
    long_tiled_kernel<<<a.long_grid, kNT, 0, s>>>(a.A.col, a.A.val, a.x, a.n_long, a.A.n_cols, a.long_seg, a.nblk,
                                                  kLongRG, a.long_partial);
  else
    long_reduce_kernel<<<(int)((a.n_long * 32 + kNT - 1) / kNT), kNT, 0, s>>>(a.long_partial, a.n_long, a.nblk,
                                                                             a.long_rows, a.y);
}

}  // namespace spmv
