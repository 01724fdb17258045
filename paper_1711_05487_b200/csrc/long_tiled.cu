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
#include "tiles.cuh"

namespace spmv {

#ifndef LONG_RG
#define LONG_RG 2
#endif
constexpr int kLongRG = LONG_RG;  // row groups per x block (CTAs per block)

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

// c16[j] = colind[j] & (kLongXB - 1) for the nonzeros of the long rows (one
// warp per row)
template <typename RP>
__global__ void long_c16_kernel(const RP* __restrict__ rp, const int32_t* __restrict__ col,
                                const int32_t* __restrict__ long_rows, int64_t n_long, uint16_t* __restrict__ c16) {
  static_assert((kLongXB & (kLongXB - 1)) == 0 && kLongXB <= 65536, "x block: a power of two <= 2^16");
  const int64_t q = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (q >= n_long) return;
  const int64_t r = long_rows[q];
  for (int64_t j = (int64_t)rp[r] + (threadIdx.x & 31); j < (int64_t)rp[r + 1]; j += 32)
    c16[j] = (uint16_t)(col[j] & (int32_t)(kLongXB - 1));
}

void launch_long_c16(const MatView& A, const int32_t* long_rows, int64_t n_long, uint16_t* c16, cudaStream_t s) {
  if (n_long == 0) return;
  const int g = (int)((n_long * 32 + kNT - 1) / kNT);
  if (A.rp_bytes == 8)
    long_c16_kernel<int64_t><<<g, kNT, 0, s>>>((const int64_t*)A.rowptr, A.col, long_rows, n_long, c16);
  else
    long_c16_kernel<int32_t><<<g, kNT, 0, s>>>((const int32_t*)A.rowptr, A.col, long_rows, n_long, c16);
}

// CTA item loop (persistent when the grid is smaller than the item count)
#ifndef LONG_LB
#define LONG_LB 4
#endif
template <bool C16>
__global__ void __launch_bounds__(kNT, LONG_LB) long_tiled_kernel(const LongP p) {
  __shared__ double xs[kLongXB];
  // PDL-launched (SPLIT concurrent mode): wait for the previous SpMV, THEN let
  // the short-row bin launch -- it skips its own wait, since every CTA of
  // this grid has seen the previous kernels complete (no-ops otherwise)
  pdl_wait();
  pdl_trigger();
  for (int64_t it = blockIdx.x; it < p.nblk * p.rg; it += gridDim.x) {
    long_item<kNT, C16>(p, it, xs);
    __syncthreads();  // every warp is done with xs before the next item restages it
  }
}

// y[long_rows[q]] = sum_b partial[q][b] (lane-strided, butterfly: fixed order)
__global__ void __launch_bounds__(kNT) long_reduce_kernel(const double* __restrict__ partial, int64_t n_long,
                                                          int64_t nblk, const int32_t* __restrict__ long_rows,
                                                          double* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  const int64_t q = ((int64_t)blockIdx.x * kNT + threadIdx.x) >> 5;
  if (q >= n_long) return;
  const double a = long_row_total(partial + q * nblk, nblk, lane);
  if (lane == 0) y[long_rows[q]] = a;
}

LongP long_params(const ExecArgs& a) {
  LongP p;
  p.col = a.A.col;
  p.val = a.A.val;
  p.x = a.x;
  p.seg = a.long_seg;
  p.col16 = a.long_c16;
  p.partial = a.long_partial;
  p.n_long = a.n_long;
  p.n_cols = a.A.n_cols;
  p.nblk = a.nblk;
  p.rg = kLongRG;
  return p;
}

int long_items(const ExecArgs& a) { return (int)(a.nblk * kLongRG); }

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
  if (part == 3) {  // programmatic launch (SPLIT concurrent mode)
    if (a.long_c16) launch_pdl(long_tiled_kernel<true>, dim3(a.long_grid), dim3(kNT), 0, s, long_params(a));
    else launch_pdl(long_tiled_kernel<false>, dim3(a.long_grid), dim3(kNT), 0, s, long_params(a));
  } else if (part == 1) {
    if (a.long_c16) long_tiled_kernel<true><<<a.long_grid, kNT, 0, s>>>(long_params(a));
    else long_tiled_kernel<false><<<a.long_grid, kNT, 0, s>>>(long_params(a));
  }
  else
    long_reduce_kernel<<<(int)((a.n_long * 32 + kNT - 1) / kNT), kNT, 0, s>>>(a.long_partial, a.n_long, a.nblk,
                                                                             a.long_rows, a.y);
}

}  // namespace spmv
