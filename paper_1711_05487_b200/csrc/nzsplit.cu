// nzsplit.cu -- nnz_split: the IMB/ML-class kernel for skewed, long-row and
// random-gather matrices, re-designed for sm_100a.
//
// The paper balances threads by giving each an equal share of nonzeros
// (static 1-D nnz-balanced partition) and, for long rows, lets
// several threads share a row and reduce their partial results (long-row
// decomposition). nnz_split does both at warp granularity:
//
//  * the rows are compacted to the non-empty ones (rpc[mc+1], rowmap[mc+1],
//    rowmap[mc] = m): with every row non-empty, an equal split of the
//    NONZEROS is also balanced in rows (rows <= nonzeros), so the merge path
//    degenerates to a plain nnz split and needs no row-axis search;
//  * warp tile k = nonzeros [k*W, (k+1)*W), W = 256; lane l owns the 8
//    consecutive nonzeros [8l, 8l+8) of the tile, loaded with one 256-bit
//    colind load and two 256-bit value loads (LDG.256, L1 no-allocate: every
//    32-B sector is consumed whole by one instruction, so the streams cost
//    exactly their bytes);
//  * the x gathers are plain L1-allocating loads and the kernel uses 256 B of
//    shared memory per CTA, leaving the unified L1 to x: on power-law column
//    distributions the hot x entries are then served from L1 (measured on
//    B200: ~280 G gathers/s vs ~150 G/s with 180 KB of smem per SM);
//  * row ends inside the tile are a 256-bit mask built from rpc; each lane
//    sums its 8 products sequentially, writes the rows that start and end in
//    its range, and ONE segmented scan across the 32 lanes completes the rows
//    cut by lane edges (15 shuffles per 256 nonzeros);
//  * a row is written (y = its in-tile piece) by the tile where it ENDS; the
//    piece of the row crossing the tile end is the tile's carry, added in
//    tile order by the ordered fix-up kernel (deterministic, no fp atomics);
//  * the empty rows between non-empty rows q and q+1 are zeroed by the tile
//    where row q ends (y is written exactly once per row).
#include <algorithm>
#include <cstdlib>

#include "tiles.cuh"

namespace spmv {

constexpr int kNzWarps = 8;  // warps per CTA (plain mode)
#ifndef NZ_HOT_WARPS
#define NZ_HOT_WARPS 32
#endif
#ifndef NZ_HOT_PF
#define NZ_HOT_PF 0
#endif
#ifndef NZ_HOT_MASK
#define NZ_HOT_MASK 0
#endif
#ifndef NZ_MASK
#define NZ_MASK 1
#endif
constexpr int kNzHotWarps = NZ_HOT_WARPS;  // warps per CTA (hot-x mode: one CTA per SM)
constexpr int kNzHotPrefetch = NZ_HOT_PF;  // 1: next tile's streams, 2: next tile's colind only
// row ends from the per-tile mask (see nz_tile_compute); B200: C4 134 -> 127 us,
// C5 as nnz_split 4.47 -> 3.91 ms, C3 hot-x 282 -> 290 us (kept on tile_q + rpc)
constexpr bool kNzHotMask = NZ_HOT_MASK;
constexpr bool kNzMask = NZ_MASK;

size_t nz_smem_bytes(int n_hot) { return n_hot > 0 ? (size_t)n_hot * 8 + 16 : 0; }

template <typename RP>
__device__ __forceinline__ void nz_col_load(const NzP<RP>& p, int64_t k, int lane, int (&c)[8]) {
  const int64_t t0 = k * kNzTile;
  const int cnt = (int)((p.nnz - t0) < kNzTile ? (p.nnz - t0) : kNzTile);
  const int e0 = lane * 8;
  if (e0 + 8 <= cnt) {
    ld256_s32(p.col + t0 + e0, c);
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i] = e0 + i < cnt ? ld_stream(p.col + t0 + e0 + i) : 0;
  }
}
template <typename RP>
__device__ __forceinline__ void nz_val_load(const NzP<RP>& p, int64_t k, int lane, double (&v)[8]) {
  const int64_t t0 = k * kNzTile;
  const int cnt = (int)((p.nnz - t0) < kNzTile ? (p.nnz - t0) : kNzTile);
  const int e0 = lane * 8;
  if (e0 + 8 <= cnt) {
    ld256_f64(p.val + t0 + e0, v);
    ld256_f64(p.val + t0 + e0 + 4, v + 4);
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = e0 + i < cnt ? ld_stream(p.val + t0 + e0 + i) : 0.0;
  }
}

// HOT: the plan re-encoded colind of the n_hot most frequent columns as
// ~slot (negative); their x values are bulk-copied into shared memory once
// per CTA and gathered from there. On B200 a divergent global gather costs
// the L1 data pipe about one wavefront per lane (~1 sector / clk / SM is the
// C3 ceiling), a shared-memory gather only its bank conflicts.
template <typename RP, bool HOT, bool L2G>
__global__ void __launch_bounds__(HOT ? 32 * kNzHotWarps : 32 * kNzWarps, HOT ? 1 : 4)
    nzsplit_kernel(const NzP<RP> p) {
  constexpr int NW = HOT ? kNzHotWarps : kNzWarps;
  constexpr bool MASK = HOT ? kNzHotMask : kNzMask;
  extern __shared__ __align__(16) double xh[];
  __shared__ __align__(16) uint32_t emask_s[MASK ? 1 : NW][8];
  pdl_trigger();
  if (!p.skip_wait) pdl_wait();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t* em = emask_s[MASK ? 0 : w];
  if constexpr (HOT) {
    uint64_t* bar = reinterpret_cast<uint64_t*>(xh + p.n_hot);
    if (threadIdx.x == 0) {
      mbar_init(bar, 1);
      fence_mbar_init();
      mbar_arrive_expect_tx(bar, (uint32_t)(p.n_hot * 8));
      bulk_g2s(xh, p.xhot, (uint32_t)(p.n_hot * 8), bar, policy_evict_last());  // read by every CTA
    }
    __syncthreads();
    mbar_wait(bar, 0);
  }
  // static round-robin, one tile at a time (warp g takes tiles g, g + W,
  // ...): the tiles in flight form one contiguous window of the streams,
  // which B200 DRAM rewards (C3: 294 us; chunks of 8 consecutive tiles per
  // warp 358 us; dynamic tickets 350 us -- same-address atomics serialise)
  const int64_t nw = (int64_t)gridDim.x * NW;
  if constexpr (HOT && kNzHotPrefetch == 2) {
    // the next tile's colind is loaded with this tile's values and gathers:
    // one round trip per tile instead of colind, then gathers
    int64_t k = p.k0 + (int64_t)blockIdx.x * NW + w;
    int c[8], cn[8];
    if (k < p.T) nz_col_load(p, k, lane, c);
    for (; k < p.T; k += nw) {
      double v[8];
      nz_val_load(p, k, lane, v);
      if (k + nw < p.T) nz_col_load(p, k + nw, lane, cn);
      NzMeta m{};
      nz_tile_compute<RP, HOT, MASK, L2G>(p, k, lane, xh, em, c, v, m);
#pragma unroll
      for (int i = 0; i < 8; ++i) c[i] = cn[i];
    }
  } else if constexpr (HOT && kNzHotPrefetch == 1) {
    // the next tile's streams are loaded while this tile gathers x
    int64_t k = p.k0 + (int64_t)blockIdx.x * NW + w;
    int c[8], cn[8];
    double v[8], vn[8];
    NzMeta m, mn;
    if (k < p.T) nz_tile_load<RP, MASK>(p, k, lane, c, v, m);
    for (; k < p.T; k += nw) {
      if (k + nw < p.T) nz_tile_load<RP, MASK>(p, k + nw, lane, cn, vn, mn);
      nz_tile_compute<RP, HOT, MASK, L2G>(p, k, lane, xh, em, c, v, m);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        c[i] = cn[i];
        v[i] = vn[i];
      }
      m = mn;
    }
  } else {
    for (int64_t k = p.k0 + (int64_t)blockIdx.x * NW + w; k < p.T; k += nw)
      nz_tile<RP, HOT, MASK, L2G>(p, k, lane, xh, em);
  }
}

// xhot[s] = x[hot_cols[s]] (once per SpMV, before the hot-x kernel)
__global__ void nz_hot_gather_kernel(const int32_t* __restrict__ hot_cols, int n_hot, const double* __restrict__ x,
                                     double* __restrict__ xhot) {
  pdl_trigger();
  pdl_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n_hot) xhot[i] = __ldg(x + hot_cols[i]);
}

// tile_q[k] = (last q with rpc[q] <= k*W) for k < T, tile_q[T] = mc
template <typename RP>
__global__ void nz_tile_rows_kernel(const RP* __restrict__ rpc, int64_t mc, int64_t T, int32_t* __restrict__ tq) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k > T) return;
  if (k == T) {
    tq[k] = (int32_t)mc;
    return;
  }
  const int64_t key = k * kNzTile;
  int64_t lo = 0, hi = mc;  // upper_bound over rpc[0..mc]
  while (lo < hi) {
    const int64_t mid = (lo + hi + 1) >> 1;
    if ((int64_t)rpc[mid] <= key) lo = mid; else hi = mid - 1;
  }
  tq[k] = (int32_t)lo;
}

__global__ void set_i32_kernel(int32_t* p, int32_t v) { *p = v; }

// emask bit e set when a (non-empty, compacted) row ends at nonzero e
template <typename RP>
__global__ void nz_emask_kernel(const RP* __restrict__ rpc, int64_t mc, uint32_t* __restrict__ emask) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= mc) return;
  const int64_t e = (int64_t)rpc[q + 1] - 1;
  atomicOr(emask + (e >> 5), 1u << (e & 31));
}

// epre[k] byte w = row ends in mask words [0, w) of tile k
__global__ void nz_epre_kernel(const uint32_t* __restrict__ emask, int64_t T, uint64_t* __restrict__ epre) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= T) return;
  uint64_t b = 0;
  uint32_t acc = 0;
  for (int w = 0; w < 8; ++w) {
    b |= (uint64_t)acc << (8 * w);
    acc += __popc(emask[k * 8 + w]);
  }
  epre[k] = b;
}

// *out = max over q of the empty run before compacted row q (q <= mc; the
// run after the last row ends at rowmap[mc] = m_out); *out zeroed by the caller
__global__ void nz_max_gap_kernel(const int32_t* __restrict__ rowmap, int64_t mc, int32_t* out) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q > mc) return;
  const int32_t g = rowmap[q] - (q > 0 ? rowmap[q - 1] + 1 : 0);
  if (g > 0) atomicMax(out, g);
}

void launch_nz_max_gap(const NzPlan& z, int32_t* out, cudaStream_t s) {
  cudaMemsetAsync(out, 0, 4, s);
  nz_max_gap_kernel<<<(unsigned)((z.mc + 1 + kNT - 1) / kNT), kNT, 0, s>>>(z.rowmap, z.mc, out);
}

void launch_nz_tiles(const NzPlan& z, cudaStream_t s) {
  const int g = (int)((z.T + 1 + kNT - 1) / kNT);
  if (z.V.rp_bytes == 8)
    nz_tile_rows_kernel<int64_t><<<g, kNT, 0, s>>>((const int64_t*)z.rpc, z.mc, z.T, z.tile_q);
  else
    nz_tile_rows_kernel<int32_t><<<g, kNT, 0, s>>>((const int32_t*)z.rpc, z.mc, z.T, z.tile_q);
  set_i32_kernel<<<1, 1, 0, s>>>(const_cast<int32_t*>(z.rowmap) + z.mc, (int32_t)z.m_out);
  cudaMemsetAsync(z.emask, 0, (size_t)z.T * 8 * sizeof(uint32_t), s);
  const int ge = (int)std::max<int64_t>(1, (z.mc + kNT - 1) / kNT);
  if (z.V.rp_bytes == 8)
    nz_emask_kernel<int64_t><<<ge, kNT, 0, s>>>((const int64_t*)z.rpc, z.mc, z.emask);
  else
    nz_emask_kernel<int32_t><<<ge, kNT, 0, s>>>((const int32_t*)z.rpc, z.mc, z.emask);
  nz_epre_kernel<<<(unsigned)std::max<int64_t>(1, (z.T + kNT - 1) / kNT), kNT, 0, s>>>(z.emask, z.T, z.epre);
}

template <typename RP>
static NzP<RP> nz_params(const NzPlan& z, const double* x, double* y) {
  NzP<RP> p;
  p.rpc = (const RP*)z.rpc;
  p.col = z.V.col;
  p.val = z.V.val;
  p.x = x;
  p.y = y;
  p.rowmap = z.rowmap;
  p.tile_q = z.tile_q;
  p.emask = z.emask;
  p.epre = z.epre;
  p.carry_row = z.carry_row;
  p.carry_val = z.carry_val;
  p.orp = (const RP*)z.skip_rp;
  p.xhot = z.xhot;
  p.nnz = z.V.nnz;
  p.T = z.T;
  p.k0 = 0;
  p.n_hot = z.n_hot;
  p.zero_gaps = z.zero_gaps ? 1 : 0;
  p.skip_wait = z.skip_wait ? 1 : 0;
  return p;
}

NzP<int32_t> nz_params32(const NzPlan& z, const double* x, double* y) { return nz_params<int32_t>(z, x, y); }
NzP<int64_t> nz_params64(const NzPlan& z, const double* x, double* y) { return nz_params<int64_t>(z, x, y); }

template <typename RP, bool HOT>
static int nz_grid_t(const NzPlan& z, int sm_count) {
  const size_t sm = nz_smem_bytes(HOT ? z.n_hot : 0);
  const int threads = HOT ? 32 * kNzHotWarps : 32 * kNzWarps;
  // (the attribute is per function: always the largest table, so plans of
  // different table sizes can share it)
  if (HOT && (cudaFuncSetAttribute(nzsplit_kernel<RP, HOT, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)nz_smem_bytes(kHotMax)) != cudaSuccess ||
              cudaFuncSetAttribute(nzsplit_kernel<RP, HOT, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)nz_smem_bytes(kHotMax)) != cudaSuccess))
    return -1;
  int per_sm = 0;
  const cudaError_t oe =
      z.gather_l2 ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, nzsplit_kernel<RP, HOT, true>, threads, sm)
                  : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, nzsplit_kernel<RP, HOT, false>, threads, sm);
  if (oe != cudaSuccess || per_sm < 1) return -1;
  if (const char* e = getenv("SPMV_NZ_CTAS")) per_sm = std::max(1, std::min(per_sm, atoi(e)));
  int64_t grid = (int64_t)sm_count * per_sm;
  const int64_t nwarps = HOT ? kNzHotWarps : kNzWarps;
  const int64_t need = (z.T + nwarps - 1) / nwarps;
  if (grid > need || !z.persistent) grid = need;  // non-persistent: one tile per warp, scheduler-balanced
  return (int)(grid > 0 ? grid : 1);
}

int nz_prepare(NzPlan& z, int sm_count) {
  const bool hot = z.n_hot > 0;
  if (z.V.rp_bytes == 8) return hot ? nz_grid_t<int64_t, true>(z, sm_count) : nz_grid_t<int64_t, false>(z, sm_count);
  return hot ? nz_grid_t<int32_t, true>(z, sm_count) : nz_grid_t<int32_t, false>(z, sm_count);
}

template <typename RP>
static NzP<RP> nz_range_params(const NzPlan& z, const double* x, double* y, int64_t k0, int64_t k1) {
  NzP<RP> p = nz_params<RP>(z, x, y);
  p.k0 = k0;
  p.T = k1;
  return p;
}

// tiles [k0, k1) (the whole pass: 0, T); grid capped to the range's warps
template <bool HOT>
static void launch_nz_main(const NzPlan& z, const double* x, double* y, cudaStream_t s, int64_t k0 = 0,
                           int64_t k1 = -1) {
  if (k1 < 0) k1 = z.T;
  const size_t sm = nz_smem_bytes(HOT ? z.n_hot : 0);
  const int nw = HOT ? kNzHotWarps : kNzWarps;
  const dim3 blk(32 * nw);
  const dim3 g((unsigned)std::max<int64_t>(1, std::min<int64_t>(z.grid, (k1 - k0 + nw - 1) / nw)));
  if (z.V.rp_bytes == 8) {
    if (z.gather_l2) launch_pdl(nzsplit_kernel<int64_t, HOT, true>, g, blk, sm, s, nz_range_params<int64_t>(z, x, y, k0, k1));
    else launch_pdl(nzsplit_kernel<int64_t, HOT, false>, g, blk, sm, s, nz_range_params<int64_t>(z, x, y, k0, k1));
  } else {
    if (z.gather_l2) launch_pdl(nzsplit_kernel<int32_t, HOT, true>, g, blk, sm, s, nz_range_params<int32_t>(z, x, y, k0, k1));
    else launch_pdl(nzsplit_kernel<int32_t, HOT, false>, g, blk, sm, s, nz_range_params<int32_t>(z, x, y, k0, k1));
  }
}

// pipelined host execute (api.cu host_pipe_*): the y clear / hot-x gather
// before the first range, the ranges, and the fix-up of a range's carries
// (run after the NEXT range: a row is assigned by the tile where it ends)
int launch_nz_prologue(const NzPlan& z, const double* x, double* y, cudaStream_t s) {
  if (z.memset_y) cudaMemsetAsync(y, 0, (size_t)z.m_out * 8, s);
  if (z.n_hot > 0) {
    launch_pdl(nz_hot_gather_kernel, dim3((z.n_hot + kNT - 1) / kNT), dim3(kNT), 0, s, z.hot_cols, z.n_hot, x,
               z.xhot);
    return 1;
  }
  return 0;
}
int launch_nz_range(const NzPlan& z, const double* x, double* y, int64_t k0, int64_t k1, cudaStream_t s) {
  if (k1 <= k0) return 0;
  if (z.n_hot > 0) launch_nz_main<true>(z, x, y, s, k0, k1);
  else launch_nz_main<false>(z, x, y, s, k0, k1);
  return 1;
}
int launch_nz_fixup_range(const NzPlan& z, double* y, int64_t k0, int64_t k1, cudaStream_t s) {
  if (k1 <= k0 || z.T <= 1) return 0;
  return launch_fixup_range(z.carry_row + k0, z.carry_val + k0, k1 - k0, y, s);
}

int launch_nz_plan(const NzPlan& z, const double* x, double* y, int stage, cudaStream_t s) {
  int n = 0;
  if (z.T == 0) {
    if (stage != 2 && z.zero_gaps && !z.skip_rp && z.m_out > 0) cudaMemsetAsync(y, 0, (size_t)z.m_out * 8, s);
    return 0;
  }
  if (stage != 2) {
    if (z.memset_y) cudaMemsetAsync(y, 0, (size_t)z.m_out * 8, s);
    if (z.n_hot > 0) {
      launch_pdl(nz_hot_gather_kernel, dim3((z.n_hot + kNT - 1) / kNT), dim3(kNT), 0, s, z.hot_cols, z.n_hot, x,
                 z.xhot);
      ++n;
      launch_nz_main<true>(z, x, y, s);
    } else {
      launch_nz_main<false>(z, x, y, s);
    }
    ++n;
  }
  if (stage != 1 && z.T > 1) n += launch_fixup(z.carry_row, z.carry_val, z.T, y, 0, z.max_run, s);
  return n;
}

// ---- hot-x set (plan time) ------------------------------------------------------
// cnt[c] = number of nonzeros in column c
__global__ void col_count_kernel(const int32_t* __restrict__ col, int64_t nnz, int32_t* __restrict__ cnt) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < nnz; j += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(cnt + col[j], 1);
}
// H[min(cnt, HB-1)] += 1 over the columns
__global__ void count_hist_kernel(const int32_t* __restrict__ cnt, int64_t n, int32_t* __restrict__ H) {
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < n; c += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(H + (cnt[c] < kHotBuckets - 1 ? cnt[c] : kHotBuckets - 1), 1);
}
// per 1024-column block: number of columns with cnt >= t
__global__ void __launch_bounds__(1024) hot_flag_count_kernel(const int32_t* __restrict__ cnt, int64_t n, int32_t t,
                                                              int32_t* __restrict__ bsum) {
  const int64_t c = (int64_t)blockIdx.x * 1024 + threadIdx.x;
  const int f = c < n && cnt[c] >= t;
  const int wc = __popc(__ballot_sync(0xffffffffu, f));
  __shared__ int ws[32];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = wc;
  __syncthreads();
  if (threadIdx.x == 0) {
    int s = 0;
    for (int i = 0; i < 32; ++i) s += ws[i];
    bsum[blockIdx.x] = s;
  }
}
// ordered compaction: slot = exclusive rank among hot columns (column order);
// slots >= K are dropped
__global__ void __launch_bounds__(1024) hot_write_kernel(const int32_t* __restrict__ cnt, int64_t n, int32_t t,
                                                         const int32_t* __restrict__ boff, int K,
                                                         int32_t* __restrict__ hot_cols, int32_t* __restrict__ slot) {
  const int64_t c = (int64_t)blockIdx.x * 1024 + threadIdx.x;
  const int f = c < n && cnt[c] >= t;
  const unsigned m = __ballot_sync(0xffffffffu, f);
  __shared__ int ws[32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) ws[w] = __popc(m);
  __syncthreads();
  int pre = boff[blockIdx.x];
  for (int i = 0; i < w; ++i) pre += ws[i];
  pre += __popc(m & ((1u << lane) - 1u));
  if (c < n) slot[c] = (f && pre < K) ? pre : -1;
  if (f && pre < K) hot_cols[pre] = (int32_t)c;
}
// col[j] = ~slot[col[j]] for hot columns (in place, the plan's own copy)
__global__ void hot_encode_kernel(int32_t* __restrict__ col, int64_t nnz, const int32_t* __restrict__ slot) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < nnz; j += (int64_t)gridDim.x * blockDim.x) {
    const int32_t s = slot[col[j]];
    if (s >= 0) col[j] = ~s;
  }
}

void launch_col_counts(const int32_t* col, int64_t nnz, int64_t n_cols, int32_t* cnt, int32_t* H, cudaStream_t s) {
  cudaMemsetAsync(cnt, 0, (size_t)n_cols * 4, s);
  cudaMemsetAsync(H, 0, (size_t)kHotBuckets * 4, s);
  if (nnz > 0) col_count_kernel<<<dev_sm_count() * 16, kNT, 0, s>>>(col, nnz, cnt);
  if (n_cols > 0) count_hist_kernel<<<dev_sm_count() * 8, kNT, 0, s>>>(cnt, n_cols, H);
}
void launch_hot_flags(const int32_t* cnt, int64_t n_cols, int32_t t, int32_t* bsum, cudaStream_t s) {
  hot_flag_count_kernel<<<(int)((n_cols + 1023) / 1024), 1024, 0, s>>>(cnt, n_cols, t, bsum);
}
void launch_hot_write(const int32_t* cnt, int64_t n_cols, int32_t t, const int32_t* boff, int K, int32_t* hot_cols,
                      int32_t* slot, cudaStream_t s) {
  hot_write_kernel<<<(int)((n_cols + 1023) / 1024), 1024, 0, s>>>(cnt, n_cols, t, boff, K, hot_cols, slot);
}
void launch_hot_encode(int32_t* col, int64_t nnz, const int32_t* slot, cudaStream_t s) {
  if (nnz > 0) hot_encode_kernel<<<dev_sm_count() * 16, kNT, 0, s>>>(col, nnz, slot);
}

}  // namespace spmv
