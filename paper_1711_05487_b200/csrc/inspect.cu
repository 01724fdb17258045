// inspect.cu -- the plan-time inspector on the device.
//
//  K0 rowstats       Theta(N) features of Table I over rowptr, the
//                    rowptr invariants and the row-head bitmap
//  K1 validate_gaps  colind range / strict order, max in-row gap
//                    (needed for the 16-bit delta width) and the
//                    Table I misses count, one pass over colind
//  K2 tile_rows      per-CTA nnz tiles: R_k = lower_bound(rowptr, k*C)
//                    (nnz-balanced partition of P:708-711 at CTA granularity)
//     merge_splits   merge-path diagonals (IMB "auto" analogue)
//     long_rows      ordered long-row list + chunk prefix (decomposition)
//  K3 d16_encode     delta colind + heads + tile anchors (MB)
//
// Every accumulator is an integer, so atomics give order-independent
// (deterministic) results.
#include <climits>
#include "common.cuh"
#include "internal.h"

namespace spmv {

// ---- distinct row-relative deltas (D8 dictionary, reading 26) ----
// per-CTA open-addressing set in smem (INT32_MIN = empty), merged into the
// global table at the end; gives up (over) past kD8Max distinct values
constexpr int kDSet = 512;
struct DeltaSet {
  int32_t tab[kDSet];
  int count, over;
};
__device__ __forceinline__ void dset_init(DeltaSet& ds) {
  for (int i = threadIdx.x; i < kDSet; i += blockDim.x) ds.tab[i] = INT32_MIN;
  if (threadIdx.x == 0) ds.count = ds.over = 0;
}
__device__ __forceinline__ void dset_insert(DeltaSet& ds, int64_t v64, int32_t& last) {
  if (v64 <= INT32_MIN || v64 > INT32_MAX) { ds.over = 1; return; }
  const int32_t v = (int32_t)v64;
  if (v == last || ds.over) return;
  last = v;
  uint32_t h = ((uint32_t)v * 2654435761u) >> 23;  // 9 bits
  for (int probe = 0; probe < kDSet; ++probe, h = (h + 1) & (kDSet - 1)) {
    const int32_t cur = ds.tab[h];
    if (cur == v) return;
    if (cur == INT32_MIN) {
      const int32_t prev = atomicCAS(&ds.tab[h], INT32_MIN, v);
      if (prev == INT32_MIN) {
        if (atomicAdd(&ds.count, 1) >= kD8Max) ds.over = 1;
        return;
      }
      if (prev == v) return;
    }
  }
  ds.over = 1;
}
// after a __syncthreads: the CTA's set into st->dtab
__device__ __forceinline__ void dset_merge(DeltaSet& ds, DevStats* st) {
  if (ds.over) {
    if (threadIdx.x == 0) st->d_over = 1;
    return;
  }
  for (int i = threadIdx.x; i < kDSet; i += blockDim.x) {
    const int32_t v = ds.tab[i];
    if (v == INT32_MIN) continue;
    uint32_t h = ((uint32_t)v * 2654435761u) >> 22;  // 10 bits
    int probe = 0;
    for (; probe < kDTab; ++probe, h = (h + 1) & (kDTab - 1)) {
      const int32_t prev = atomicCAS(&st->dtab[h], INT32_MIN, v);
      if (prev == INT32_MIN) {
        if (atomicAdd(&st->d_count, 1) >= kD8Max) st->d_over = 1;
        break;
      }
      if (prev == v) break;
    }
    if (probe == kDTab) st->d_over = 1;
  }
}

template <typename RP>
__global__ void __launch_bounds__(kNT) rowstats_kernel(const RP* __restrict__ rp, const int32_t* __restrict__ col,
                                                       int64_t m, int64_t nnz, int64_t l_split, int64_t row0,
                                                       uint32_t* __restrict__ headbits, DevStats* st) {
  __shared__ DeltaSet ds;
  dset_init(ds);
  __syncthreads();
  int32_t last = INT32_MIN;
  unsigned long long s1 = 0, s2 = 0, s1s = 0, s2s = 0;
  long long mn = LLONG_MAX, mx = 0, ne = 0, nl = 0, nnzl = 0, ns = 0, mxs = 0, err = LLONG_MAX;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += stride) {
    const int64_t a = (int64_t)rp[i], b = (int64_t)rp[i + 1];
    const long long len = b - a;
    if (len < 0) { err = err < i ? err : i; continue; }
    const unsigned long long ul = (unsigned long long)len;
    s1 += ul; s2 += ul * ul;
    mn = len < mn ? len : mn;
    mx = len > mx ? len : mx;
    ne += (len == 0);
    if (len > l_split) { nl++; nnzl += len; }
    else { ns++; s1s += ul; s2s += ul * ul; mxs = len > mxs ? len : mxs; }
    if (len > 0 && a >= 0 && a < nnz) {
      atomicOr(&headbits[a >> 5], 1u << (a & 31));
      dset_insert(ds, (int64_t)col[a] - (row0 + i), last);  // head delta
    }
  }
  __syncthreads();
  dset_merge(ds, st);
  s1 = warp_sum(s1); s2 = warp_sum(s2); s1s = warp_sum(s1s); s2s = warp_sum(s2s);
  ne = warp_sum(ne); nl = warp_sum(nl); nnzl = warp_sum(nnzl); ns = warp_sum(ns);
  mn = warp_min(mn); mx = warp_max(mx); mxs = warp_max(mxs); err = warp_min(err);
  if ((threadIdx.x & 31) == 0) {
    if (s1) atomicAdd(&st->s1, s1);
    if (s2) atomicAdd(&st->s2, s2);
    if (s1s) atomicAdd(&st->s1_short, s1s);
    if (s2s) atomicAdd(&st->s2_short, s2s);
    if (ne) atomicAdd((unsigned long long*)&st->n_empty, (unsigned long long)ne);
    if (nl) atomicAdd((unsigned long long*)&st->n_long, (unsigned long long)nl);
    if (nnzl) atomicAdd((unsigned long long*)&st->nnz_long, (unsigned long long)nnzl);
    if (ns) atomicAdd((unsigned long long*)&st->n_short, (unsigned long long)ns);
    atomicMin(&st->nnz_min, mn);
    atomicMax(&st->nnz_max, mx);
    atomicMax(&st->max_short, mxs);
    if (err != LLONG_MAX) atomicMin(&st->rp_err, err);
  }
}

__global__ void __launch_bounds__(kNT) validate_gaps_kernel(const int32_t* __restrict__ col, int64_t nnz,
                                                            int64_t n_cols, const uint32_t* __restrict__ headbits,
                                                            DevStats* st) {
  // distinct large gaps (>= kEsc0): deduplicated in a per-CTA smem set first
  // (a stencil repeats a handful of values ~2x per row), merged at the end
  __shared__ int32_t tab[kBigTab];
  __shared__ int over;
  __shared__ DeltaSet ds;
  for (int i = threadIdx.x; i < kBigTab; i += blockDim.x) tab[i] = 0;
  if (threadIdx.x == 0) over = 0;
  dset_init(ds);
  __syncthreads();
  int32_t last = INT32_MIN;
  long long mg = 0, miss = 0, err = LLONG_MAX, cmin = LLONG_MAX, cmax = -1;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < nnz; j += stride) {
    const int64_t c = col[j];
    if (c < 0 || c >= n_cols) { long long k = 2 * j; err = k < err ? k : err; continue; }
    cmin = c < cmin ? c : cmin;
    cmax = c > cmax ? c : cmax;
    const bool head = (headbits[j >> 5] >> (j & 31)) & 1u;
    if (!head && j > 0) {
      const int64_t g = c - (int64_t)col[j - 1];
      if (g <= 0) { long long k = 2 * j + 1; err = k < err ? k : err; continue; }
      mg = g > mg ? g : mg;
      miss += (g > 16);
      dset_insert(ds, g, last);  // in-row gap
      if (g >= kEsc0) {
        const int32_t v = (int32_t)g;
        uint32_t h = ((uint32_t)v * 2654435761u) % kBigTab;
        for (int probe = 0;; ++probe, h = (h + 1) % kBigTab) {
          if (probe == kBigTab) { over = 1; break; }
          const int32_t cur = tab[h];
          if (cur == v) break;
          if (cur == 0) {
            const int32_t prev = atomicCAS(&tab[h], 0, v);
            if (prev == 0 || prev == v) break;
          }
        }
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kBigTab; i += blockDim.x) {
    const int32_t v = tab[i];
    if (v == 0) continue;
    uint32_t h = ((uint32_t)v * 2654435761u) % kBigTab;
    for (int probe = 0;; ++probe, h = (h + 1) % kBigTab) {
      if (probe == kBigTab) { st->big_over = 1; break; }
      const int32_t prev = atomicCAS(&st->bigtab[h], 0, v);
      if (prev == 0 || prev == v) break;
    }
  }
  if (threadIdx.x == 0 && over) st->big_over = 1;
  dset_merge(ds, st);
  mg = warp_max(mg); miss = warp_sum(miss); err = warp_min(err);
  cmin = warp_min(cmin); cmax = warp_max(cmax);
  if ((threadIdx.x & 31) == 0) {
    if (cmin != LLONG_MAX) atomicMin(&st->col_min, cmin);
    if (cmax >= 0) atomicMax(&st->col_max, cmax);
    if (mg) atomicMax(&st->maxgap, mg);
    if (miss) atomicAdd((unsigned long long*)&st->misses, (unsigned long long)miss);
    if (err != LLONG_MAX) atomicMin(&st->col_err, err);
  }
}

static int grid_for(int64_t work, int per_cta_min = kNT) {
  int64_t g = (work + per_cta_min - 1) / per_cta_min;
  if (g < 1) g = 1;
  if (g > dev_sm_count() * 16) g = dev_sm_count() * 16;
  return (int)g;
}

void launch_rowstats(const MatView& A, int64_t l_split, int64_t row0, uint32_t* headbits, DevStats* st,
                     cudaStream_t s) {
  const int g = grid_for(A.m);
  if (A.m == 0) return;
  if (A.rp_bytes == 8)
    rowstats_kernel<int64_t><<<g, kNT, 0, s>>>((const int64_t*)A.rowptr, A.col, A.m, A.nnz, l_split, row0, headbits,
                                               st);
  else
    rowstats_kernel<int32_t><<<g, kNT, 0, s>>>((const int32_t*)A.rowptr, A.col, A.m, A.nnz, l_split, row0, headbits,
                                               st);
}

void launch_validate_gaps(const MatView& A, const uint32_t* headbits, DevStats* st, cudaStream_t s) {
  if (A.nnz == 0) return;
  validate_gaps_kernel<<<grid_for(A.nnz), kNT, 0, s>>>(A.col, A.nnz, A.n_cols, headbits, st);
}

// x-line reuse probe (plan-time heuristic for the nnz_split gather cache
// mode): kReuseRows rows sampled (all rows when fewer), a warp per row r >= 1, up to 256
// nonzeros of r each; hit when row r-1 holds a column in the same 16-column
// (128-B) line -- the L1 reuse a row-ordered sweep can expect
constexpr int64_t kReuseRows = 4096;
template <typename RP>
__global__ void x_reuse_kernel(const RP* __restrict__ rp, const int32_t* __restrict__ col, int64_t m,
                               DevStats* st) {
  const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t S = (m - 1) < kReuseRows ? (m - 1) : kReuseRows;
  if (wid >= S) return;
  // pseudo-random rows (splitmix64 of the warp id): evenly spaced rows alias
  // with structured matrices (C2: rows 512w all sit on a 16-column line edge)
  uint64_t z = (uint64_t)wid + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z ^= z >> 31;
  const int64_t r = S == m - 1 ? 1 + wid : 1 + (int64_t)(z % (uint64_t)(m - 1));
  const int64_t a0 = rp[r - 1], a1 = rp[r], b0 = a1, b1 = rp[r + 1];
  const int64_t nb = (b1 - b0) < 256 ? (b1 - b0) : 256;
  unsigned hit = 0, tot = 0;
  for (int64_t j = lane; j < nb; j += 32) {
    const int64_t line0 = ((int64_t)col[b0 + j] >> 4) << 4;
    int64_t lo = a0, hi = a1;  // first column >= line0 in row r-1
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (col[mid] < line0) lo = mid + 1;
      else hi = mid;
    }
    hit += (lo < a1 && col[lo] < line0 + 16) ? 1u : 0u;
    ++tot;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    hit += __shfl_xor_sync(0xffffffffu, hit, o);
    tot += __shfl_xor_sync(0xffffffffu, tot, o);
  }
  if (lane == 0 && tot) {
    atomicAdd(&st->reuse_hit, (unsigned long long)hit);
    atomicAdd(&st->reuse_tot, (unsigned long long)tot);
  }
}

void launch_x_reuse(const MatView& A, DevStats* st, cudaStream_t s) {
  if (A.m < 2 || A.nnz == 0) return;
  const int64_t S = (A.m - 1) < kReuseRows ? (A.m - 1) : kReuseRows;
  const int g = (int)((S * 32 + kNT - 1) / kNT);
  if (A.rp_bytes == 8)
    x_reuse_kernel<int64_t><<<g, kNT, 0, s>>>((const int64_t*)A.rowptr, A.col, A.m, st);
  else
    x_reuse_kernel<int32_t><<<g, kNT, 0, s>>>((const int32_t*)A.rowptr, A.col, A.m, st);
}

// ---- K2: tiles, merge splits -------------------------------------------------
template <typename RP>
__global__ void tile_rows_kernel(const RP* __restrict__ rp, int64_t m, int64_t C, int64_t T,
                                 int32_t* __restrict__ tile_row, DevStats* st) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k > T) return;
  int64_t R;
  if (k == 0) R = 0;
  else if (k == T) R = m;
  else { R = lower_bound_dev(rp, 0, m, k * C); R = R > m ? m : R; }
  tile_row[k] = (int32_t)R;
  // tile k (< T) has an incoming row iff rowptr[R_k] > k*C
  if (k < T && (int64_t)rp[R] > k * C) atomicAdd((unsigned long long*)&st->n_incoming, 1ull);
}

void launch_tile_rows(const MatView& A, int64_t C, int64_t T, int32_t* tile_row, DevStats* st, cudaStream_t s) {
  const int g = (int)((T + 1 + kNT - 1) / kNT);
  if (A.rp_bytes == 8)
    tile_rows_kernel<int64_t><<<g, kNT, 0, s>>>((const int64_t*)A.rowptr, A.m, C, T, tile_row, st);
  else
    tile_rows_kernel<int32_t><<<g, kNT, 0, s>>>((const int32_t*)A.rowptr, A.m, C, T, tile_row, st);
}

// split(d) = (i, d-i): binary search over [max(0,d-nnz), min(d,m)] advancing
// while rowptr[mid+1] <= d-mid-1 (row end precedes the nonzero, ties to rows)
template <typename RP>
__global__ void merge_splits_kernel(const RP* __restrict__ rp, int64_t m, int64_t nnz, int64_t items, int64_t T,
                                    int32_t* __restrict__ mrow, int64_t* __restrict__ mnnz) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k > T) return;
  int64_t d = k * items;
  if (d > m + nnz) d = m + nnz;
  int64_t lo = d - nnz > 0 ? d - nnz : 0, hi = d < m ? d : m;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if ((int64_t)rp[mid + 1] <= d - mid - 1) lo = mid + 1; else hi = mid;
  }
  mrow[k] = (int32_t)lo;
  mnnz[k] = d - lo;
}

void launch_merge_splits(const MatView& A, int64_t items, int64_t T, int32_t* mrow, int64_t* mnnz, cudaStream_t s) {
  const int g = (int)((T + 1 + kNT - 1) / kNT);
  if (A.rp_bytes == 8)
    merge_splits_kernel<int64_t><<<g, kNT, 0, s>>>((const int64_t*)A.rowptr, A.m, A.nnz, items, T, mrow, mnnz);
  else
    merge_splits_kernel<int32_t><<<g, kNT, 0, s>>>((const int32_t*)A.rowptr, A.m, A.nnz, items, T, mrow, mnnz);
}

// ---- long rows: ordered compaction (count / scan / write) -------------------
template <typename RP>
__device__ __forceinline__ bool is_long(const RP* rp, int64_t i, int64_t l_split) {
  return (int64_t)rp[i + 1] - (int64_t)rp[i] > l_split;
}

template <typename RP>
__global__ void __launch_bounds__(kNT) long_count_kernel(const RP* __restrict__ rp, int64_t m, int64_t l_split,
                                                         int64_t rows_per_cta, int32_t* __restrict__ counts) {
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_cta;
  const int64_t r1 = r0 + rows_per_cta < m ? r0 + rows_per_cta : m;
  int c = 0;
  for (int64_t i = r0 + threadIdx.x; i < r1; i += kNT) c += is_long(rp, i, l_split);
  c = warp_sum(c);
  __shared__ int ws[kNT / 32];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int w = 0; w < kNT / 32; ++w) t += ws[w];
    counts[blockIdx.x] = t;
  }
}

// single-CTA exclusive scan of n int64 values given by f(i), written to out[0..n]
template <typename F>
__device__ void cta_exclusive_scan(int64_t n, F f, int64_t* out) {
  __shared__ int64_t wsum[kNT / 32];
  __shared__ int64_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int64_t base = 0; base < n; base += kNT) {
    const int64_t i = base + threadIdx.x;
    const int64_t v = i < n ? f(i) : 0;
    int64_t inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int64_t t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    if (lane == 31) wsum[w] = inc;
    __syncthreads();
    int64_t wpre = 0;
    for (int q = 0; q < w; ++q) wpre += wsum[q];
    if (i < n) out[i] = carry + wpre + inc - v;
    __syncthreads();
    if (threadIdx.x == kNT - 1) carry += wpre + inc;
    __syncthreads();
  }
  if (threadIdx.x == 0) out[n] = carry;
}

__global__ void __launch_bounds__(kNT) scan_counts_kernel(const int32_t* counts, int64_t nb, int64_t* offs) {
  cta_exclusive_scan(nb, [&](int64_t i) { return (int64_t)counts[i]; }, offs);
}

template <typename RP>
__global__ void __launch_bounds__(kNT) long_write_kernel(const RP* __restrict__ rp, int64_t m, int64_t l_split,
                                                         int64_t rows_per_cta, const int64_t* __restrict__ offs,
                                                         int32_t* __restrict__ long_rows) {
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_cta;
  const int64_t r1 = r0 + rows_per_cta < m ? r0 + rows_per_cta : m;
  __shared__ int wcnt[kNT / 32];
  __shared__ int64_t base;
  if (threadIdx.x == 0) base = offs[blockIdx.x];
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int64_t b = r0; b < r1; b += kNT) {
    const int64_t i = b + threadIdx.x;
    const bool f = i < r1 && is_long(rp, i, l_split);
    const unsigned bal = __ballot_sync(0xffffffffu, f);
    if (lane == 0) wcnt[w] = __popc(bal);
    __syncthreads();
    int pre = 0;
    for (int q = 0; q < w; ++q) pre += wcnt[q];
    if (f) long_rows[base + pre + __popc(bal & ((1u << lane) - 1))] = (int32_t)i;
    __syncthreads();
    if (threadIdx.x == 0) { int t = 0; for (int q = 0; q < kNT / 32; ++q) t += wcnt[q]; base += t; }
    __syncthreads();
  }
}

template <typename RP>
__global__ void __launch_bounds__(kNT) chunk_prefix_kernel(const RP* __restrict__ rp, const int32_t* long_rows,
                                                           int64_t n_long, int64_t chunk, int64_t* chunk_start) {
  cta_exclusive_scan(n_long, [&](int64_t q) {
    const int64_t r = long_rows[q];
    const int64_t len = (int64_t)rp[r + 1] - (int64_t)rp[r];
    return (len + chunk - 1) / chunk;
  }, chunk_start);
}

void launch_long_rows(const MatView& A, int64_t l_split, int64_t chunk, int32_t* long_rows, int64_t n_long,
                      int64_t* chunk_start, int32_t* scratch_counts, int nb, cudaStream_t s) {
  // scratch_counts: nb int32 counts followed by (nb+1) int64 offsets (8-B aligned by the caller)
  const int64_t rpc = (A.m + nb - 1) / nb;
  int64_t* offs = reinterpret_cast<int64_t*>(scratch_counts + ((nb + 1) & ~1));
  if (A.rp_bytes == 8) {
    auto rp = (const int64_t*)A.rowptr;
    long_count_kernel<<<nb, kNT, 0, s>>>(rp, A.m, l_split, rpc, scratch_counts);
    scan_counts_kernel<<<1, kNT, 0, s>>>(scratch_counts, nb, offs);
    long_write_kernel<<<nb, kNT, 0, s>>>(rp, A.m, l_split, rpc, offs, long_rows);
    chunk_prefix_kernel<<<1, kNT, 0, s>>>(rp, long_rows, n_long, chunk, chunk_start);
  } else {
    auto rp = (const int32_t*)A.rowptr;
    long_count_kernel<<<nb, kNT, 0, s>>>(rp, A.m, l_split, rpc, scratch_counts);
    scan_counts_kernel<<<1, kNT, 0, s>>>(scratch_counts, nb, offs);
    long_write_kernel<<<nb, kNT, 0, s>>>(rp, A.m, l_split, rpc, offs, long_rows);
    chunk_prefix_kernel<<<1, kNT, 0, s>>>(rp, long_rows, n_long, chunk, chunk_start);
  }
}

// ---- K3: delta colind ------------------------------------------------------------
// dcol[j] = colind[j] - colind[j-1] for non-head j, 0 at row heads;
// head[i] = colind[rowptr[i]] or n_cols for an empty row; anchor[k] = colind[k*C].
__global__ void __launch_bounds__(kNT) d16_dcol_kernel(const int32_t* __restrict__ col, int64_t nnz,
                                                       const uint32_t* __restrict__ headbits, uint16_t* dcol,
                                                       const int32_t* __restrict__ esc, int n_esc) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < nnz; j += stride) {
    const bool h = (headbits[j >> 5] >> (j & 31)) & 1u;
    int32_t d = h ? 0 : col[j] - col[j - 1];
    if (d >= kEsc0) {  // escape code: index in the sorted table
      int lo = 0, hi = n_esc - 1;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (esc[mid] < d) lo = mid + 1; else hi = mid;
      }
      d = kEsc0 + lo;
    }
    dcol[j] = (uint16_t)d;
  }
}
template <typename RP>
__global__ void __launch_bounds__(kNT) d16_head_kernel(const RP* __restrict__ rp, const int32_t* __restrict__ col,
                                                       int64_t m, int64_t n_cols, int32_t* head) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += stride) {
    const int64_t a = rp[i], b = rp[i + 1];
    head[i] = b > a ? col[a] : (int32_t)n_cols;
  }
}
__global__ void d16_anchor_kernel(const int32_t* __restrict__ col, int64_t nnz, int64_t C, int64_t T, int32_t* anchor) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < T) anchor[k] = k * C < nnz ? col[k * C] : 0;
}

void launch_d16_encode(const MatView& A, const uint32_t* headbits, int64_t C, int64_t T, uint16_t* dcol,
                       int32_t* head, int32_t* anchor, const int32_t* esc_dev, int n_esc, cudaStream_t s) {
  if (A.nnz) d16_dcol_kernel<<<grid_for(A.nnz), kNT, 0, s>>>(A.col, A.nnz, headbits, dcol, esc_dev, n_esc);
  if (A.m) {
    if (A.rp_bytes == 8)
      d16_head_kernel<int64_t><<<grid_for(A.m), kNT, 0, s>>>((const int64_t*)A.rowptr, A.col, A.m, A.n_cols, head);
    else
      d16_head_kernel<int32_t><<<grid_for(A.m), kNT, 0, s>>>((const int32_t*)A.rowptr, A.col, A.m, A.n_cols, head);
  }
  d16_anchor_kernel<<<(int)((T + kNT - 1) / kNT), kNT, 0, s>>>(A.col, A.nnz, C, T, anchor);
}

// rowptr slice of a shard: subtract the shard's first offset
template <typename RP>
__global__ void rebase_kernel(RP* rp, int64_t count, int64_t base) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) rp[i] = (RP)(rp[i] - base);
}

void launch_rebase(void* rowptr, int rp_bytes, int64_t count, int64_t base, cudaStream_t s) {
  if (base == 0 || count == 0) return;
  if (rp_bytes == 8) rebase_kernel<int64_t><<<grid_for(count), kNT, 0, s>>>((int64_t*)rowptr, count, base);
  else rebase_kernel<int32_t><<<grid_for(count), kNT, 0, s>>>((int32_t*)rowptr, count, base);
}

}  // namespace spmv
