// vector.cu -- csr_vector<VS>, long_row_split and the shared carry fix-up.
//
//  csr_vector<VS>  VS lanes per row, 4 independent accumulators per lane so
//                  each lane keeps 4 gathers in flight (CMP class: "inner loop
//                  unrolling + vectorization", P:629-630 / Table II)
//  long_row_split  csr_vector over short rows that skips long rows, then one
//                  CTA per C-nonzero chunk of each long row and an ordered
//                  per-row reduction of the chunk partials (IMB decomposition,
//                  P:608-621, Fig. 7 semantics per SURVEY 8(c3) #11).
// All sums are formed in an order fixed by the plan (deterministic).
#include "common.cuh"
#include "internal.h"

namespace spmv {

template <int VS, typename RP, bool SKIP_LONG>
__global__ void __launch_bounds__(kNT) vector_kernel(const RP* __restrict__ rp, const int32_t* __restrict__ col,
                                                     const double* __restrict__ val, const double* __restrict__ x,
                                                     double* __restrict__ y, int64_t m, int64_t l_split) {
  const int lane = threadIdx.x % VS;
  const int gi = (threadIdx.x & 31) / VS;
  const int64_t ngroups = (int64_t)gridDim.x * (kNT / VS);
  const int64_t wfirst = ((int64_t)blockIdx.x * kNT + (threadIdx.x & ~31)) / VS;
  for (int64_t rb = wfirst; rb < m; rb += ngroups) {
    const int64_t r = rb + gi;
    const bool active = r < m;
    int64_t a = 0, b = 0;
    if (active) { a = (int64_t)ld_ro(rp + r); b = (int64_t)ld_ro(rp + r + 1); }
    const bool skip = SKIP_LONG && (b - a > l_split);
    double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0, acc3 = 0.0;
    if (active && !skip) {
      int64_t j = a + lane;
      for (; j + 3 * VS < b; j += 4 * VS) {
        const int c0 = ld_stream(col + j), c1 = ld_stream(col + j + VS), c2 = ld_stream(col + j + 2 * VS),
                  c3 = ld_stream(col + j + 3 * VS);
        const double v0 = ld_stream(val + j), v1 = ld_stream(val + j + VS), v2 = ld_stream(val + j + 2 * VS),
                     v3 = ld_stream(val + j + 3 * VS);
        acc0 = fma(v0, ld_x(x + c0), acc0);
        acc1 = fma(v1, ld_x(x + c1), acc1);
        acc2 = fma(v2, ld_x(x + c2), acc2);
        acc3 = fma(v3, ld_x(x + c3), acc3);
      }
      for (; j < b; j += VS) acc0 = fma(ld_stream(val + j), ld_x(x + ld_stream(col + j)), acc0);
    }
    const double s = group_sum<VS>((acc0 + acc1) + (acc2 + acc3));
    if (active && !skip && lane == 0) y[r] = s;
  }
}

template <int VS, bool SKIP>
static void vector_dispatch_rp(const ExecArgs& a, int grid, cudaStream_t s) {
  if (a.A.rp_bytes == 8)
    vector_kernel<VS, int64_t, SKIP><<<grid, kNT, 0, s>>>((const int64_t*)a.A.rowptr, a.A.col, a.A.val, a.x, a.y,
                                                         a.A.m, a.l_split);
  else
    vector_kernel<VS, int32_t, SKIP><<<grid, kNT, 0, s>>>((const int32_t*)a.A.rowptr, a.A.col, a.A.val, a.x, a.y,
                                                         a.A.m, a.l_split);
}

template <bool SKIP>
static void vector_dispatch(const ExecArgs& a, int grid, cudaStream_t s) {
  switch (a.vs) {
    case 1: vector_dispatch_rp<1, SKIP>(a, grid, s); break;
    case 2: vector_dispatch_rp<2, SKIP>(a, grid, s); break;
    case 4: vector_dispatch_rp<4, SKIP>(a, grid, s); break;
    case 8: vector_dispatch_rp<8, SKIP>(a, grid, s); break;
    case 16: vector_dispatch_rp<16, SKIP>(a, grid, s); break;
    default: vector_dispatch_rp<32, SKIP>(a, grid, s); break;
  }
}

int launch_vector(const ExecArgs& a, bool skip_long, cudaStream_t s) {
  if (a.A.m == 0 || a.stage == 2) return 0;
  int64_t grid = (a.A.m * a.vs + kNT - 1) / kNT;
  const int64_t cap = (int64_t)a.sm_count * 8;
  if (grid > cap) grid = cap;
  if (grid < 1) grid = 1;
  if (skip_long) vector_dispatch<true>(a, (int)grid, s);
  else vector_dispatch<false>(a, (int)grid, s);
  return 1;
}

// ============================================================================
// carry fix-up (shared by STREAM, MERGE, SPLIT): for each maximal run of
// consecutive entries k..k' with the same row r >= 0, in increasing k:
// y[r] = (set ? 0 : y[r]) + (v_k + v_{k+1} + ... + v_k')
// ============================================================================
__global__ void __launch_bounds__(kNT) fixup_kernel(const int32_t* __restrict__ crow,
                                                    const double* __restrict__ cval, int64_t T,
                                                    double* __restrict__ y, int set) {
  const int64_t k = (int64_t)blockIdx.x * kNT + threadIdx.x;
  if (k >= T) return;
  const int32_t r = crow[k];
  if (r < 0) return;
  if (k > 0 && crow[k - 1] == r) return;
  double s = cval[k];
  for (int64_t q = k + 1; q < T && crow[q] == r; ++q) s += cval[q];
  y[r] = set ? s : y[r] + s;
}

void launch_fixup(const int32_t* crow, const double* cval, int64_t T, double* y, int set, cudaStream_t s) {
  fixup_kernel<<<(int)((T + kNT - 1) / kNT), kNT, 0, s>>>(crow, cval, T, y, set);
}

// ============================================================================
// long_row_split
// ============================================================================
// chunk c of the long-row table: row = long_rows[q] with chunk_start[q] <= c < chunk_start[q+1],
// nonzeros [rowptr[row] + (c - chunk_start[q])*chunk, min(.. + chunk, rowptr[row+1]))
template <typename RP>
__device__ __forceinline__ void chunk_range(const RP* rp, const int32_t* long_rows, const int64_t* chunk_start,
                                            int64_t n_long, int64_t chunk, int64_t c, int64_t& r, int64_t& b,
                                            int64_t& e) {
  int64_t lo = 0, hi = n_long - 1;  // last q with chunk_start[q] <= c
  while (lo < hi) {
    const int64_t mid = (lo + hi + 1) >> 1;
    if (chunk_start[mid] <= c) lo = mid; else hi = mid - 1;
  }
  r = long_rows[lo];
  b = (int64_t)rp[r] + (c - chunk_start[lo]) * chunk;
  const int64_t re = (int64_t)rp[r + 1];
  e = b + chunk < re ? b + chunk : re;
}

template <typename RP>
__global__ void chunk_export_kernel(const RP* __restrict__ rp, const int32_t* __restrict__ long_rows,
                                    const int64_t* __restrict__ chunk_start, int64_t n_long, int64_t chunk,
                                    int64_t n_chunks, int64_t* out) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n_chunks) return;
  int64_t r, b, e;
  chunk_range(rp, long_rows, chunk_start, n_long, chunk, c, r, b, e);
  out[c] = r;
  out[n_chunks + c] = b;
  out[2 * n_chunks + c] = e;
}

void launch_chunk_export(const ExecArgs& a, int64_t* out, cudaStream_t s) {
  if (a.n_chunks == 0) return;
  const int g = (int)((a.n_chunks + kNT - 1) / kNT);
  if (a.A.rp_bytes == 8)
    chunk_export_kernel<int64_t><<<g, kNT, 0, s>>>((const int64_t*)a.A.rowptr, a.long_rows, a.chunk_start, a.n_long,
                                                   a.chunk, a.n_chunks, out);
  else
    chunk_export_kernel<int32_t><<<g, kNT, 0, s>>>((const int32_t*)a.A.rowptr, a.long_rows, a.chunk_start, a.n_long,
                                                   a.chunk, a.n_chunks, out);
}

template <typename RP>
__global__ void __launch_bounds__(kNT) long_chunk_kernel(const RP* __restrict__ rp, const int32_t* __restrict__ col,
                                                         const double* __restrict__ val, const double* __restrict__ x,
                                                         const int32_t* __restrict__ long_rows,
                                                         const int64_t* __restrict__ chunk_start, int64_t n_long,
                                                         int64_t chunk, int32_t* __restrict__ crow,
                                                         double* __restrict__ cval) {
  const int64_t c = blockIdx.x;
  int64_t r, b, e;
  chunk_range(rp, long_rows, chunk_start, n_long, chunk, c, r, b, e);
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  int64_t j = b + threadIdx.x;
  for (; j + 3 * kNT < e; j += 4 * kNT) {
    const int c0 = ld_stream(col + j), c1 = ld_stream(col + j + kNT), c2 = ld_stream(col + j + 2 * kNT),
              c3 = ld_stream(col + j + 3 * kNT);
    const double v0 = ld_stream(val + j), v1 = ld_stream(val + j + kNT), v2 = ld_stream(val + j + 2 * kNT),
                 v3 = ld_stream(val + j + 3 * kNT);
    a0 = fma(v0, ld_x(x + c0), a0);
    a1 = fma(v1, ld_x(x + c1), a1);
    a2 = fma(v2, ld_x(x + c2), a2);
    a3 = fma(v3, ld_x(x + c3), a3);
  }
  for (; j < e; j += kNT) a0 = fma(ld_stream(val + j), ld_x(x + ld_stream(col + j)), a0);
  const double t = warp_sum((a0 + a1) + (a2 + a3));
  __shared__ double ws[kNT / 32];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = t;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < kNT / 32; ++w) s += ws[w];
    crow[c] = (int32_t)r;
    cval[c] = s;
  }
}

int launch_split(const ExecArgs& a, cudaStream_t s) {
  int n = 0;
  // 0. rows in no bin (empty rows) must read 0: clear y once
  if (a.zero_y && a.stage != 2 && a.A.m > 0) cudaMemsetAsync(a.y, 0, (size_t)a.A.m * 8, s);
  // 1. short / medium bins: cta_stream over each compacted bin (rows mapped
  //    back to y through the bin's row map); the bins own disjoint rows
  for (int b = 0; b < a.n_sp; ++b) n += launch_stream_plan(a.sp[b], a.x, a.y, a.stage, s);
  // 2. long rows: column-tiled (x blocks in smem) or nonzero chunks, then the
  //    ordered per-row reduction (sets y)
  if (a.long_tiled) return n + launch_long_tiled(a, s);
  if (a.n_chunks > 0) {
    if (a.stage != 2) {
      ++n;
      if (a.A.rp_bytes == 8)
        long_chunk_kernel<int64_t><<<(int)a.n_chunks, kNT, 0, s>>>((const int64_t*)a.A.rowptr, a.A.col, a.A.val,
                                                                   a.x, a.long_rows, a.chunk_start, a.n_long, a.chunk,
                                                                   a.chunk_row, a.chunk_val);
      else
        long_chunk_kernel<int32_t><<<(int)a.n_chunks, kNT, 0, s>>>((const int32_t*)a.A.rowptr, a.A.col, a.A.val,
                                                                   a.x, a.long_rows, a.chunk_start, a.n_long, a.chunk,
                                                                   a.chunk_row, a.chunk_val);
    }
    if (a.stage != 1) { launch_fixup(a.chunk_row, a.chunk_val, a.n_chunks, a.y, 1, s); ++n; }
  }
  return n;
}

}  // namespace spmv
