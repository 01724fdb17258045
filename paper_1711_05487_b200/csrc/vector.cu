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
#include <cstdlib>

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
// ---- ordered carry fix-up ----------------------------------------------------
// T carries (row, value) in tile order; a run of equal consecutive rows holds
// the pieces of one row cut by tile edges. Each run is summed in order and
// added to (set = 0) or stored in (set = 1) y[row]; rows < 0 are no carry.
// Runs up to 2048 carries (plan-time bound max_run): fixup_seg_kernel, one
// launch. Longer runs (long rows cut into many tiles): a hierarchical
// reduce-by-key, 1024 carries per CTA (block segmented scan); runs cut by a
// CTA edge are passed up as (head, tail) pieces to the next level, stored
// after the T carries (fixup_capacity). Deterministic, no fp atomics.
constexpr int64_t kFixItems = 1024;  // carries per CTA (256 threads x 4)

int64_t fixup_capacity(int64_t T) {
  int64_t tot = T, n = T;
  while (n > kFixItems) {
    n = 2 * ((n + kFixItems - 1) / kFixItems);
    tot += n;
  }
  return tot > 1 ? tot : 1;
}

// one CTA of a reduce-by-key level: carries [b*1024, min(n, (b+1)*1024))
__device__ __forceinline__ void fixup_block(const int32_t* __restrict__ crow, const double* __restrict__ cval,
                                            int64_t n, int64_t blk, double* __restrict__ y, int set,
                                            int32_t* __restrict__ orow, double* __restrict__ oval) {
  __shared__ double wv[kNT / 32];
  __shared__ int wf[kNT / 32];
  __shared__ unsigned long long first_end;
  const int64_t bs = blk * kFixItems;
  const int64_t be = (bs + kFixItems) < n ? (bs + kFixItems) : n;
  const bool head_open = bs > 0 && __ldcg(crow + bs - 1) == __ldcg(crow + bs);
  const bool tail_open = be < n && __ldcg(crow + be) == __ldcg(crow + be - 1);
  if (threadIdx.x == 0) {
    first_end = (unsigned long long)(be - 1);
    if (orow) {
      orow[2 * blk] = -1;
      orow[2 * blk + 1] = -1;
      oval[2 * blk] = 0.0;
      oval[2 * blk + 1] = 0.0;
    }
  }
  __syncthreads();
  const int64_t i0 = bs + 4 * (int64_t)threadIdx.x;
  int32_t r[4];
  double v[4], inc[4];
  bool st[4], en[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int64_t i = i0 + u;
    const bool ok = i < be;
    r[u] = ok ? __ldcg(crow + i) : INT32_MIN;
    v[u] = ok ? __ldcg(cval + i) : 0.0;
    st[u] = ok && (i == bs || __ldcg(crow + i - 1) != r[u]);
    en[u] = ok && (i == be - 1 || __ldcg(crow + i + 1) != r[u]);
    if (en[u] && i < be - 1) atomicMin(&first_end, (unsigned long long)i);
  }
  // thread-local segmented inclusive sums
  double acc = 0.0;
  bool any = false;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    acc = st[u] ? v[u] : acc + v[u];
    any = any || st[u];
    inc[u] = acc;
  }
  // block exclusive segmented scan of (acc, any) over threads
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double S = acc;
  int f = any;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double su = __shfl_up_sync(0xffffffffu, S, o);
    const int fu = __shfl_up_sync(0xffffffffu, f, o);
    if (lane >= o) {
      if (!f) S += su;
      f |= fu;
    }
  }
  if (lane == 31) {
    wv[w] = S;
    wf[w] = f;
  }
  __syncthreads();
  double ex = __shfl_up_sync(0xffffffffu, S, 1);
  int exf = __shfl_up_sync(0xffffffffu, f, 1);
  if (lane == 0) {
    ex = 0.0;
    exf = 0;
  }
  // prefix from earlier warps (until a warp containing a run start)
  if (!exf) {
    double pre = 0.0;
    for (int q = w - 1; q >= 0; --q) {
      pre = wv[q] + pre;
      if (wf[q]) break;
    }
    ex = pre + ex;
  }
  const int64_t e1 = (int64_t)first_end;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    if (!en[u] || r[u] < 0) continue;
    const int64_t i = i0 + u;
    // inclusive run sum at i: items of the run inside this thread + the prefix
    // when the run started in an earlier thread
    bool started_here = false;
    for (int t = 0; t <= u; ++t) started_here = started_here || st[t];
    const double sum = started_here ? inc[u] : ex + inc[u];
    const bool in_first = i <= e1;  // the run holds item bs
    if (i == be - 1 && tail_open) {
      // continues into the next CTA; a run over the whole CTA fills both
      // slots (sum, +0.0) so the next level sees it contiguous with its
      // neighbours' pieces
      const bool whole = in_first && head_open;
      if (whole) {
        orow[2 * blk] = r[u];
        oval[2 * blk] = sum;
      }
      orow[2 * blk + 1] = r[u];
      oval[2 * blk + 1] = whole ? 0.0 : sum;
    } else if (in_first && head_open) {
      orow[2 * blk] = r[u];
      oval[2 * blk] = sum;
    } else {
      y[r[u]] = set ? sum : y[r[u]] + sum;
    }
  }
  __syncthreads();  // smem reuse by a following fixup_block in the same CTA
}

// level kernel; the last CTA to finish also runs the next level when it fits
// in one CTA (the usual case: saves a launch)
__global__ void __launch_bounds__(kNT) fixup_level_kernel(const int32_t* __restrict__ crow,
                                                          const double* __restrict__ cval, int64_t n,
                                                          double* __restrict__ y, int set,
                                                          int32_t* __restrict__ orow, double* __restrict__ oval,
                                                          unsigned int* __restrict__ done) {
  pdl_trigger();
  pdl_wait();
  fixup_block(crow, cval, n, blockIdx.x, y, set, orow, oval);
  const int64_t n2 = 2 * (int64_t)gridDim.x;
  if (!orow || !done || n2 > kFixItems) return;
  __shared__ int last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    last = atomicAdd(done, 1u) == gridDim.x - 1;
    if (last) *done = 0u;  // ready for the next launch
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  fixup_block(orow, oval, n2, 0, y, set, nullptr, nullptr);
}

// Runs up to kWarpRunMax carries (rows cut into at most that many tiles)
constexpr int64_t kWarpRunMax = 2048;

// Runs up to kWarpRunMax carries, one launch and no serial walk: each warp
// loads 32 consecutive carries, a segmented warp scan sums every run piece
// in it; a run that starts in the warp is written by its last lane there, or
// -- when it continues past the warp -- finished by the whole warp reading
// 256 carries per step. Pieces of runs that started in an earlier warp are
// left to that warp. Deterministic (fixed shuffle trees).
__global__ void __launch_bounds__(kNT) fixup_seg_kernel(const int32_t* __restrict__ crow,
                                                        const double* __restrict__ cval, int64_t T,
                                                        double* __restrict__ y, int set) {
  pdl_trigger();
  pdl_wait();
  const int64_t k = (int64_t)blockIdx.x * kNT + threadIdx.x;
  const int lane = threadIdx.x & 31;
  const int32_t r = k < T ? __ldcg(crow + k) : -1;
  const double v = k < T ? __ldcg(cval + k) : 0.0;
  int32_t prev = __shfl_up_sync(0xffffffffu, r, 1);
  if (lane == 0) prev = (k > 0 && k < T) ? __ldcg(crow + k - 1) : INT32_MIN;
  int32_t nxt = __shfl_down_sync(0xffffffffu, r, 1);
  if (lane == 31) nxt = (k + 1 < T) ? __ldcg(crow + k + 1) : INT32_MIN;
  double S = v;
  int f = r != prev;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double su = __shfl_up_sync(0xffffffffu, S, o);
    const int fu = __shfl_up_sync(0xffffffffu, f, o);
    if (lane >= o) {
      if (!f) S += su;
      f |= fu;
    }
  }
  const bool own = r >= 0 && f;  // the run piece started inside this warp
  if (own && nxt != r) y[r] = set ? S : y[r] + S;
  const bool open = __shfl_sync(0xffffffffu, own && nxt == r, 31);  // lane 31's run goes on
  if (!open) return;
  const int32_t rr = __shfl_sync(0xffffffffu, r, 31);
  const double s31 = __shfl_sync(0xffffffffu, S, 31);
  double acc = lane == 0 ? s31 : 0.0;
  for (int64_t base = k - lane + 32;; base += 256) {
    int32_t cr[8];
    double cv[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int64_t q = base + u * 32 + lane;
      cr[u] = q < T ? __ldcg(crow + q) : -1;
      cv[u] = q < T ? __ldcg(cval + q) : 0.0;
    }
    bool all = true;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      acc += cr[u] == rr ? cv[u] : 0.0;
      all = all && cr[u] == rr;
    }
    if (!__all_sync(0xffffffffu, all)) break;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) y[rr] = set ? acc : y[rr] + acc;
}

// Carries [0, T) of a tile RANGE (pointers offset by the range start): always
// the single-launch forward walk, which needs no scratch -- the hierarchical
// path keeps its levels and counter after the plan's T carries, i.e. inside
// the next range's carries when called with offset pointers. A run of any
// length is summed by one warp walking it 256 carries per step.
int launch_fixup_range(const int32_t* crow, const double* cval, int64_t T, double* y, cudaStream_t s) {
  if (T <= 0) return 0;
  launch_pdl(fixup_seg_kernel, dim3((unsigned)((T + kNT - 1) / kNT)), dim3(kNT), 0, s, crow, cval, T, y, 0);
  return 1;
}

int launch_fixup(int32_t* crow, double* cval, int64_t T, double* y, int set, int64_t max_run, cudaStream_t s) {
  if (T <= 0) return 0;
  if (max_run <= kWarpRunMax) {
    launch_pdl(fixup_seg_kernel, dim3((unsigned)((T + kNT - 1) / kNT)), dim3(kNT), 0, s, (const int32_t*)crow,
               (const double*)cval, T, y, set);
    return 1;
  }
  unsigned int* done = reinterpret_cast<unsigned int*>(crow + fixup_capacity(T));
  int launches = 0;
  int64_t n = T;
  int32_t* cr = crow;
  double* cv = cval;
  int64_t off = T;
  for (;;) {
    const int64_t nb = (n + kFixItems - 1) / kFixItems;
    int32_t* orow = nb > 1 ? crow + off : nullptr;
    double* oval = nb > 1 ? cval + off : nullptr;
    launch_pdl(fixup_level_kernel, dim3((unsigned)nb), dim3(kNT), 0, s, (const int32_t*)cr, (const double*)cv, n, y,
               set, orow, oval, done);
    ++launches;
    if (nb == 1 || 2 * nb <= kFixItems) break;  // the last CTA ran the final level
    cr = orow;
    cv = oval;
    n = 2 * nb;
    off += n;
  }
  return launches;
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

static int diag_skip() {  // diagnostics only (SPMV_DIAG_SKIP=1: no long rows, 2: no bins); y is then wrong
  static int v = [] { const char* e = getenv("SPMV_DIAG_SKIP"); return e ? atoi(e) : 0; }();
  return v;
}

int launch_split(const ExecArgs& a, cudaStream_t s) {
  static const bool pdlconc = getenv("SPMV_SPLIT_PDLCONC") && atoi(getenv("SPMV_SPLIT_PDLCONC")) != 0;  // experiment
  if (pdlconc && a.use_nz && a.long_tiled && !a.long_tma && a.n_long > 0 && a.nz.T > 0 && !a.nz.memset_y &&
      a.nz.n_hot == 0 && diag_skip() == 0) {
    // one stream, no fork: the long rows' persistent grid first (PDL; it
    // waits for the previous SpMV, then triggers), the short-row bin behind
    // it with PDL and no wait of its own, so both grids share the SMs; the
    // bin's fix-up (PDL, waits for the bin), then the long-row reduction as
    // a plain launch (waits for everything before it)
    int n = 0;
    if (a.stage != 2) {
      launch_long_tiled(a, 3, s);
      ++n;
      NzPlan z = a.nz;
      z.skip_wait = true;
      n += launch_nz_plan(z, a.x, a.y, 1, s);
    }
    if (a.stage != 1) {
      n += launch_nz_plan(a.nz, a.x, a.y, 2, s);
      launch_long_tiled(a, 2, s);
      ++n;
    }
    return n;
  }
  if (a.split_fused && a.use_nz && a.long_tiled && a.n_long > 0 && a.nz.T > 0 && diag_skip() == 0)
    return launch_split_fused(a, s);
  int n = 0;
  const bool longs = a.n_long > 0 && (a.long_tiled || a.n_chunks > 0) && diag_skip() != 1;
  // 0. rows in no bin must read 0: legacy stream bins (empty rows), or an
  //    nnz_split bin without nonzeros
  if (a.stage != 2 && a.A.m > 0 && ((!a.use_nz && a.zero_y) || (a.use_nz && a.nz.T == 0)))
    cudaMemsetAsync(a.y, 0, (size_t)a.A.m * 8, s);
  // 1. long rows (column-tiled x blocks or nonzero chunks) and their ordered
  //    per-row reduction run on the side stream, concurrently with the bins
  //    (gather-bound bins + stream-bound long rows overlap); the bins never
  //    write the long rows' y
  const bool conc = longs && a.side;
  cudaStream_t ls = conc ? a.side : s;
  if (conc) {
    cudaEventRecord(a.ev_fork, s);
    cudaStreamWaitEvent(a.side, a.ev_fork, 0);
  }
  if (longs && a.stage != 2) {
    ++n;
    if (a.long_tma && ((uintptr_t)a.x & 15) == 0) launch_long_tma(a, a.sm_count, ls);
    else if (a.long_tiled) launch_long_tiled(a, 1, ls);
    else if (a.A.rp_bytes == 8)
      long_chunk_kernel<int64_t><<<(int)a.n_chunks, kNT, 0, ls>>>((const int64_t*)a.A.rowptr, a.A.col, a.A.val,
                                                                  a.x, a.long_rows, a.chunk_start, a.n_long, a.chunk,
                                                                  a.chunk_row, a.chunk_val);
    else
      long_chunk_kernel<int32_t><<<(int)a.n_chunks, kNT, 0, ls>>>((const int32_t*)a.A.rowptr, a.A.col, a.A.val,
                                                                  a.x, a.long_rows, a.chunk_start, a.n_long, a.chunk,
                                                                  a.chunk_row, a.chunk_val);
  }
  if (longs && a.stage != 1) {
    if (a.long_tiled) {
      launch_long_tiled(a, 2, ls);
      ++n;
    } else {
      n += launch_fixup(a.chunk_row, a.chunk_val, a.n_chunks, a.y, 1, (a.nnz_max + a.chunk - 1) / a.chunk, ls);
    }
  }
  if (conc) cudaEventRecord(a.ev_join, ls);
  // 2. short / medium rows: one nnz_split bin, or cta_stream length bins
  //    (rows mapped back to y through the bin's row map; disjoint rows)
  if (diag_skip() == 2) {
  } else if (a.use_nz) {
    n += launch_nz_plan(a.nz, a.x, a.y, a.stage, s);
  } else {
    for (int b = 0; b < a.n_sp; ++b) n += launch_stream_plan(a.sp[b], a.x, a.y, a.stage, s);
  }
  if (conc) cudaStreamWaitEvent(s, a.ev_join, 0);
  return n;
}

// NNZSPLIT: one nnz_split pass over the whole shard
int launch_nzsplit(const ExecArgs& a, cudaStream_t s) { return launch_nz_plan(a.nz, a.x, a.y, a.stage, s); }

}  // namespace spmv
