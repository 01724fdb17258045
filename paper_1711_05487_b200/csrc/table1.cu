// table1.cu -- the full Table I feature vector,
// computed on demand on the device (spmv_plan_table1): the Theta(N) row-span
// features bw / scatter and the Theta(NNZ) clustering / misses features the
// feature-guided selection does not need. One warp per row (grid-stride),
// per-warp partials in a fixed row order, summed by the host in warp order:
// deterministic. Readings: bw_i = last - first + 1 (inclusive,
// S:426); bw / scatter / clustering statistics over the non-empty rows (they
// are undefined for empty rows); misses_avg over all N rows (empty rows
// contribute 0); a miss is a gap > 16 doubles (one 128-B line, reading 13).
#include <algorithm>
#include <climits>
#include <cmath>
#include <vector>

#include "common.cuh"
#include "internal.h"

namespace spmv {

constexpr int kT1Threads = 256;

struct T1Part {
  double bw, bw2, sc, sc2, cl;
  long long bw_min, bw_max, nonempty, misses;
};

// PASS 0: sums; PASS 1: sums of squared deviations from the given averages
template <typename RP, int PASS>
__global__ void __launch_bounds__(kT1Threads) table1_kernel(const RP* __restrict__ rp, const int32_t* __restrict__ col,
                                                            int64_t m, int line, double bw_avg, double sc_avg,
                                                            const int32_t* __restrict__ hot_cols,
                                                            T1Part* __restrict__ part) {
  // (a plan with the hot-x table stores ~slot for hot columns: decode)
  auto colat = [&](int64_t j) -> int64_t {
    const int32_t c = ld_ro(col + j);
    return c >= 0 ? (int64_t)c : (int64_t)ld_ro(hot_cols + ~c);
  };
  const int lane = threadIdx.x & 31;
  const int64_t wid = ((int64_t)blockIdx.x * kT1Threads + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * kT1Threads) >> 5;
  T1Part a{0, 0, 0, 0, 0, LLONG_MAX, 0, 0, 0};
  for (int64_t r = wid; r < m; r += nw) {
    const int64_t s0 = (int64_t)ld_ro(rp + r), s1 = (int64_t)ld_ro(rp + r + 1);
    const int64_t len = s1 - s0;
    if (len == 0) continue;
    const int64_t bw = colat(s1 - 1) - colat(s0) + 1;
    const double sc = (double)len / (double)bw;
    if (PASS == 1) {
      const double d1 = (double)bw - bw_avg, d2 = sc - sc_avg;
      a.bw2 += d1 * d1;
      a.sc2 += d2 * d2;
      continue;
    }
    long long groups_gt1 = 0, miss = 0;  // non-head gaps > 1 (new group) and > line (miss)
    for (int64_t j = s0 + 1 + lane; j < s1; j += 32) {
      const int64_t g = colat(j) - colat(j - 1);
      groups_gt1 += g > 1;
      miss += g > line;
    }
    groups_gt1 = warp_sum(groups_gt1);
    miss = warp_sum(miss);
    a.bw += (double)bw;
    a.sc += sc;
    a.cl += (double)(1 + groups_gt1) / (double)len;
    a.bw_min = bw < a.bw_min ? bw : a.bw_min;
    a.bw_max = bw > a.bw_max ? bw : a.bw_max;
    a.nonempty += 1;
    a.misses += miss;
  }
  if (lane == 0) part[wid] = a;
}

template <typename RP>
static int table1_t(const MatView& A, const int32_t* hot_cols, int sm_count, int line, Table1& out,
                    cudaStream_t s) {
  const int grid = std::max(1, sm_count * 4);
  const int64_t nw = (int64_t)grid * (kT1Threads / 32);
  T1Part* part = nullptr;
  if (cudaMalloc(&part, (size_t)nw * sizeof(T1Part)) != cudaSuccess) return -1;
  std::vector<T1Part> h((size_t)nw);
  table1_kernel<RP, 0><<<grid, kT1Threads, 0, s>>>((const RP*)A.rowptr, A.col, A.m, line, 0.0, 0.0, hot_cols, part);
  cudaMemcpyAsync(h.data(), part, (size_t)nw * sizeof(T1Part), cudaMemcpyDeviceToHost, s);
  if (cudaStreamSynchronize(s) != cudaSuccess) {
    cudaFree(part);
    return -1;
  }
  double bw = 0, sc = 0, cl = 0;
  long long bmin = LLONG_MAX, bmax = 0, ne = 0, miss = 0;
  for (const auto& p : h) {  // warp order: deterministic
    bw += p.bw;
    sc += p.sc;
    cl += p.cl;
    bmin = std::min(bmin, p.bw_min);
    bmax = std::max(bmax, p.bw_max);
    ne += p.nonempty;
    miss += p.misses;
  }
  out.n_nonempty = ne;
  out.misses_total = miss;
  out.bw_min = ne ? (double)bmin : 0.0;
  out.bw_max = (double)bmax;
  out.bw_avg = ne ? bw / (double)ne : 0.0;
  out.scatter_avg = ne ? sc / (double)ne : 0.0;
  out.clustering_avg = ne ? cl / (double)ne : 0.0;
  table1_kernel<RP, 1><<<grid, kT1Threads, 0, s>>>((const RP*)A.rowptr, A.col, A.m, line, out.bw_avg,
                                                   out.scatter_avg, hot_cols, part);
  cudaMemcpyAsync(h.data(), part, (size_t)nw * sizeof(T1Part), cudaMemcpyDeviceToHost, s);
  const cudaError_t e = cudaStreamSynchronize(s);
  cudaFree(part);
  if (e != cudaSuccess) return -1;
  double bw2 = 0, sc2 = 0;
  for (const auto& p : h) {
    bw2 += p.bw2;
    sc2 += p.sc2;
  }
  out.bw_sd = ne ? std::sqrt(bw2 / (double)ne) : 0.0;
  out.scatter_sd = ne ? std::sqrt(sc2 / (double)ne) : 0.0;
  return 0;
}

int compute_table1(const MatView& A, const int32_t* hot_cols, int sm_count, Table1& out, cudaStream_t s) {
  if (A.m == 0) return 0;
  return A.rp_bytes == 8 ? table1_t<int64_t>(A, hot_cols, sm_count, 16, out, s)
                         : table1_t<int32_t>(A, hot_cols, sm_count, 16, out, s);
}

}  // namespace spmv
