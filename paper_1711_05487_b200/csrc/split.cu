// split.cu -- the fused long_row_split pass (IMB decomposition).
//
// The dense long rows run as column-tiled items (x block in smem, streams from
// HBM) and the other rows as one nnz_split bin (random x gathers, bound by the
// L1 miss path). Launched as two kernels, even on two streams, they hardly
// overlap on B200: the first fills every SM and the block scheduler runs the
// second behind it (measured C4: 57 + 80 us -> 140 us). Here ONE grid
// interleaves both kinds of CTAs in blockIdx order -- long item i sits at
// block floor(i * total / n_items) -- so every SM mixes HBM-bound long-row
// CTAs with gather-bound short-row CTAs for the whole pass. The epilogue
// (ordered carry fix-up of the bin + per-row reduction of the long-row
// partials, disjoint rows) is one launch as well.
#include <type_traits>

#include "tiles.cuh"

namespace spmv {

constexpr int kSplitThreads = 256;
#ifndef SPLIT_LB
#define SPLIT_LB 4
#endif
#ifndef SPLIT_TPW
#define SPLIT_TPW 4
#endif
// nz tiles per warp of a short-row CTA: fewer, longer-lived CTAs (B200, C4:
// 1 tile 117.7 us, 2 113.4, 3 112.4, 4 111.2, 5 111.7, 6 113.6)
constexpr int kSplitTPW = SPLIT_TPW;

template <typename RP, bool L2G, bool C16>
__global__ void __launch_bounds__(kSplitThreads, SPLIT_LB) split_fused_kernel(const NzP<RP> z, const LongP l, int64_t n_items,
                                                                         int64_t n_groups) {
  __shared__ double xs[kLongXB];
  __shared__ __align__(16) uint32_t emask_s[kSplitThreads / 32][8];  // tile_q + rpc path only
  pdl_trigger();
  pdl_wait();
  const int64_t total = n_items + n_groups;
  const int64_t b = blockIdx.x;
  const int64_t Lb = (b + 1) * n_items / total;  // long items among blocks [0, b]
  if (Lb > b * n_items / total) {
    long_item<kSplitThreads, C16>(l, Lb - 1, xs);
    return;
  }
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int NW = kSplitThreads / 32;
  // nz group (b - Lb): kSplitTPW tiles per warp, the group's tiles contiguous
  for (int j = 0; j < kSplitTPW; ++j) {
    const int64_t k = ((b - Lb) * kSplitTPW + j) * NW + w;
    if (k < z.T) nz_tile<RP, false, true, L2G>(z, k, lane, nullptr, emask_s[w]);
  }
}

// blocks [0, nfb): ordered carry fix-up of the bin (runs <= 16: one thread
// per run start); blocks [nfb, ...): y[long_rows[q]] = sum_b partial[q][b]
__global__ void __launch_bounds__(kNT) split_epilogue_kernel(const int32_t* __restrict__ crow,
                                                             const double* __restrict__ cval, int64_t T, int nfb,
                                                             const double* __restrict__ partial, int64_t n_long,
                                                             int64_t nblk, const int32_t* __restrict__ long_rows,
                                                             double* __restrict__ y) {
  pdl_trigger();
  pdl_wait();
  if ((int)blockIdx.x < nfb) {
    const int64_t k = (int64_t)blockIdx.x * kNT + threadIdx.x;
    if (k >= T) return;
    // (carries / partials / y come from the previous kernel: L2-coherent loads)
    const int32_t r = __ldcg(crow + k);
    if (r < 0 || (k > 0 && __ldcg(crow + k - 1) == r)) return;
    double s = __ldcg(cval + k);
    for (int64_t q = k + 1; q < T && __ldcg(crow + q) == r; ++q) s += __ldcg(cval + q);
    y[r] = __ldcg(y + r) + s;
    return;
  }
  const int lane = threadIdx.x & 31;
  const int64_t q = ((int64_t)(blockIdx.x - nfb) * kNT + threadIdx.x) >> 5;
  if (q >= n_long) return;
  const double a = long_row_total(partial + q * nblk, nblk, lane);
  if (lane == 0) y[long_rows[q]] = a;
}

NzP<int32_t> nz_params32(const NzPlan& z, const double* x, double* y);
NzP<int64_t> nz_params64(const NzPlan& z, const double* x, double* y);
LongP long_params(const ExecArgs& a);
int long_items(const ExecArgs& a);

int launch_split_fused(const ExecArgs& a, cudaStream_t s) {
  int n = 0;
  const NzPlan& z = a.nz;
  if (a.stage != 2) {
    if (z.memset_y) cudaMemsetAsync(a.y, 0, (size_t)z.m_out * 8, s);
    const int64_t items = long_items(a), per = (int64_t)kSplitTPW * (kSplitThreads / 32),
                  groups = (z.T + per - 1) / per;
    const int grid = (int)(items + groups);
    const dim3 g(grid), b(kSplitThreads);
    // one instantiation per (rowptr width, gather path, long-row column
    // format): a kernel holding both long-row paths spills at 64 registers
    auto go = [&](auto rp, auto l2g, auto c16) {
      using RP = decltype(rp);
      constexpr bool L2G = decltype(l2g)::value, C16 = decltype(c16)::value;
      if constexpr (sizeof(RP) == 8)
        launch_pdl(split_fused_kernel<RP, L2G, C16>, g, b, 0, s, nz_params64(z, a.x, a.y), long_params(a), items,
                   groups);
      else
        launch_pdl(split_fused_kernel<RP, L2G, C16>, g, b, 0, s, nz_params32(z, a.x, a.y), long_params(a), items,
                   groups);
    };
    using T_ = std::true_type;
    using F_ = std::false_type;
    auto go2 = [&](auto rp) {
      if (z.gather_l2) {
        if (a.long_c16) go(rp, T_{}, T_{}); else go(rp, T_{}, F_{});
      } else {
        if (a.long_c16) go(rp, F_{}, T_{}); else go(rp, F_{}, F_{});
      }
    };
    if (z.V.rp_bytes == 8) go2(int64_t{}); else go2(int32_t{});
    ++n;
  }
  if (a.stage != 1) {
    if (z.T > 1 && z.max_run > 16) {
      n += launch_fixup(z.carry_row, z.carry_val, z.T, a.y, 0, z.max_run, s);
      launch_long_tiled(a, 2, s);
      ++n;
    } else {
      const int nfb = z.T > 1 ? (int)((z.T + kNT - 1) / kNT) : 0;
      const int nrb = (int)((a.n_long * 32 + kNT - 1) / kNT);
      launch_pdl(split_epilogue_kernel, dim3(nfb + nrb), dim3(kNT), 0, s, (const int32_t*)z.carry_row,
                 (const double*)z.carry_val, z.T, nfb, (const double*)a.long_partial, a.n_long, a.nblk, a.long_rows,
                 a.y);
      ++n;
    }
  }
  return n;
}

}  // namespace spmv
