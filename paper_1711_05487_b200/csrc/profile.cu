// profile.cu -- the profile-guided classifier's micro-benchmarks (SURVEY
// 8(f) f1; paper Sec. III-B bound-and-bottleneck analysis, and
// Fig. 4), re-designed for a GPU.
//
// The baseline is the paper's CSR kernel under its static 1-D nnz-balanced
// partition (Fig. 2): CTA c of a resident grid owns the
// contiguous row block [b_c, b_{c+1}) with ~nnz/G nonzeros, VS lanes per
// row. Three runs of it give the measured bounds:
//   P_CSR  the plain kernel's rate;
//   P_IMB  2*NNZ / t_median, t_median = the median CTA busy time (the CTA is
//          the GPU's "thread" of the static partition; median, not mean,
//          P:319-325), from %globaltimer stamps of the same run;
//   P_ML   the kernel reading colind but gathering x[row] instead of
//          x[colind[j]] ("colind := row index"): regular x access;
//   P_CMP  the kernel gathering x[row] without reading colind.
// P_MB and P_peak are analytic from B_max, the device
// copy bandwidth measured once per process (the STREAM analogue of Table III):
// main memory for working sets above L2, L2-resident otherwise (footnote
// P:306-307).
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "common.cuh"
#include "internal.h"

namespace spmv {

constexpr int kProbeThreads = 256;

__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// MODE 0: CSR; 1: colind read, x[row] gathered (ML probe); 2: x[row], colind unread (CMP probe)
template <int VS, typename RP, int MODE>
__global__ void __launch_bounds__(kProbeThreads) probe_kernel(const RP* __restrict__ rp, const int32_t* __restrict__ col,
                                                              const double* __restrict__ val,
                                                              const double* __restrict__ x, double* __restrict__ y,
                                                              const int64_t* __restrict__ blk, int64_t ncols,
                                                              unsigned long long* __restrict__ busy) {
  __shared__ uint64_t t_start;
  if (threadIdx.x == 0) t_start = global_ns();
  __syncthreads();
  const int64_t r0 = blk[blockIdx.x], r1 = blk[blockIdx.x + 1];
  const int lane = threadIdx.x % VS;
  const int gi = threadIdx.x / VS;
  constexpr int G = kProbeThreads / VS;
  for (int64_t rb = r0; rb < r1; rb += G) {
    const int64_t r = rb + gi;
    const bool active = r < r1;
    const int64_t rx = r < ncols ? r : ncols - 1;  // x index of the probes (row blocks may be rectangular)
    int64_t a = 0, b = 0;
    if (active) {
      a = (int64_t)ld_ro(rp + r);
      b = (int64_t)ld_ro(rp + r + 1);
    }
    double acc0 = 0.0, acc1 = 0.0;
    for (int64_t j = a + lane; j < b; j += 2 * VS) {
      const bool two = j + VS < b;
      int64_t c0, c1;
      if (MODE == 2) {
        c0 = c1 = rx;
      } else {
        const int32_t k0 = ld_stream(col + j), k1 = two ? ld_stream(col + j + VS) : 0;
        // ML probe: the colind stream is read (same traffic), x is indexed by
        // the row (k >= 0 always, so the select keeps the loads live)
        c0 = MODE == 1 ? rx + (k0 < 0 ? k0 : 0) : k0;
        c1 = MODE == 1 ? rx + (k1 < 0 ? k1 : 0) : k1;
      }
      acc0 = fma(ld_stream(val + j), ld_x(x + c0), acc0);
      if (two) acc1 = fma(ld_stream(val + j + VS), ld_x(x + c1), acc1);
    }
    const double s = group_sum<VS>(acc0 + acc1);
    if (active && lane == 0) y[r] = s;
  }
  __syncthreads();
  if (threadIdx.x == 0 && busy) busy[blockIdx.x] = global_ns() - t_start;
}

// b_c = min{ r : rowptr[r] >= ceil(c * nnz / G) } (the shard rule of P:708-711 at CTA granularity)
template <typename RP>
__global__ void probe_blocks_kernel(const RP* __restrict__ rp, int64_t m, int64_t nnz, int G, int64_t* __restrict__ blk) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c > G) return;
  if (c == 0) { blk[0] = 0; return; }
  if (c == G) { blk[G] = m; return; }
  const int64_t key = ((int64_t)c * nnz + G - 1) / G;
  int64_t lo = 0, hi = m;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if ((int64_t)rp[mid] < key) lo = mid + 1; else hi = mid;
  }
  blk[c] = lo;
}

template <int VS, typename RP, int MODE>
static void probe_launch(const MatView& A, const double* x, double* y, const int64_t* blk, int G,
                         unsigned long long* busy, cudaStream_t s) {
  probe_kernel<VS, RP, MODE><<<G, kProbeThreads, 0, s>>>((const RP*)A.rowptr, A.col, A.val, x, y, blk, A.n_cols,
                                                         busy);
}

template <typename RP, int MODE>
static void probe_vs(int vs, const MatView& A, const double* x, double* y, const int64_t* blk, int G,
                     unsigned long long* busy, cudaStream_t s) {
  switch (vs) {
    case 1: probe_launch<1, RP, MODE>(A, x, y, blk, G, busy, s); break;
    case 2: probe_launch<2, RP, MODE>(A, x, y, blk, G, busy, s); break;
    case 4: probe_launch<4, RP, MODE>(A, x, y, blk, G, busy, s); break;
    case 8: probe_launch<8, RP, MODE>(A, x, y, blk, G, busy, s); break;
    case 16: probe_launch<16, RP, MODE>(A, x, y, blk, G, busy, s); break;
    default: probe_launch<32, RP, MODE>(A, x, y, blk, G, busy, s); break;
  }
}

static void probe_run(int mode, int vs, const MatView& A, const double* x, double* y, const int64_t* blk, int G,
                      unsigned long long* busy, cudaStream_t s) {
  if (A.rp_bytes == 8) {
    if (mode == 0) probe_vs<int64_t, 0>(vs, A, x, y, blk, G, busy, s);
    else if (mode == 1) probe_vs<int64_t, 1>(vs, A, x, y, blk, G, busy, s);
    else probe_vs<int64_t, 2>(vs, A, x, y, blk, G, busy, s);
  } else {
    if (mode == 0) probe_vs<int32_t, 0>(vs, A, x, y, blk, G, busy, s);
    else if (mode == 1) probe_vs<int32_t, 1>(vs, A, x, y, blk, G, busy, s);
    else probe_vs<int32_t, 2>(vs, A, x, y, blk, G, busy, s);
  }
}

// device copy bandwidth (read + write bytes / s), best of 5; cached per device and size class
static double copy_bandwidth(int dev, size_t bytes, cudaStream_t s) {
  static double cache[16][2] = {};
  const int cls = bytes > (64u << 20) ? 0 : 1;
  if (dev < 16 && cache[dev][cls] > 0) return cache[dev][cls];
  void *a = nullptr, *b = nullptr;
  if (cudaMalloc(&a, bytes) != cudaSuccess || cudaMalloc(&b, bytes) != cudaSuccess) {
    cudaFree(a);
    cudaGetLastError();
    return 0.0;
  }
  cudaMemsetAsync(a, 0, bytes, s);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  const int reps = cls == 0 ? 1 : 8;  // L2-class buffers: several copies per timing
  for (int t = 0; t < 6; ++t) {
    cudaEventRecord(e0, s);
    for (int r = 0; r < reps; ++r) cudaMemcpyAsync(b, a, bytes, cudaMemcpyDeviceToDevice, s);
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (t > 0) best = std::min(best, ms / reps);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(a);
  cudaFree(b);
  const double bw = 2.0 * (double)bytes / (best * 1e-3);
  if (dev < 16) cache[dev][cls] = bw;
  return bw;
}

// Runs the three timed probes (reps SpMVs each, mean time) and the analytic
// bounds. x / y: scratch device vectors of the view's sizes.
int run_profile_probes(const MatView& A, int vs, int sm_count, int64_t l2_bytes, double* x, double* y,
                       ProfileBounds& out, cudaStream_t s) {
  if (A.nnz == 0 || A.m == 0) return 0;
  int dev = 0;
  cudaGetDevice(&dev);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, probe_kernel<32, int32_t, 0>, kProbeThreads, 0);
  const int G = std::max(1, sm_count * std::max(per_sm, 1));
  int64_t* blk = nullptr;
  unsigned long long* busy = nullptr;
  if (cudaMalloc(&blk, (size_t)(G + 1) * 8) != cudaSuccess) return -1;
  if (cudaMalloc(&busy, (size_t)G * 8) != cudaSuccess) {
    cudaFree(blk);
    return -1;
  }
  const int gb = (G + 1 + 255) / 256;
  if (A.rp_bytes == 8)
    probe_blocks_kernel<int64_t><<<gb, 256, 0, s>>>((const int64_t*)A.rowptr, A.m, A.nnz, G, blk);
  else
    probe_blocks_kernel<int32_t><<<gb, 256, 0, s>>>((const int32_t*)A.rowptr, A.m, A.nnz, G, blk);
  cudaMemsetAsync(x, 0, (size_t)A.n_cols * 8, s);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int reps = 8;
  double t_mode[3] = {0, 0, 0};
  for (int mode = 0; mode < 3; ++mode) {
    probe_run(mode, vs, A, x, y, blk, G, nullptr, s);  // warm-up
    cudaEventRecord(e0, s);
    for (int r = 0; r < reps; ++r) probe_run(mode, vs, A, x, y, blk, G, nullptr, s);
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    t_mode[mode] = ms * 1e-3 / reps;
  }
  // per-CTA busy times of one more baseline run (the P_IMB median)
  probe_run(0, vs, A, x, y, blk, G, busy, s);
  std::vector<unsigned long long> h((size_t)G);
  cudaMemcpyAsync(h.data(), busy, (size_t)G * 8, cudaMemcpyDeviceToHost, s);
  const cudaError_t err = cudaStreamSynchronize(s);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(blk);
  cudaFree(busy);
  if (err != cudaSuccess) return -1;
  std::sort(h.begin(), h.end());
  const double med_ns = (G % 2) ? (double)h[(size_t)G / 2] : 0.5 * ((double)h[(size_t)G / 2 - 1] + (double)h[(size_t)G / 2]);
  const double flops = 2.0 * (double)A.nnz;
  out.p_csr = flops / t_mode[0];
  out.p_ml = flops / t_mode[1];
  out.p_cmp = flops / t_mode[2];
  out.p_imb = med_ns > 0 ? flops / (med_ns * 1e-9) : out.p_csr;
  const double ws = 12.0 * (double)A.nnz + (double)A.rp_bytes * (double)(A.m + 1) + 8.0 * (double)A.n_cols +
                    8.0 * (double)A.m;
  const bool fits = ws <= (double)l2_bytes;
  out.bmax = copy_bandwidth(dev, fits ? (size_t)std::max<int64_t>(l2_bytes / 4, 1 << 20) : (size_t)1 << 30, s);
  out.p_mb = flops / (ws / out.bmax);
  out.p_peak = flops / ((8.0 * (double)A.nnz + 8.0 * (double)A.n_cols + 8.0 * (double)A.m) / out.bmax);
  out.ws_fits_l2 = fits ? 1 : 0;
  out.vs = vs;
  out.ctas = G;
  return 0;
}

}  // namespace spmv
