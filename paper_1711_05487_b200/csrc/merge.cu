// merge.cu -- merge_path: the IMB-class kernel (GPU analogue of the OpenMP
// "auto" schedule). CTA k owns a fixed slice [k*ITEMS,
// (k+1)*ITEMS) of the merge path of (row ends, nonzeros);
// products are formed cooperatively in smem (coalesced loads, IPT independent
// x gathers per thread), then each thread walks IPT consecutive path items.
// Rows cut by a thread edge are completed in smem in thread order; rows cut by
// a CTA edge are completed by the ordered carry fix-up (deterministic).
#include "common.cuh"
#include "internal.h"

namespace spmv {

constexpr int kIPT = 8;  // merge-path items per thread (ITEMS = kNT * kIPT = 2048)

template <typename RP>
__global__ void __launch_bounds__(kNT) merge_kernel(const RP* __restrict__ rp, const int32_t* __restrict__ col,
                                                    const double* __restrict__ val, const double* __restrict__ x,
                                                    double* __restrict__ y, int64_t m,
                                                    const int32_t* __restrict__ mrow, const int64_t* __restrict__ mnnz,
                                                    int32_t* __restrict__ crow, double* __restrict__ cval) {
  constexpr int ITEMS = kNT * kIPT;
  __shared__ int32_t rend[ITEMS];
  __shared__ double prod[ITEMS];
  __shared__ int32_t tcr[kNT];
  __shared__ double tcv[kNT];
  const int tid = threadIdx.x;
  const int64_t k = blockIdx.x;
  const int64_t i0 = mrow[k], i1 = mrow[k + 1];
  const int64_t j0 = mnnz[k], j1 = mnnz[k + 1];
  const int nr = (int)(i1 - i0), nz = (int)(j1 - j0);
  for (int q = tid; q < nr; q += kNT) rend[q] = (int)((int64_t)ld_ro(rp + i0 + q + 1) - j0);
  {
    int c[kIPT];
#pragma unroll
    for (int u = 0; u < kIPT; ++u) {
      const int q = u * kNT + tid;
      c[u] = q < nz ? ld_stream(col + j0 + q) : 0;
    }
    double v[kIPT], xv[kIPT];
#pragma unroll
    for (int u = 0; u < kIPT; ++u) {
      const int q = u * kNT + tid;
      v[u] = q < nz ? ld_stream(val + j0 + q) : 0.0;
      xv[u] = q < nz ? ld_x(x + c[u]) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kIPT; ++u) {
      const int q = u * kNT + tid;
      if (q < nz) prod[q] = v[u] * xv[u];
    }
  }
  __syncthreads();
  const int tot = nr + nz;
  const int d0 = tid * kIPT < tot ? tid * kIPT : tot;
  const int d1 = d0 + kIPT < tot ? d0 + kIPT : tot;
  int lo = d0 - nz > 0 ? d0 - nz : 0, hi = d0 < nr ? d0 : nr;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (rend[mid] <= d0 - mid - 1) lo = mid + 1; else hi = mid;
  }
  int ii = lo, jj = d0 - lo;
  double acc = 0.0, first_val = 0.0;
  int first_row = -1;
  for (int d = d0; d < d1; ++d) {
    if (ii < nr && rend[ii] <= jj) {
      if (first_row < 0) { first_row = ii; first_val = acc; }
      else y[i0 + ii] = acc;
      acc = 0.0;
      ++ii;
    } else {
      acc += prod[jj];
      ++jj;
    }
  }
  tcr[tid] = ii;
  tcv[tid] = acc;
  __syncthreads();
  if (first_row >= 0) {
    double pre = 0.0;
    for (int t = tid - 1; t >= 0 && tcr[t] == first_row; --t) pre = tcv[t] + pre;
    y[i0 + first_row] = pre + first_val;
  }
  if (tid == 0) {
    double s = 0.0;
    for (int t = kNT - 1; t >= 0 && tcr[t] == nr; --t) s = tcv[t] + s;
    crow[k] = i1 < m ? (int32_t)i1 : -1;
    cval[k] = s;
  }
}

int launch_merge(const ExecArgs& a, cudaStream_t s) {
  if (a.Tm == 0) return 0;
  int n = 0;
  if (a.stage != 2) {
    ++n;
    if (a.A.rp_bytes == 8)
      merge_kernel<int64_t><<<(int)a.Tm, kNT, 0, s>>>((const int64_t*)a.A.rowptr, a.A.col, a.A.val, a.x, a.y, a.A.m,
                                                      a.mrow, a.mnnz, a.mcarry_row, a.mcarry_val);
    else
      merge_kernel<int32_t><<<(int)a.Tm, kNT, 0, s>>>((const int32_t*)a.A.rowptr, a.A.col, a.A.val, a.x, a.y, a.A.m,
                                                      a.mrow, a.mnnz, a.mcarry_row, a.mcarry_val);
  }
  if (a.stage != 1) n += launch_fixup(a.mcarry_row, a.mcarry_val, a.Tm, a.y, 0, a.nnz_max / 2048 + 2, s);
  return n;
}

}  // namespace spmv
