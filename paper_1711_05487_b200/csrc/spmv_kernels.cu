// spmv_kernels.cu -- the SpMV variants for sm_100a.
//
// All variants compute y_i = sum_j a_ij x_colind[j] (Fig. 2, read
// as accumulation), overwrite y, give exactly 0.0 for empty rows, and are
// deterministic: every sum is formed in an order fixed by the plan (tiles,
// lane groups, butterfly shuffles, carries summed in tile order), never by
// scheduling or atomics.
//
//  csr_vector<VS>  VS lanes per row, 2 accumulators per lane (CMP class:
//                  "inner loop unrolling + vectorization", P:629-630 / Table II)
//  cta_stream      persistent CTAs; fixed C-nonzero tiles staged global->smem
//                  by TMA bulk copies (cp.async.bulk + mbarrier, S-stage ring,
//                  L2 evict_first); products formed tile-wide so every thread
//                  has C/256 independent x gathers in flight; per-row sums
//                  from smem; rows cut by a tile edge finish in a fix-up pass.
//                  Optional 16-bit delta colind decoded in smem by a tile
//                  scan (MB class, P:589-597 / Table II).
//  merge_path      CTA = fixed slice of the (row ends, nonzeros) merge path,
//                  thread = IPT consecutive path items (IMB class, OpenMP
//                  "auto" schedule analogue).
//  long_row_split  csr_vector over short rows that skips long rows, then one
//                  CTA per C-nonzero chunk of each long row and an ordered
//                  per-row reduction of the chunk partials (IMB decomposition,
//                  P:608-621, Fig. 7 semantics per SURVEY 8(c3) #11).
#include <climits>
#include <cstdio>
#include "common.cuh"
#include "internal.h"

namespace spmv {

constexpr int kRowCap = 1024;  // rowptr entries staged in smem per STREAM tile
constexpr int kIPT = 8;        // merge-path items per thread

// ============================================================================
// csr_vector<VS>
// ============================================================================
template <int VS, typename RP, bool SKIP_LONG>
__global__ void __launch_bounds__(kNT) vector_kernel(const RP* __restrict__ rp, const int32_t* __restrict__ col,
                                                     const double* __restrict__ val, const double* __restrict__ x,
                                                     double* __restrict__ y, int64_t m, int64_t l_split) {
  constexpr int GPW = 32 / VS;
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
    double acc0 = 0.0, acc1 = 0.0;
    if (active && !skip) {
      int64_t j = a + lane;
      for (; j + VS < b; j += 2 * VS) {
        const int c0 = ld_stream(col + j), c1 = ld_stream(col + j + VS);
        const double v0 = ld_stream(val + j), v1 = ld_stream(val + j + VS);
        acc0 = fma(v0, ld_x(x + c0), acc0);
        acc1 = fma(v1, ld_x(x + c1), acc1);
      }
      if (j < b) acc0 = fma(ld_stream(val + j), ld_x(x + ld_stream(col + j)), acc0);
    }
    double s = group_sum<VS>(acc0 + acc1);
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
  const int64_t groups_needed = a.A.m;
  int64_t grid = (groups_needed * a.vs + kNT - 1) / kNT;
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

static void launch_fixup(const int32_t* crow, const double* cval, int64_t T, double* y, int set, cudaStream_t s) {
  fixup_kernel<<<(int)((T + kNT - 1) / kNT), kNT, 0, s>>>(crow, cval, T, y, set);
}

// ============================================================================
// cta_stream
// ============================================================================
template <typename RP>
struct StreamP {
  const RP* rp;
  const void* idx;        // int32 colind or uint16 dcol
  const int32_t* head;
  const int32_t* anchor;
  const double* val;
  const double* x;
  double* y;
  const int32_t* tile_row;
  int32_t* carry_row;
  double* carry_val;
  int64_t nnz, C, T;
  int stages;
};

__host__ __device__ __forceinline__ size_t align128(size_t v) { return (v + 127) & ~(size_t)127; }

struct StreamLayout {
  size_t vals, idx, stage, rp, flag, base, S, P, bar, total;
};

__host__ __device__ inline StreamLayout stream_layout(int64_t C, int stages, int rp_bytes, bool d16) {
  StreamLayout L;
  L.vals = 0;
  L.idx = align128((size_t)C * 8);
  L.stage = align128(L.idx + (size_t)C * (d16 ? 2 : 4));
  size_t o = L.stage * stages;
  L.rp = o; o = align128(o + (size_t)(kRowCap + 4) * rp_bytes);
  if (d16) {
    L.flag = o; o = align128(o + (size_t)C);
    L.base = o; o = align128(o + (size_t)C * 4);
    L.S = o; o = align128(o + (size_t)C * 4);
    L.P = o; o = align128(o + (size_t)C * 2);
  } else {
    L.flag = L.base = L.S = L.P = 0;
  }
  L.bar = o; o += 8 * (size_t)stages;
  L.total = align128(o);
  return L;
}

size_t stream_smem_bytes(int64_t C, int stages, int rp_bytes, bool d16) {
  return stream_layout(C, stages, rp_bytes, d16).total;
}

// Row accessor: smem-staged rowptr slice [fr0, fr0+nst) or the global array.
template <typename RP>
struct Rows {
  const RP* g;
  const RP* s;
  int64_t fr0;
  bool staged;
  __device__ __forceinline__ int64_t operator()(int64_t r) const {
    return staged ? (int64_t)s[r - fr0] : (int64_t)ld_ro(g + r);
  }
};

// Block-wide exclusive scan of (sum, max) pairs, one pair per thread.
__device__ __forceinline__ void block_scan_sum_max(uint32_t v, int p, uint32_t& ex_sum, int& ex_max,
                                                   uint32_t* ws, int* wm) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t s = v;
  int mx = p;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t ts = __shfl_up_sync(0xffffffffu, s, o);
    const int tm = __shfl_up_sync(0xffffffffu, mx, o);
    if (lane >= o) { s += ts; mx = mx > tm ? mx : tm; }
  }
  if (lane == 31) { ws[w] = s; wm[w] = mx; }
  __syncthreads();
  uint32_t ps = 0;
  int pm = -1;
  for (int q = 0; q < w; ++q) { ps += ws[q]; pm = pm > wm[q] ? pm : wm[q]; }
  // exclusive within warp
  uint32_t es = __shfl_up_sync(0xffffffffu, s, 1);
  int em = __shfl_up_sync(0xffffffffu, mx, 1);
  if (lane == 0) { es = 0; em = -1; }
  ex_sum = ps + es;
  ex_max = pm > em ? pm : em;
  __syncthreads();
}

// Decode the delta colind of one tile held in smem (dcol_s[0..cnt)).
// Afterwards column(l) = base_s[P_s[l]] + (S_s[l] - S_s[P_s[l]]), where P_s[l]
// is the tile-local start of l's row (or 0 for the row entering the tile),
// base_s[P] its absolute first column (head[r], or anchor for the entering
// row) and S_s the tile prefix sum of the deltas with element 0 taken as 0.
template <typename RP>
__device__ void d16_tile_decode(const uint16_t* dcol_s, int cnt, int E, const Rows<RP>& rows, int64_t fr,
                                int64_t nloc, int64_t t0, int64_t t1, const int32_t* __restrict__ head,
                                int32_t anchor_k, uint8_t* flag_s, int32_t* base_s, uint32_t* S_s, uint16_t* P_s) {
  __shared__ uint32_t ws[kNT / 32];
  __shared__ int wm[kNT / 32];
  for (int l = threadIdx.x; l < cnt; l += kNT) flag_s[l] = 0;
  __syncthreads();
  for (int64_t q = threadIdx.x; q < nloc; q += kNT) {
    const int64_t r = fr + q;
    const int64_t a = rows(r), b = rows(r + 1);
    const int64_t ls = (a > t0 ? a : t0) - t0, le = (b < t1 ? b : t1) - t0;
    if (le > ls) {
      flag_s[ls] = 1;
      base_s[ls] = a >= t0 ? ld_ro(head + r) : anchor_k;
    }
  }
  __syncthreads();
  const int l0 = threadIdx.x * E;
  uint32_t sum = 0;
  int last = -1;
  for (int e = 0; e < E; ++e) {
    const int l = l0 + e;
    if (l < cnt) {
      sum += (l == 0) ? 0u : (uint32_t)dcol_s[l];
      if (flag_s[l]) last = l;
    }
  }
  uint32_t ex_sum;
  int ex_max;
  block_scan_sum_max(sum, last, ex_sum, ex_max, ws, wm);
  uint32_t run = ex_sum;
  int p = ex_max;
  for (int e = 0; e < E; ++e) {
    const int l = l0 + e;
    if (l < cnt) {
      run += (l == 0) ? 0u : (uint32_t)dcol_s[l];
      if (flag_s[l]) p = l;
      S_s[l] = run;
      P_s[l] = (uint16_t)p;
    }
  }
  __syncthreads();
}

template <int VS, typename RP, bool D16>
__global__ void __launch_bounds__(kNT, 2) stream_kernel(const StreamP<RP> p) {
  extern __shared__ __align__(128) unsigned char smem[];
  const StreamLayout L = stream_layout(p.C, p.stages, (int)sizeof(RP), D16);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L.bar);
  RP* rp_s = reinterpret_cast<RP*>(smem + L.rp);
  const int tid = threadIdx.x;
  const int idx_bytes = D16 ? 2 : 4;

  uint64_t policy = 0;
  if (tid == 0) {
    policy = policy_evict_first();
    for (int s = 0; s < p.stages; ++s) mbar_init(&bar[s], 1);
    fence_mbar_init();
  }
  __syncthreads();

  auto issue = [&](int64_t k, int s) {
    const int64_t t0 = k * p.C;
    const int64_t cnt = (p.nnz - t0) < p.C ? (p.nnz - t0) : p.C;
    const uint32_t vb = (uint32_t)((cnt * 8 + 15) & ~15ll);
    const uint32_t ib = (uint32_t)((cnt * idx_bytes + 15) & ~15ll);
    unsigned char* st = smem + L.stage * s;
    mbar_arrive_expect_tx(&bar[s], vb + ib);
    if (vb) {
      bulk_g2s(st + L.vals, p.val + t0, vb, &bar[s], policy);
      bulk_g2s(st + L.idx, static_cast<const unsigned char*>(p.idx) + t0 * idx_bytes, ib, &bar[s], policy);
    }
  };

  if (tid == 0) {
    int s = 0;
    for (int64_t k = blockIdx.x; k < p.T && s < p.stages; k += gridDim.x, ++s) issue(k, s);
  }

  int64_t it = 0;
  for (int64_t k = blockIdx.x; k < p.T; k += gridDim.x, ++it) {
    const int s = (int)(it % p.stages);
    const uint32_t parity = (uint32_t)((it / p.stages) & 1);
    unsigned char* st = smem + L.stage * s;
    double* vals_s = reinterpret_cast<double*>(st + L.vals);

    const int64_t t0 = k * p.C;
    const int64_t t1 = (t0 + p.C) < p.nnz ? (t0 + p.C) : p.nnz;
    const int cnt = (int)(t1 - t0);
    const int64_t R0 = ld_ro(p.tile_row + k), R1 = ld_ro(p.tile_row + k + 1);
    const int64_t fr0 = R0 > 0 ? R0 - 1 : 0;
    const int64_t nst = R1 - fr0 + 1;
    const bool staged = nst <= kRowCap;
    if (staged)
      for (int64_t i = tid; i < nst; i += kNT) rp_s[i] = ld_ro(p.rp + fr0 + i);

    mbar_wait(&bar[s], parity);

    if (!D16) {
      const int32_t* idx_s = reinterpret_cast<const int32_t*>(st + L.idx);
      for (int lb = 0; lb < cnt; lb += kNT * 8) {
        int c[8];
        double xv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int l = lb + u * kNT + tid;
          c[u] = l < cnt ? idx_s[l] : 0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int l = lb + u * kNT + tid;
          xv[u] = l < cnt ? ld_x(p.x + c[u]) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int l = lb + u * kNT + tid;
          if (l < cnt) vals_s[l] *= xv[u];
        }
      }
    }
    __syncthreads();  // rp_s staged (and products formed for int32 colind)

    Rows<RP> rows{p.rp, rp_s, fr0, staged};
    const bool incoming = R0 > 0 && rows(R0) > t0;
    const int64_t fr = R0 - (incoming ? 1 : 0);
    const int64_t nloc = (R1 - R0) + (incoming ? 1 : 0);

    if (D16) {
      const uint16_t* dcol_s = reinterpret_cast<const uint16_t*>(st + L.idx);
      uint8_t* flag_s = smem + L.flag;
      int32_t* base_s = reinterpret_cast<int32_t*>(smem + L.base);
      uint32_t* S_s = reinterpret_cast<uint32_t*>(smem + L.S);
      uint16_t* P_s = reinterpret_cast<uint16_t*>(smem + L.P);
      const int E = (int)(p.C / kNT);
      d16_tile_decode<RP>(dcol_s, cnt, E, rows, fr, nloc, t0, t1, p.head, ld_ro(p.anchor + k), flag_s, base_s, S_s,
                          P_s);
      for (int lb = 0; lb < cnt; lb += kNT * 8) {
        int c[8];
        double xv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int l = lb + u * kNT + tid;
          if (l < cnt) {
            const int pp = P_s[l];
            c[u] = base_s[pp] + (int)(S_s[l] - S_s[pp]);
          } else {
            c[u] = 0;
          }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int l = lb + u * kNT + tid;
          xv[u] = l < cnt ? ld_x(p.x + c[u]) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int l = lb + u * kNT + tid;
          if (l < cnt) vals_s[l] *= xv[u];
        }
      }
      __syncthreads();
    }

    // per-row sums of the products (VS lanes per row, warp-uniform loop)
    {
      constexpr int GPW = 32 / VS;
      constexpr int NG = kNT / VS;
      const int lane = tid % VS, gi = (tid & 31) / VS, w = tid >> 5;
      for (int64_t qb = (int64_t)w * GPW; qb < nloc; qb += NG) {
        const int64_t q = qb + gi;
        const bool active = q < nloc;
        double acc = 0.0;
        int64_t r = 0;
        if (active) {
          r = fr + q;
          const int64_t a = rows(r), b = rows(r + 1);
          const int ls = (int)((a > t0 ? a : t0) - t0), le = (int)((b < t1 ? b : t1) - t0);
          for (int l = ls + lane; l < le; l += VS) acc += vals_s[l];
        }
        acc = group_sum<VS>(acc);
        if (active && lane == 0) {
          if (incoming && q == 0) {
            p.carry_row[k] = (int32_t)r;
            p.carry_val[k] = acc;
          } else {
            p.y[r] = acc;
          }
        }
      }
      if (!incoming && tid == 0) p.carry_row[k] = -1;
    }
    __syncthreads();  // stage s and rp_s free
    if (tid == 0) {
      const int64_t kn = k + (int64_t)p.stages * gridDim.x;
      if (kn < p.T) {
        fence_proxy_async();
        issue(kn, s);
      }
    }
  }
}

template <int VS, typename RP, bool D16>
static void stream_launch_t(const ExecArgs& a, cudaStream_t s) {
  StreamP<RP> p;
  p.rp = (const RP*)a.A.rowptr;
  p.idx = D16 ? (const void*)a.dcol : (const void*)a.A.col;
  p.head = a.head;
  p.anchor = a.anchor;
  p.val = a.A.val;
  p.x = a.x;
  p.y = a.y;
  p.tile_row = a.tile_row;
  p.carry_row = a.carry_row;
  p.carry_val = a.carry_val;
  p.nnz = a.A.nnz;
  p.C = a.C;
  p.T = a.T;
  p.stages = a.stages;
  const size_t smem = stream_smem_bytes(a.C, a.stages, sizeof(RP), D16);
  const int grid = a.stream_grid;
  stream_kernel<VS, RP, D16><<<grid, kNT, smem, s>>>(p);
}

// Per device/instantiation: opt into large dynamic smem; return the persistent grid.
template <int VS, typename RP, bool D16>
static int stream_prepare_t(const ExecArgs& a) {
  const size_t smem = stream_smem_bytes(a.C, a.stages, sizeof(RP), D16);
  if (cudaFuncSetAttribute(stream_kernel<VS, RP, D16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
      cudaSuccess)
    return -1;
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, stream_kernel<VS, RP, D16>, kNT, smem) != cudaSuccess ||
      per_sm < 1)
    return -1;
  int64_t grid = (int64_t)a.sm_count * per_sm;
  if (grid > a.T) grid = a.T;
  return (int)grid;
}

template <typename RP, bool D16>
static int stream_prepare_vs(const ExecArgs& a) {
  switch (a.vs) {
    case 1: return stream_prepare_t<1, RP, D16>(a);
    case 2: return stream_prepare_t<2, RP, D16>(a);
    case 4: return stream_prepare_t<4, RP, D16>(a);
    case 8: return stream_prepare_t<8, RP, D16>(a);
    case 16: return stream_prepare_t<16, RP, D16>(a);
    default: return stream_prepare_t<32, RP, D16>(a);
  }
}

int stream_prepare(const ExecArgs& a) {
  const bool d16 = a.dcol != nullptr;
  if (a.A.rp_bytes == 8) return d16 ? stream_prepare_vs<int64_t, true>(a) : stream_prepare_vs<int64_t, false>(a);
  return d16 ? stream_prepare_vs<int32_t, true>(a) : stream_prepare_vs<int32_t, false>(a);
}

template <typename RP, bool D16>
static void stream_vs(const ExecArgs& a, cudaStream_t s) {
  switch (a.vs) {
    case 1: stream_launch_t<1, RP, D16>(a, s); break;
    case 2: stream_launch_t<2, RP, D16>(a, s); break;
    case 4: stream_launch_t<4, RP, D16>(a, s); break;
    case 8: stream_launch_t<8, RP, D16>(a, s); break;
    case 16: stream_launch_t<16, RP, D16>(a, s); break;
    default: stream_launch_t<32, RP, D16>(a, s); break;
  }
}

int launch_stream(const ExecArgs& a, cudaStream_t s) {
  const bool d16 = a.dcol != nullptr;
  int n = 0;
  if (a.stage != 2) {
    ++n;
    if (a.A.rp_bytes == 8) {
    if (d16) stream_vs<int64_t, true>(a, s); else stream_vs<int64_t, false>(a, s);
  } else {
    if (d16) stream_vs<int32_t, true>(a, s); else stream_vs<int32_t, false>(a, s);
    }
  }
  if (a.need_fixup && a.stage != 1) { launch_fixup(a.carry_row, a.carry_val, a.T, a.y, 0, s); ++n; }
  return n;
}

// Export: re-decode the delta colind on the device with the STREAM kernel's
// own tile decoder (bit-exact round-trip check).
template <typename RP>
__global__ void __launch_bounds__(kNT) d16_decode_kernel(const RP* __restrict__ rp, const uint16_t* __restrict__ dcol,
                                                         const int32_t* __restrict__ head,
                                                         const int32_t* __restrict__ anchor,
                                                         const int32_t* __restrict__ tile_row, int64_t nnz, int64_t C,
                                                         int32_t* __restrict__ out) {
  extern __shared__ __align__(128) unsigned char smem[];
  const StreamLayout L = stream_layout(C, 1, (int)sizeof(RP), true);
  const int64_t k = blockIdx.x;
  const int64_t t0 = k * C, t1 = (t0 + C) < nnz ? (t0 + C) : nnz;
  const int cnt = (int)(t1 - t0);
  uint16_t* dcol_s = reinterpret_cast<uint16_t*>(smem + L.idx);
  for (int l = threadIdx.x; l < cnt; l += kNT) dcol_s[l] = dcol[t0 + l];
  const int64_t R0 = tile_row[k], R1 = tile_row[k + 1];
  Rows<RP> rows{rp, nullptr, 0, false};
  __syncthreads();
  const bool incoming = R0 > 0 && rows(R0) > t0;
  const int64_t fr = R0 - (incoming ? 1 : 0);
  const int64_t nloc = (R1 - R0) + (incoming ? 1 : 0);
  uint8_t* flag_s = smem + L.flag;
  int32_t* base_s = reinterpret_cast<int32_t*>(smem + L.base);
  uint32_t* S_s = reinterpret_cast<uint32_t*>(smem + L.S);
  uint16_t* P_s = reinterpret_cast<uint16_t*>(smem + L.P);
  d16_tile_decode<RP>(dcol_s, cnt, (int)(C / kNT), rows, fr, nloc, t0, t1, head, anchor[k], flag_s, base_s, S_s, P_s);
  for (int l = threadIdx.x; l < cnt; l += kNT) {
    const int pp = P_s[l];
    out[t0 + l] = base_s[pp] + (int)(S_s[l] - S_s[pp]);
  }
}

void launch_d16_decode_export(const MatView& A, const uint16_t* dcol, const int32_t* head, const int32_t* anchor,
                              const int32_t* tile_row, int64_t C, int64_t T, int32_t* out, cudaStream_t s) {
  if (A.nnz == 0) return;
  const size_t smem = stream_smem_bytes(C, 1, A.rp_bytes, true);
  if (A.rp_bytes == 8) {
    cudaFuncSetAttribute(d16_decode_kernel<int64_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    d16_decode_kernel<int64_t><<<(int)T, kNT, smem, s>>>((const int64_t*)A.rowptr, dcol, head, anchor, tile_row,
                                                         A.nnz, C, out);
  } else {
    cudaFuncSetAttribute(d16_decode_kernel<int32_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    d16_decode_kernel<int32_t><<<(int)T, kNT, smem, s>>>((const int32_t*)A.rowptr, dcol, head, anchor, tile_row,
                                                         A.nnz, C, out);
  }
}

// ============================================================================
// merge_path
// ============================================================================
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
  if (a.stage != 1) { launch_fixup(a.mcarry_row, a.mcarry_val, a.Tm, a.y, 0, s); ++n; }
  return n;
}

// ============================================================================
// long_row_split: chunk partials of the long rows
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
  double t = warp_sum((a0 + a1) + (a2 + a3));
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
  int n = a.stage != 2 ? launch_vector(a, true, s) : 0;
  if (a.n_chunks > 0) {
    if (a.stage != 2) {
    ++n;
    if (a.A.rp_bytes == 8)
      long_chunk_kernel<int64_t><<<(int)a.n_chunks, kNT, 0, s>>>((const int64_t*)a.A.rowptr, a.A.col, a.A.val, a.x,
                                                                 a.long_rows, a.chunk_start, a.n_long, a.chunk,
                                                                 a.chunk_row, a.chunk_val);
    else
      long_chunk_kernel<int32_t><<<(int)a.n_chunks, kNT, 0, s>>>((const int32_t*)a.A.rowptr, a.A.col, a.A.val, a.x,
                                                                 a.long_rows, a.chunk_start, a.n_long, a.chunk,
                                                                 a.chunk_row, a.chunk_val);
    }
    if (a.stage != 1) { launch_fixup(a.chunk_row, a.chunk_val, a.n_chunks, a.y, 1, s); ++n; }
  }
  return n;
}

// ============================================================================
// iterated mode: nu = ||y||_2 with fixed chunking, x = y / nu
// ============================================================================
__global__ void __launch_bounds__(kNT) norm_partials_kernel(const double* __restrict__ y, int64_t m,
                                                            double* __restrict__ partials) {
  const int64_t b = blockIdx.x;
  const int64_t r0 = b * m / kNormPartials, r1 = (b + 1) * m / kNormPartials;
  double a0 = 0.0, a1 = 0.0;
  int64_t i = r0 + threadIdx.x;
  for (; i + kNT < r1; i += 2 * kNT) {
    const double v0 = ld_stream(y + i), v1 = ld_stream(y + i + kNT);
    a0 = fma(v0, v0, a0);
    a1 = fma(v1, v1, a1);
  }
  if (i < r1) { const double v = ld_stream(y + i); a0 = fma(v, v, a0); }
  double t = warp_sum(a0 + a1);
  __shared__ double ws[kNT / 32];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = t;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < kNT / 32; ++w) s += ws[w];
    partials[b] = s;
  }
}

__global__ void __launch_bounds__(kNT) normalize_kernel(const double* __restrict__ y, int64_t m,
                                                        const double* __restrict__ partials, int count,
                                                        double* __restrict__ x_out, double* __restrict__ nu_dev) {
  __shared__ double nu_s;
  if (threadIdx.x == 0) {
    double ss = 0.0;
    for (int q = 0; q < count; ++q) ss += partials[q];
    nu_s = sqrt(ss);
    if (blockIdx.x == 0 && nu_dev) *nu_dev = nu_s;
  }
  __syncthreads();
  const double nu = nu_s;
  const int64_t stride = (int64_t)gridDim.x * kNT;
  for (int64_t i = (int64_t)blockIdx.x * kNT + threadIdx.x; i < m; i += stride) x_out[i] = y[i] / nu;
}

int launch_norm_partials(const double* y, int64_t m, double* partials, cudaStream_t s) {
  norm_partials_kernel<<<kNormPartials, kNT, 0, s>>>(y, m, partials);
  return 1;
}

int launch_normalize(const double* y, int64_t m, const double* partials, int count, double* x_out, double* nu_dev,
                     cudaStream_t s) {
  int64_t grid = (m + kNT - 1) / kNT;
  if (grid > 148 * 8) grid = 148 * 8;
  if (grid < 1) grid = 1;
  normalize_kernel<<<(int)grid, kNT, 0, s>>>(y, m, partials, count, x_out, nu_dev);
  return 1;
}

}  // namespace spmv
