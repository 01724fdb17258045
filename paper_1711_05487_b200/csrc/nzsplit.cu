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
#include "common.cuh"
#include "internal.h"

namespace spmv {

constexpr int kNzThreads = 256;
constexpr int kNzWarps = kNzThreads / 32;

template <typename RP>
struct NzP {
  const RP* rpc;
  const int32_t* col;
  const double* val;
  const double* x;
  double* y;
  const int32_t* rowmap;
  const int32_t* tile_q;
  int32_t* carry_row;
  double* carry_val;
  int64_t nnz, T;
  int zero_gaps;
};

__device__ __forceinline__ void ld256_s32(const int32_t* p, int (&c)[8]) {
  asm volatile("ld.global.nc.L1::no_allocate.v8.s32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(c[0]), "=r"(c[1]), "=r"(c[2]), "=r"(c[3]), "=r"(c[4]), "=r"(c[5]), "=r"(c[6]), "=r"(c[7])
               : "l"(p));
}
__device__ __forceinline__ void ld256_f64(const double* p, double& a, double& b, double& c, double& d) {
  asm volatile("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
               : "=d"(a), "=d"(b), "=d"(c), "=d"(d)
               : "l"(p));
}

template <typename RP>
__global__ void __launch_bounds__(kNzThreads, 4) nzsplit_kernel(const NzP<RP> p) {
  __shared__ __align__(16) uint32_t emask_s[kNzWarps][8];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t* em = emask_s[w];
  const int64_t nw = (int64_t)gridDim.x * kNzWarps;
  for (int64_t k = (int64_t)blockIdx.x * kNzWarps + w; k < p.T; k += nw) {
    const int64_t t0 = k * kNzTile;
    const int cnt = (int)((p.nnz - t0) < kNzTile ? (p.nnz - t0) : kNzTile);
    const int e0 = lane * 8;
    int c[8];
    double v[8];
    if (e0 + 8 <= cnt) {
      ld256_s32(p.col + t0 + e0, c);
      ld256_f64(p.val + t0 + e0, v[0], v[1], v[2], v[3]);
      ld256_f64(p.val + t0 + e0 + 4, v[4], v[5], v[6], v[7]);
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const bool ok = e0 + i < cnt;
        c[i] = ok ? ld_stream(p.col + t0 + e0 + i) : -1;
        v[i] = ok ? ld_stream(p.val + t0 + e0 + i) : 0.0;
      }
    }
    double xv[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) xv[i] = c[i] >= 0 ? ld_x(p.x + c[i]) : 0.0;

    // rows ending in the tile: q in [q0, q1), end position rpc[q+1]-1
    const int64_t q0 = ld_ro(p.tile_q + k), q1 = ld_ro(p.tile_q + k + 1);
    const int n_end = (int)(q1 - q0);
    if (lane < 8) em[lane] = 0u;
    __syncwarp();
    for (int j = lane; j < n_end; j += 32) {
      const int64_t q = q0 + j;
      const int e = (int)((int64_t)ld_ro(p.rpc + q + 1) - 1 - t0);
      atomicOr(&em[e >> 5], 1u << (e & 31));
      if (p.zero_gaps) {
        const int32_t ra = ld_ro(p.rowmap + q), rb = ld_ro(p.rowmap + q + 1);
        for (int32_t r = ra + 1; r < rb; ++r) p.y[r] = 0.0;
      }
    }
    if (k == 0 && p.zero_gaps) {
      const int32_t r0 = ld_ro(p.rowmap);
      for (int32_t r = lane; r < r0; r += 32) p.y[r] = 0.0;
    }
    __syncwarp();
    const uint4 m0 = *reinterpret_cast<const uint4*>(em);
    const uint4 m1 = *reinterpret_cast<const uint4*>(em + 4);
    const uint32_t words[8] = {m0.x, m0.y, m0.z, m0.w, m1.x, m1.y, m1.z, m1.w};
    const int wi = lane >> 2, sh = (lane & 3) * 8;
    uint32_t word = 0;
    int before = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (i < wi) before += __popc(words[i]);
      if (i == wi) word = words[i];
    }
    before += __popc(word & ((1u << sh) - 1u));
    const uint32_t my = (word >> sh) & 0xffu;

    // lane-sequential sums; the first row end of the lane is completed after
    // the cross-lane scan, later ones are complete inside the lane
    const int64_t qf = q0 + before;
    double acc = 0.0, head = 0.0;
    int ne = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      acc = fma(v[i], xv[i], acc);
      if ((my >> i) & 1u) {
        if (ne == 0) head = acc;
        else p.y[ld_ro(p.rowmap + qf + ne)] = acc;
        ++ne;
        acc = 0.0;
      }
    }
    // segmented inclusive scan of the lane tails, reset at lanes with a row end
    double S = acc;
    int f = ne > 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double su = __shfl_up_sync(0xffffffffu, S, o);
      const int fu = __shfl_up_sync(0xffffffffu, f, o);
      if (lane >= o) {
        if (!f) S += su;
        f |= fu;
      }
    }
    const double cin = __shfl_up_sync(0xffffffffu, S, 1);
    if (ne > 0) p.y[ld_ro(p.rowmap + qf)] = (lane > 0 ? cin : 0.0) + head;
    if (lane == 31) {
      if (cnt == kNzTile && !(my & 0x80u)) {
        p.carry_row[k] = ld_ro(p.rowmap + q1);
        p.carry_val[k] = S;
      } else {
        p.carry_row[k] = -1;
      }
    }
  }
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

void launch_nz_tiles(const NzPlan& z, cudaStream_t s) {
  const int g = (int)((z.T + 1 + kNT - 1) / kNT);
  if (z.V.rp_bytes == 8)
    nz_tile_rows_kernel<int64_t><<<g, kNT, 0, s>>>((const int64_t*)z.rpc, z.mc, z.T, z.tile_q);
  else
    nz_tile_rows_kernel<int32_t><<<g, kNT, 0, s>>>((const int32_t*)z.rpc, z.mc, z.T, z.tile_q);
  set_i32_kernel<<<1, 1, 0, s>>>(const_cast<int32_t*>(z.rowmap) + z.mc, (int32_t)z.m_out);
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
  p.carry_row = z.carry_row;
  p.carry_val = z.carry_val;
  p.nnz = z.V.nnz;
  p.T = z.T;
  p.zero_gaps = z.zero_gaps ? 1 : 0;
  return p;
}

int nz_prepare(const NzPlan& z, int sm_count) {
  int per_sm = 0;
  const cudaError_t e = z.V.rp_bytes == 8
                            ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, nzsplit_kernel<int64_t>, kNzThreads, 0)
                            : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, nzsplit_kernel<int32_t>, kNzThreads, 0);
  if (e != cudaSuccess || per_sm < 1) return -1;
  int64_t grid = (int64_t)sm_count * per_sm;
  const int64_t need = (z.T + kNzWarps - 1) / kNzWarps;
  if (grid > need) grid = need;
  return (int)(grid > 0 ? grid : 1);
}

int launch_nz_plan(const NzPlan& z, const double* x, double* y, int stage, cudaStream_t s) {
  int n = 0;
  if (z.T == 0) {
    if (stage != 2 && z.zero_gaps && z.m_out > 0) cudaMemsetAsync(y, 0, (size_t)z.m_out * 8, s);
    return 0;
  }
  if (stage != 2) {
    if (z.V.rp_bytes == 8) nzsplit_kernel<int64_t><<<z.grid, kNzThreads, 0, s>>>(nz_params<int64_t>(z, x, y));
    else nzsplit_kernel<int32_t><<<z.grid, kNzThreads, 0, s>>>(nz_params<int32_t>(z, x, y));
    ++n;
  }
  if (stage != 1 && z.T > 1) n += launch_fixup(z.carry_row, z.carry_val, z.T, y, 0, z.max_run, s);
  return n;
}

}  // namespace spmv
