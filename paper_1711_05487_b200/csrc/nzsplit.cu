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

#include "common.cuh"
#include "internal.h"

namespace spmv {

constexpr int kNzThreads = 256;
constexpr int kNzWarps = kNzThreads / 32;
constexpr int64_t kNzChunk = 8;  // tiles per scheduling ticket

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
  unsigned long long* sched;  // [0] tile ticket counter, [1] finished warps (both 0 between launches)
  int64_t nnz, T;
  const RP* orp;  // non-null: zero a gap row only if it is empty in this rowptr (SPLIT: long rows are not ours)
  int zero_gaps, dynamic;
  int64_t chunk;
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

// per-warp TMA stage: colind [256] | values [256] | mbarrier
constexpr int kNzStage = 1024 + 2048 + 128;
size_t nz_smem_bytes(bool tma) { return tma ? (size_t)kNzWarps * kNzStage : 0; }

template <typename RP, bool TMA>
__global__ void __launch_bounds__(kNzThreads, 4) nzsplit_kernel(const NzP<RP> p) {
  extern __shared__ __align__(128) unsigned char nz_smem[];
  __shared__ __align__(16) uint32_t emask_s[kNzWarps][8];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t* em = emask_s[w];
  // TMA mode: the colind / value streams of the warp's next tile are bulk
  // copied into its stage while the current tile gathers x (the stage is
  // drained into registers first), so the streams bypass the L1 miss path
  // and leave it to the x gathers
  unsigned char* st = nz_smem + (size_t)w * kNzStage;
  const int32_t* cs = reinterpret_cast<const int32_t*>(st);
  const double* vs = reinterpret_cast<const double*>(st + 1024);
  uint64_t* bar = reinterpret_cast<uint64_t*>(st + 3072);
  uint64_t pol = 0;
  auto issue = [&](int64_t kk) {
    const int64_t u0 = kk * kNzTile;
    const int64_t n = (p.nnz - u0) < kNzTile ? (p.nnz - u0) : kNzTile;
    const uint32_t cb = (uint32_t)((n * 4 + 15) & ~15ll), vb = (uint32_t)((n * 8 + 15) & ~15ll);
    mbar_arrive_expect_tx(bar, cb + vb);
    bulk_g2s(st, p.col + u0, cb, bar, pol);
    bulk_g2s(st + 1024, p.val + u0, vb, bar, pol);
  };
  // tile scheduling. Default: static round-robin, one tile at a time (warp g
  // takes tiles g, g + W, ...): the tiles in flight form one contiguous
  // window of the streams, which B200 DRAM rewards (C3: 294 us; chunks of 8
  // consecutive tiles per warp 358 us). Option: dynamic tickets claimed one
  // chunk ahead (the last warp to finish resets the counters); measured
  // slower on C3 and C4 (same-address atomics serialise, wider window).
  // (lane 0 holds the raw ticket; it is broadcast only when needed)
  // Tickets hand out chunks of kNzChunk tiles (same-address atomics
  // serialise in L2: one ticket per tile measured 350 us vs 284 us on C3).
  // (p.dynamic == 0: static round-robin chunks, no atomics)
  unsigned long long rr = (unsigned long long)blockIdx.x * kNzWarps + w;
  const unsigned long long nwarps = (unsigned long long)gridDim.x * kNzWarps;
  auto claim = [&]() -> unsigned long long {
    if (!p.dynamic) {
      const unsigned long long t = rr;
      rr += nwarps;
      return t;
    }
    return lane == 0 ? atomicAdd(p.sched, 1ull) : 0ull;
  };
  auto bcast = [&](unsigned long long t) -> int64_t { return (int64_t)__shfl_sync(0xffffffffu, t, 0) * p.chunk; };
  const int64_t kfirst = bcast(claim());
  int64_t kend = kfirst + p.chunk < p.T ? kfirst + p.chunk : p.T;
  unsigned long long tnext = kfirst < p.T ? claim() : (unsigned long long)p.T;
  if constexpr (TMA) {
    if (lane == 0) {
      mbar_init(bar, 1);
      fence_mbar_init();
      pol = policy_evict_first();
      if (kfirst < p.T) issue(kfirst);
    }
    __syncwarp();
  }
  uint32_t phase = 0;
  for (int64_t k = kfirst; k < p.T;) {
    const int64_t t0 = k * kNzTile;
    const int cnt = (int)((p.nnz - t0) < kNzTile ? (p.nnz - t0) : kNzTile);
    const int e0 = lane * 8;
    int c[8];
    double v[8];
    if constexpr (TMA) {
      mbar_wait(bar, phase);
      phase ^= 1u;
      if (e0 + 8 <= cnt) {
        const int4 a = *reinterpret_cast<const int4*>(cs + e0), b = *reinterpret_cast<const int4*>(cs + e0 + 4);
        c[0] = a.x; c[1] = a.y; c[2] = a.z; c[3] = a.w; c[4] = b.x; c[5] = b.y; c[6] = b.z; c[7] = b.w;
#pragma unroll
        for (int i = 0; i < 8; i += 2) {
          const double2 d = *reinterpret_cast<const double2*>(vs + e0 + i);
          v[i] = d.x;
          v[i + 1] = d.y;
        }
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const bool ok = e0 + i < cnt;
          c[i] = ok ? cs[e0 + i] : -1;
          v[i] = ok ? vs[e0 + i] : 0.0;
        }
      }
      __syncwarp();
      const int64_t kn = k + 1 < kend ? k + 1 : bcast(tnext);  // TMA mode needs the next tile now
      if (lane == 0 && kn < p.T) {
        fence_proxy_async();
        issue(kn);
      }
    } else if (e0 + 8 <= cnt) {
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
        for (int32_t r = ra + 1; r < rb; ++r)
          if (!p.orp || ld_ro(p.orp + r + 1) == ld_ro(p.orp + r)) p.y[r] = 0.0;
      }
    }
    if (k == 0 && p.zero_gaps) {
      const int32_t r0 = ld_ro(p.rowmap);
      for (int32_t r = lane; r < r0; r += 32)
        if (!p.orp || ld_ro(p.orp + r + 1) == ld_ro(p.orp + r)) p.y[r] = 0.0;
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
    if (++k >= kend) {
      k = bcast(tnext);
      kend = k + p.chunk < p.T ? k + p.chunk : p.T;
      tnext = k < p.T ? claim() : (unsigned long long)p.T;
    }
  }
  if (p.dynamic && lane == 0) {
    const unsigned long long total = (unsigned long long)gridDim.x * kNzWarps;
    if (atomicAdd(p.sched + 1, 1ull) == total - 1) {
      p.sched[0] = 0ull;
      p.sched[1] = 0ull;
      __threadfence();
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

static bool nz_use_tma() {
  const char* e = getenv("SPMV_NZ_TMA");
  return e ? atoi(e) != 0 : false;  // measured on B200: LDG.256 284 us vs TMA 326 us on C3
}

template <typename RP, bool TMA>
static int nz_occupancy(int* per_sm) {
  const size_t sm = nz_smem_bytes(TMA);
  if (TMA) {
    // carve out only what the resident CTAs need: the rest of the unified
    // 256 KB stays L1 for the x gathers
    cudaFuncSetAttribute(nzsplit_kernel<RP, TMA>, cudaFuncAttributePreferredSharedMemoryCarveout,
                         (int)((4 * (sm + 256 + 1024) * 100 + 228 * 1024 - 1) / (228 * 1024)));
  }
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(per_sm, nzsplit_kernel<RP, TMA>, kNzThreads, sm) ==
                 cudaSuccess
             ? 0
             : -1;
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
  p.sched = z.sched;
  p.nnz = z.V.nnz;
  p.T = z.T;
  p.zero_gaps = z.zero_gaps ? 1 : 0;
  p.orp = (const RP*)z.skip_rp;
  p.dynamic = z.dynamic ? 1 : 0;
  p.chunk = z.chunk;
  return p;
}

int nz_prepare(NzPlan& z, int sm_count) {
  int per_sm = 0;
  if (const char* e = getenv("SPMV_NZ_DYN")) z.dynamic = atoi(e) != 0;
  if (const char* e = getenv("SPMV_NZ_CHUNK")) z.chunk = atoi(e);
  const bool tma = nz_use_tma();
  z.tma = tma;
  const int e = z.V.rp_bytes == 8 ? (tma ? nz_occupancy<int64_t, true>(&per_sm) : nz_occupancy<int64_t, false>(&per_sm))
                                  : (tma ? nz_occupancy<int32_t, true>(&per_sm) : nz_occupancy<int32_t, false>(&per_sm));
  if (e != 0 || per_sm < 1) return -1;
  if (const char* e = getenv("SPMV_NZ_CTAS")) per_sm = std::min(per_sm, atoi(e));
  int64_t grid = (int64_t)sm_count * per_sm;
  const int64_t need = (z.T + kNzWarps - 1) / kNzWarps;
  if (grid > need) grid = need;
  return (int)(grid > 0 ? grid : 1);
}

int launch_nz_plan(const NzPlan& z, const double* x, double* y, int stage, cudaStream_t s) {
  int n = 0;
  if (z.T == 0) {
    if (stage != 2 && z.zero_gaps && !z.skip_rp && z.m_out > 0) cudaMemsetAsync(y, 0, (size_t)z.m_out * 8, s);
    return 0;
  }
  if (stage != 2) {
    const size_t sm = nz_smem_bytes(z.tma);
    if (z.V.rp_bytes == 8) {
      if (z.tma) nzsplit_kernel<int64_t, true><<<z.grid, kNzThreads, sm, s>>>(nz_params<int64_t>(z, x, y));
      else nzsplit_kernel<int64_t, false><<<z.grid, kNzThreads, 0, s>>>(nz_params<int64_t>(z, x, y));
    } else {
      if (z.tma) nzsplit_kernel<int32_t, true><<<z.grid, kNzThreads, sm, s>>>(nz_params<int32_t>(z, x, y));
      else nzsplit_kernel<int32_t, false><<<z.grid, kNzThreads, 0, s>>>(nz_params<int32_t>(z, x, y));
    }
    ++n;
  }
  if (stage != 1 && z.T > 1) n += launch_fixup(z.carry_row, z.carry_val, z.T, y, 0, z.max_run, s);
  return n;
}

}  // namespace spmv
