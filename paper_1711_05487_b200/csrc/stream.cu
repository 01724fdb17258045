// stream.cu -- cta_stream: the MB-class kernel (Table II "vectorization" +
// delta colind) re-designed for sm_100a; also the engine of the
// long_row_split bins.
//
// Persistent, warp-specialised CTAs: 1 producer warp + W = 4 consumer warps,
// one consumer WARP per tile. Tile k covers the fixed nonzero range
// [k*C, min((k+1)*C, nnz)) and owns rows [R_k, R_{k+1}).
//  * producer warp (one lane): TMA bulk copies (cp.async.bulk + mbarrier
//    complete_tx, L2 evict_first) of the tile's values, colind (or 16-bit
//    deltas), rowptr slice and (D16) row heads into the consumer warp's smem
//    stage. Tile i of the CTA goes to stage i % S and warp i % W; S is a
//    multiple of W, so a stage's mbarrier phases are consumed in order. One
//    stage per warp by default: on B200 more resident warps beat a deeper
//    ring (the x gathers are latency-bound). No __syncthreads after set-up.
//  * row-step mode (default): VS lanes per row, lanes of a warp walk
//    consecutive rows in step (VS = 1 for rows up to 32 nonzeros), so a
//    banded matrix gathers x from 2-3 cache lines per warp instruction; each
//    lane keeps 8 predicated gathers in flight. D16 rows are decoded per lane
//    piece (head or tile anchor + subgroup scan + running sum).
//  * segmented mode (option): products first, then a warp-balanced walk of
//    row ends over 16-element lane ranges (any row-length mix).
//  Rows are written to y[rowmap[r]] (identity without a map). In row-step
//  mode the row entering a tile is the tile's carry; in segmented mode the
//  row leaving it is; the ordered fix-up kernel adds carries in tile order.
#include <cstdlib>
#include <algorithm>

#include "common.cuh"
#include "internal.h"
#include "iterfuse.cuh"

namespace spmv {

#ifndef SPMV_STREAM_LB
#define SPMV_STREAM_LB 5
#endif
#ifndef SPMV_D16_LB
#define SPMV_D16_LB 5
#endif
constexpr int kConsumerWarps = kStreamConsumerWarps;
constexpr int kStreamThreads = 32 * (kConsumerWarps + 1);

struct TileMeta {
  int64_t t0;       // first nonzero of the tile
  int32_t cnt;      // nonzeros in the tile
  int32_t voff, ioff;  // position of nonzero t0 in the staged values / index arrays
  int32_t R0, R1;   // owned rows [R0, R1)
  int32_t rp_off;   // element offset of row max(R0-1,0) in the staged rowptr slice; -1 = read global
  int32_t hd_off;   // element offset of row R0 in the staged head slice; -1 = read global
  int32_t anchor;   // D16: absolute column of nonzero k*C (nnz-aligned tiles)
};

__host__ __device__ __forceinline__ size_t al128(size_t v) { return (v + 127) & ~(size_t)127; }

struct StreamLayout {
  size_t vals, idx, rp, hd, stage, full, empty, meta, prod, total;
  uint32_t rp_cap, hd_cap;  // bytes
};

// rows_cap: rowptr entries staged per tile (plan-time, from the view's
// average row length); tiles with more rows read rowptr from global memory.
__host__ __device__ inline StreamLayout stream_layout(int64_t C, int stages, int rp_bytes, int rows_cap, bool d16,
                                                      bool seg) {
  StreamLayout L;
  L.rp_cap = (uint32_t)(((size_t)(rows_cap + 2) * rp_bytes + 32 + 15) & ~(size_t)15);
  L.hd_cap = d16 ? (uint32_t)(((size_t)(rows_cap + 2) * 4 + 32 + 15) & ~(size_t)15) : 0u;
  // slack past C: a row-aligned tile's copies start at the 128-B line of its
  // first element (values: <= 15 entries before it, int32 colind: <= 31);
  // the D16 stream keeps 128 entries (its branch-free decode reads up to 8
  // codes past a row end)
  L.vals = 0;
  L.idx = al128((size_t)(C + 16) * 8);
  L.rp = al128(L.idx + (size_t)(C + (d16 ? 128 : 32)) * (d16 ? 2 : 4));
  L.hd = al128(L.rp + L.rp_cap);
  L.stage = al128(L.hd + L.hd_cap);
  size_t o = L.stage * stages;
  L.full = o; o += 8 * (size_t)stages;
  L.empty = o; o += 8 * (size_t)stages;
  L.meta = al128(o); o = L.meta + sizeof(TileMeta) * (size_t)stages;
  L.prod = al128(o);
  o = L.prod + (seg ? (size_t)kConsumerWarps * C * 8 : 0);
  L.total = al128(o);
  return L;
}

size_t stream_smem_bytes(int64_t C, int stages, int rp_bytes, int rows_cap, bool d16, bool seg) {
  return stream_layout(C, stages, rp_bytes, rows_cap, d16, seg).total;
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// escape-coded delta (kEsc0 + i -> the plan's i-th large delta)
struct EscTab {
  int32_t v[kEscMax];
};
// (esc: the table in shared memory -- a dynamically indexed kernel-parameter
// array spills to local memory)
// ESC is a template flag: plans without escape codes keep the plain add
// (any per-element check -- a select with a predicated LDS or a branch --
// measured ~25 % slower on a 27-point stencil, 451 vs 352 us)
template <bool ESC>
__device__ __forceinline__ int d16_delta(uint32_t code, const int32_t* esc) {
  if constexpr (ESC) return code >= (uint32_t)kEsc0 ? esc[code - kEsc0] : (int)code;
  else return (int)code;
}

template <typename RP>
struct StreamP {
  const RP* rp;
  const void* idx;  // int32 colind or uint16 dcol
  const int32_t* head;
  const int32_t* anchor;
  const double* val;
  const double* x;
  double* y;
  const int32_t* rowmap;
  const int32_t* tile_row;
  const int64_t* tile_nz;  // row-aligned tiles: first nonzero of tile k (= rowptr[tile_row[k]])
  int32_t* carry_row;
  double* carry_val;
  int64_t nnz, C, T;  // T: end of the tile range
  int64_t n_cols;     // (checked build only)
  int64_t k0;         // first tile of the range
  IterOut it;         // row-aligned tiles: iterated-mode epilogue (iterfuse.cuh)
  int stages, rows_cap;
  int aligned;  // 1: row-aligned tiles (no row crosses a tile, no carries)
  int l2pf;     // 1: the producer prefetches the stage's next tile into L2
  EscTab esc;   // D16: escape table (sorted large deltas)
};

template <typename RP>
__device__ __forceinline__ int64_t out_row(const StreamP<RP>& p, int64_t r) {
  return p.rowmap ? (int64_t)ld_ro(p.rowmap + r) : r;
}

// D16 columns of one row's lane piece: calls f(t, col) for t in the lane's
// contiguous sub-range of [ls, le). Every lane of the VS-group must call it.
template <int VS, bool ESC, typename F>
__device__ __forceinline__ void d16_row_cols(const uint16_t* __restrict__ d_s, int ls, int le, int lane, int base,
                                             const int32_t* e, F&& f) {
  const int len = le - ls;
  const int chunk = (len + VS - 1) / VS;
  int a = ls + lane * chunk;
  a = a < le ? a : le;
  int b = a + chunk;
  b = b < le ? b : le;
  uint32_t ps = 0;
  for (int t = a; t < b; ++t) ps += (t == ls) ? 0u : (uint32_t)d16_delta<ESC>(d_s[t], e);
  uint32_t inc = ps;
#pragma unroll
  for (int o = 1; o < VS; o <<= 1) {
    const uint32_t v = __shfl_up_sync(0xffffffffu, inc, o, VS);
    if (lane >= o) inc += v;
  }
  int c = base + (int)(inc - ps);
#pragma unroll 4
  for (int t = a; t < b; ++t) {
    c += (t == ls) ? 0 : d16_delta<ESC>(d_s[t], e);
    f(t, c);
  }
}

// Segmented consumer mode: products first (lane l owns elements l + 32u, 16
// independent gathers in flight), stored XOR-swizzled so the contiguous
// 16-element reads of the row pass are bank-conflict free; lane l then walks
// elements [16l, 16l+16) and the row ends inside them; rows cut by lane edges
// are combined by a segmented shuffle scan in lane order. A row is written by
// the tile where it ENDS; the row crossing the tile end is the tile's carry.
__device__ __forceinline__ int seg_swz(int e) { return e ^ ((e >> 4) & 15); }

template <typename RP, typename Rows>
__device__ __forceinline__ void seg_tile(const StreamP<RP>& p, const double* __restrict__ vals_s,
                                         const int32_t* __restrict__ idx_s, double* __restrict__ prod,
                                         const Rows& rows, int64_t fr, int nloc, int64_t t0, int cnt, int64_t k,
                                         int lane) {
  for (int ub = 0; ub < cnt; ub += 512) {
    int c[16];
    double xv[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int e = ub + lane + 32 * u;
      c[u] = e < cnt ? idx_s[e] : -1;
    }
#pragma unroll
    for (int u = 0; u < 16; ++u) xv[u] = c[u] >= 0 ? ld_x(p.x + c[u]) : 0.0;
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int e = ub + lane + 32 * u;
      if (e < cnt) prod[seg_swz(e)] = vals_s[e] * xv[u];
    }
  }
  __syncwarp();
  const int E = (int)(p.C >> 5);
  const int a = lane * E < cnt ? lane * E : cnt;
  const int b = a + E < cnt ? a + E : cnt;
  auto rend = [&](int q) -> int64_t { return rows(fr + q + 1) - t0; };  // unclamped
  int q = 0;
  if (lane > 0) {  // first row with end > a
    int lo = 0, hi = nloc;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (rend(mid) > a) hi = mid; else lo = mid + 1;
    }
    q = lo;
  }
  double acc = 0.0, first_val = 0.0;
  int first = -1;
  int64_t e_q = q < nloc ? rend(q) : INT64_MAX;
  for (int t = a; t < b; ++t) {
    while (e_q <= t) {
      if (first < 0) { first = q; first_val = acc; }
      else p.y[out_row(p, fr + q)] = acc;
      acc = 0.0;
      ++q;
      e_q = q < nloc ? rend(q) : INT64_MAX;
    }
    acc += prod[seg_swz(t)];
  }
  while (e_q <= b) {
    if (first < 0) { first = q; first_val = acc; }
    else p.y[out_row(p, fr + q)] = acc;
    acc = 0.0;
    ++q;
    e_q = q < nloc ? rend(q) : INT64_MAX;
  }
  int key = (q < nloc && b > a) ? q : -1 - lane;
  double S = acc;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int k2 = __shfl_up_sync(0xffffffffu, key, o);
    const double S2 = __shfl_up_sync(0xffffffffu, S, o);
    if (lane >= o && k2 == key) S += S2;
  }
  const int pk = __shfl_up_sync(0xffffffffu, key, 1);
  const double pS = __shfl_up_sync(0xffffffffu, S, 1);
  if (first >= 0) p.y[out_row(p, fr + first)] = (lane > 0 && pk == first) ? pS + first_val : first_val;
  const int key31 = __shfl_sync(0xffffffffu, key, 31);
  const double S31 = __shfl_sync(0xffffffffu, S, 31);
  if (lane == 0) {
    if (key31 >= 0) {
      p.carry_row[k] = (int32_t)out_row(p, fr + key31);
      p.carry_val[k] = S31;
    } else {
      p.carry_row[k] = -1;
    }
  }
}

#ifndef STREAM_UNR1
#define STREAM_UNR1 8
#endif
constexpr int kStreamUnroll1 = STREAM_UNR1;  // gathers in flight per lane, one lane per row (VS = 1)

// y[r] *= f over the rows of this warp's tiles (rare launch of the iterated
// mode whose exact rescale factor is not 1; out of line, off the tile loop)
__device__ __noinline__ void stream_rescale_rows(const int32_t* tile_row, double* y, int64_t k0, int64_t T, int CW,
                                                 double f) {
  const int w = (threadIdx.x >> 5) - 1, lane = threadIdx.x & 31;
  for (int64_t k = k0 + blockIdx.x + (int64_t)w * gridDim.x; k < T; k += (int64_t)CW * gridDim.x) {
    const int64_t r0 = __ldg(tile_row + k), r1 = __ldg(tile_row + k + 1);
    for (int64_t r = r0 + lane; r < r1; r += 32) y[r] = __ldcg(y + r) * f;
  }
}
// ... and again in the neighbours' replicas the rows were pushed to (MODE 3)
__device__ __noinline__ void stream_rescale_rows_push(const int32_t* tile_row, double* y, int64_t k0, int64_t T,
                                                      int CW, double f, double* plo, int64_t lo_end, double* phi,
                                                      int64_t hi_begin) {
  const int w = (threadIdx.x >> 5) - 1, lane = threadIdx.x & 31;
  for (int64_t k = k0 + blockIdx.x + (int64_t)w * gridDim.x; k < T; k += (int64_t)CW * gridDim.x) {
    const int64_t r0 = __ldg(tile_row + k), r1 = __ldg(tile_row + k + 1);
    for (int64_t r = r0 + lane; r < r1; r += 32) {
      const double v = __ldcg(y + r) * f;
      y[r] = v;
      if (plo && r < lo_end) plo[r] = v;
      if (phi && r >= hi_begin) phi[r] = v;
    }
  }
}

// MODE: 0 = row-step over nnz-aligned tiles, 1 = segmented, 2 = row-step over
// row-aligned tiles (compile-time so the nnz-tile path carries no per-tile
// offsets: measured ~9% faster on C5 than a runtime switch). D16: 0 = int32
// colind, 1 = 16-bit deltas, 2 = 16-bit deltas with escape codes.
// CW: consumer warps per CTA (one smem stage each); 6 for small row-aligned
// stages (C2: 4 CTAs x 6 x 8.8 KB in flight per SM, 31.4 vs 32.5 us with
// 5 x 4), else 4 (C5's 11.4-KB stages: 5 x 4 fills the 228 KB)
template <int VS, typename RP, int D16, int MODE, int CW = kConsumerWarps>
__global__ void __launch_bounds__(32 * (CW + 1),
                                  MODE == 1 ? 4 : (CW != 4 ? 24 / CW : (D16 ? SPMV_D16_LB : SPMV_STREAM_LB)))
    stream_kernel(const StreamP<RP> p) {
  constexpr bool SEG = MODE == 1;
  constexpr bool AL = MODE >= 2;
  constexpr bool PUSH = MODE == 3;  // row-aligned + the multi-shard halo push (IterOut::push_*)
  constexpr bool ESC = D16 == 2;
  extern __shared__ __align__(128) unsigned char smem[];
  const StreamLayout L = stream_layout(p.C, p.stages, (int)sizeof(RP), p.rows_cap, D16, SEG);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.full);
  uint64_t* empty = reinterpret_cast<uint64_t*>(smem + L.empty);
  TileMeta* meta = reinterpret_cast<TileMeta*>(smem + L.meta);
  constexpr int IB = D16 ? 2 : 4;
  constexpr int RPB = (int)sizeof(RP);
  const int S = p.stages;

  pdl_trigger();
  __shared__ int32_t esc_s[D16 ? kEscMax : 1];
  if constexpr (D16) {
    if (threadIdx.x < kEscMax) esc_s[threadIdx.x] = p.esc.v[threadIdx.x];
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (threadIdx.x < 32) {
    // ------------------------------ producer ------------------------------
    if (threadIdx.x == 0) {
      const uint64_t pol = policy_evict_first();
      // tile metadata is prefetched one tile ahead (independent loads issued
      // before waiting on the stage), keeping global latency off the serial
      // producer path
      int64_t nR0 = 0, nR1 = 0, nT0 = 0, nT1 = 0;
      auto fetch = [&](int64_t kk) {
        if (kk < p.T) {
          nR0 = ld_ro(p.tile_row + kk);
          nR1 = ld_ro(p.tile_row + kk + 1);
          if constexpr (AL) {
            nT0 = ld_ro(p.tile_nz + kk);
            nT1 = ld_ro(p.tile_nz + kk + 1);
          }
        }
      };
      fetch(p.k0 + blockIdx.x);
      // L2 prefetch of the tile that will next reuse this stage (S tiles
      // ahead): its DRAM latency then overlaps the consumer's current tile
      // and the later TMA copy hits L2 (metadata fetched one tile earlier)
      int64_t pR0 = 0, pR1 = 0, pT0 = 0, pT1 = 0;
      auto pfetch = [&](int64_t kk) {
        if (p.l2pf && kk < p.T) {
          pR0 = ld_ro(p.tile_row + kk);
          pR1 = ld_ro(p.tile_row + kk + 1);
          if constexpr (AL) {
            pT0 = ld_ro(p.tile_nz + kk);
            pT1 = ld_ro(p.tile_nz + kk + 1);
          }
        }
      };
      pfetch(p.k0 + blockIdx.x + (int64_t)S * gridDim.x);
      int i = 0;
      for (int64_t k = p.k0 + blockIdx.x; k < p.T; k += gridDim.x, ++i) {
        const int s = i % S;
        const int64_t R0 = nR0, R1 = nR1, aT0 = nT0, aT1 = nT1;
        fetch(k + gridDim.x);
        const int64_t k2 = k + (int64_t)S * gridDim.x;
        if (p.l2pf && k2 < p.T) {
          int64_t u0, u1;
          if constexpr (AL) {
            u0 = pT0;
            u1 = pT1;
          } else {
            u0 = k2 * p.C;
            u1 = (u0 + p.C) < p.nnz ? (u0 + p.C) : p.nnz;
          }
          if (u1 > u0) {
            const int64_t a0 = u0 & ~15ll, a1 = (u1 + 15) & ~15ll;  // whole 128-B lines of values
            bulk_prefetch_l2(p.val + a0, (uint32_t)((a1 - a0) * 8));
            const int64_t b0 = (u0 * IB) & ~127ll, b1 = (u1 * IB + 127) & ~127ll;
            bulk_prefetch_l2(static_cast<const unsigned char*>(p.idx) + b0, (uint32_t)(b1 - b0));
          }
          const int64_t r0 = ((pR0 > 0 ? pR0 - 1 : 0) * RPB) & ~127ll, r1 = ((pR1 + 1) * RPB + 127) & ~127ll;
          bulk_prefetch_l2(reinterpret_cast<const unsigned char*>(p.rp) + r0, (uint32_t)(r1 - r0));
        }
        pfetch(k2 + gridDim.x);
        if (i >= S) mbar_wait(&empty[s], (uint32_t)(((i / S) - 1) & 1));
        // nnz-aligned tile [k*C, ...) or row-aligned tile [rowptr[R0], rowptr[R1])
        // (copies rounded out to 16 B; voff/ioff = offsets of t0 in the stage)
        int64_t t0, cnt, v0, i0;
        if constexpr (AL) {
          t0 = aT0;
          cnt = aT1 - aT0;
          v0 = t0 & ~15ll;                    // 128-B line of the first value
          i0 = t0 & ~(int64_t)(128 / IB - 1);  // 128-B line of the first index
        } else {
          t0 = k * p.C;
          cnt = (p.nnz - t0) < p.C ? (p.nnz - t0) : p.C;
          v0 = i0 = t0;
        }
        const uint32_t vb = cnt > 0 ? (uint32_t)(((t0 + cnt - v0) * 8 + 15) & ~15ll) : 0u;
        const uint32_t ib = cnt > 0 ? (uint32_t)(((t0 + cnt - i0) * IB + 15) & ~15ll) : 0u;
        const int64_t fr0 = R0 > 0 ? R0 - 1 : 0;
        const int64_t b0 = (fr0 * RPB) & ~15ll, b1 = ((R1 + 1) * RPB + 15) & ~15ll;
        const bool rp_ok = (b1 - b0) <= (int64_t)L.rp_cap;
        uint32_t hb = 0;
        int64_t h0 = 0;
        TileMeta mt;
        mt.t0 = t0;
        mt.cnt = (int32_t)cnt;
        mt.voff = (int32_t)(t0 - v0);
        mt.ioff = (int32_t)(t0 - i0);
        mt.R0 = (int32_t)R0;
        mt.R1 = (int32_t)R1;
        mt.rp_off = rp_ok ? (int32_t)((fr0 * RPB - b0) / RPB) : -1;
        mt.hd_off = -1;
        mt.anchor = 0;
        if (D16) {
          h0 = (R0 * 4) & ~15ll;
          const int64_t h1 = (R1 * 4 + 15) & ~15ll;
          const bool hd_ok = (h1 - h0) <= (int64_t)L.hd_cap;
          hb = hd_ok ? (uint32_t)(h1 - h0) : 0u;
          mt.hd_off = hd_ok ? (int32_t)((R0 * 4 - h0) / 4) : -1;
          mt.anchor = ld_ro(p.anchor + k);
        }
        meta[s] = mt;
        unsigned char* st = smem + L.stage * s;
        mbar_arrive_expect_tx(&full[s], vb + ib + (rp_ok ? (uint32_t)(b1 - b0) : 0u) + hb);
        if (cnt > 0) {
          bulk_g2s(st + L.vals, p.val + v0, vb, &full[s], pol);
          bulk_g2s(st + L.idx, static_cast<const unsigned char*>(p.idx) + i0 * IB, ib, &full[s], pol);
        }
        if (rp_ok) bulk_g2s(st + L.rp, reinterpret_cast<const unsigned char*>(p.rp) + b0, (uint32_t)(b1 - b0),
                            &full[s], pol);
        if (hb) bulk_g2s(st + L.hd, reinterpret_cast<const unsigned char*>(p.head) + h0, hb, &full[s], pol);
      }
    } else if (AL && p.it.cta_only && p.it.prev_part && blockIdx.x == gridDim.x - 1) {
      iter_lag_fold_lanes(p.it);  // lagged iteration: the previous launch's norm (lanes 1..31)
    }
    return;
  }

  // ------------------------------- consumers --------------------------------
  // (the producer streams plan-constant matrix data only; x, y and the
  // carries wait for the previous kernel in the stream)
  pdl_wait();
  const int w = (threadIdx.x >> 5) - 1;
  const int lane32 = threadIdx.x & 31;
  constexpr int GPW = 32 / VS;
  const int lane = lane32 % VS;
  const int gi = lane32 / VS;
  // iterated mode (AL): the launch's exact factor, fetched by one thread;
  // rows rescaled after the tiles in the rare launch where it is not 1
  __shared__ double f_s;
  if constexpr (AL)
    if (threadIdx.x == 32 && p.it.cta_part) f_s = iter_factor(p.it);
  double sqa = 0.0;  // (AL) this lane's squares over all its rows, its tiles in order (one warp sum at the end)
  for (int i = w;; i += CW) {
    const int64_t k = p.k0 + blockIdx.x + (int64_t)i * gridDim.x;
    if (k >= p.T) break;
    const int s = i % S;
    mbar_wait(&full[s], (uint32_t)((i / S) & 1));
    const TileMeta mt = meta[s];
    unsigned char* st = smem + L.stage * s;
    const RP* rp_s = reinterpret_cast<const RP*>(st + L.rp);
    const double* vals_s;
    const unsigned char* idx_b;
    int64_t t0, t1;
    int cnt;
    if constexpr (AL) {
      t0 = mt.t0;
      cnt = mt.cnt;
      t1 = t0 + cnt;
      vals_s = reinterpret_cast<const double*>(st + L.vals) + mt.voff;
      idx_b = st + L.idx + (size_t)mt.ioff * IB;
    } else {
      t0 = k * p.C;
      t1 = (t0 + p.C) < p.nnz ? (t0 + p.C) : p.nnz;
      cnt = (int)(t1 - t0);
      vals_s = reinterpret_cast<const double*>(st + L.vals);
      idx_b = st + L.idx;
    }
    const int64_t R0 = mt.R0, R1 = mt.R1;
    const int64_t fr0 = R0 > 0 ? R0 - 1 : 0;
    auto rows = [&](int64_t r) -> int64_t {
      return mt.rp_off >= 0 ? (int64_t)rp_s[r - fr0 + mt.rp_off] : (int64_t)ld_ro(p.rp + r);
    };
    const bool incoming = R0 > 0 && rows(R0) > t0;
    const int64_t fr = R0 - (incoming ? 1 : 0);
    const int nloc = (int)(R1 - R0) + (incoming ? 1 : 0);

    if constexpr (SEG) {
      seg_tile(p, vals_s, reinterpret_cast<const int32_t*>(idx_b),
               reinterpret_cast<double*>(smem + L.prod) + (size_t)w * p.C, rows, fr, nloc, t0, cnt, k, lane32);
    } else {
      for (int qb = 0; qb < nloc; qb += GPW) {
        const int q = qb + gi;
        const bool active = q < nloc;
        int ls = 0, le = 0;
        int64_t r = 0;
        if (active) {
          r = fr + q;
          const int64_t a = rows(r), b = rows(r + 1);
          ls = (int)((a > t0 ? a : t0) - t0);
          le = (int)((b < t1 ? b : t1) - t0);
          SPMV_CHECK(ls >= 0 && ls <= le && le <= cnt);
        }
        double acc;
        if constexpr (!D16) {
          // batches of UN predicated elements per lane: UN independent gathers
          // in flight (values read from smem after the gathers are issued)
          constexpr int UN = VS == 1 ? kStreamUnroll1 : 8;
          const int32_t* idx_s = reinterpret_cast<const int32_t*>(idx_b);
          double a0 = 0.0, a1 = 0.0;
          for (int l0 = ls + lane; l0 < le; l0 += UN * VS) {
            double xv[UN];
#pragma unroll
            for (int u = 0; u < UN; ++u) {
              const int l = l0 + u * VS;
              SPMV_CHECK(l >= le || (idx_s[l] >= 0 && (int64_t)idx_s[l] < p.n_cols));
#ifdef D8_EXP_XHIT  // timing experiment only: every gather an L1 hit (wrong results)
              xv[u] = l < le ? ld_x(p.x + (idx_s[l] & 2047)) : 0.0;
#else
              xv[u] = l < le ? ld_x(p.x + idx_s[l]) : 0.0;
#endif
            }
#pragma unroll
            for (int u = 0; u < UN; u += 2) {
              const int l = l0 + u * VS;
              a0 = fma(l < le ? vals_s[l] : 0.0, xv[u], a0);
              a1 = fma(l + VS < le ? vals_s[l + VS] : 0.0, xv[u + 1], a1);
            }
          }
          acc = a0 + a1;
        } else {
          const uint16_t* d_s = reinterpret_cast<const uint16_t*>(idx_b);
          const int32_t* hd_s = reinterpret_cast<const int32_t*>(st + L.hd);
          int base = mt.anchor;
          if (active && (!incoming || q > 0))
            base = mt.hd_off >= 0 ? hd_s[r - R0 + mt.hd_off] : ld_ro(p.head + r);
          double a0 = 0.0;
          if constexpr (VS == 1) {
            // one lane per row: running column sum, batches of 8 gathers
            double a1 = 0.0;
            int c = base;
            for (int l0 = ls; l0 < le; l0 += 8) {
              // branch-free decode: the 8 codes are read unconditionally (the
              // stage's index area has >= 64 entries of slack past any tile
              // end; a stale code indexes inside the 64-entry escape table)
              // and masked by selects -- a per-element `if` compiled to a
              // branch + reconvergence around every LDS.U16
              uint32_t dd[8];
#pragma unroll
              for (int u = 0; u < 8; ++u) dd[u] = d_s[l0 + u];
              int cc[8];
              double xv[8];
#pragma unroll
              for (int u = 0; u < 8; ++u) {
                const int l = l0 + u;
                const int d = d16_delta<ESC>(dd[u], esc_s);
                c += (l > ls && l < le) ? d : 0;
                cc[u] = c;
              }
#pragma unroll
              for (int u = 0; u < 8; ++u) xv[u] = l0 + u < le ? ld_x(p.x + cc[u]) : 0.0;
#pragma unroll
              for (int u = 0; u < 8; u += 2) {
                const int l = l0 + u;
                a0 = fma(l < le ? vals_s[l] : 0.0, xv[u], a0);
                a1 = fma(l + 1 < le ? vals_s[l + 1] : 0.0, xv[u + 1], a1);
              }
            }
            a0 += a1;
          } else {
            d16_row_cols<VS, ESC>(d_s, ls, le, lane, base, esc_s,
                             [&](int t, int c) { a0 = fma(vals_s[t], ld_x(p.x + c), a0); });
          }
          acc = a0;
        }
        acc = group_sum<VS>(acc);
        if (active && lane == 0) {
          if (incoming && q == 0) {
            p.carry_row[k] = (int32_t)out_row(p, r);
            p.carry_val[k] = acc;
          } else {
            if constexpr (PUSH) iter_store(p.it, p.y, out_row(p, r), acc);
            else p.y[out_row(p, r)] = acc;
            if constexpr (AL) sqa = fma(acc, acc, sqa);
          }
        }
      }
      if (!incoming && lane32 == 0) p.carry_row[k] = -1;
    }
    __syncwarp();
    if (lane32 == 0) mbar_arrive(&empty[s]);
  }
  if constexpr (AL) {
    double wsq = p.it.cta_part ? warp_sum(sqa) : 0.0;  // fixed butterfly
    if (p.it.cta_part) {
      asm volatile("bar.sync 1, %0;" ::"r"(32 * CW) : "memory");
      const double f = f_s;
      if (f != 1.0) {  // rescale the rows this warp wrote (rowmap is null on this path; out of line)
        if constexpr (PUSH)
          stream_rescale_rows_push(p.tile_row, p.y, p.k0, p.T, CW, f, p.it.push_lo, p.it.push_lo_end, p.it.push_hi,
                                   p.it.push_hi_begin);
        else
          stream_rescale_rows(p.tile_row, p.y, p.k0, p.T, CW, f);
        wsq *= f * f;  // exact: f is a power of two
      }
    }
    if constexpr (PUSH) __threadfence_system();  // the peer stores, before the partials / kernel end
    iter_epilogue<32 * CW>(p.it, wsq);
  }
}

template <typename RP>
static StreamP<RP> make_params(const StreamPlan& sp, const double* x, double* y) {
  StreamP<RP> p;
  p.rp = (const RP*)sp.V.rowptr;
  p.idx = sp.dcol ? (const void*)sp.dcol : (const void*)sp.V.col;
  p.head = sp.head;
  p.anchor = sp.anchor;
  p.val = sp.V.val;
  p.x = x;
  p.y = y;
  p.rowmap = sp.rowmap;
  p.tile_row = sp.tile_row;
  p.tile_nz = sp.tile_nz;
  p.carry_row = sp.carry_row;
  p.carry_val = sp.carry_val;
  p.nnz = sp.V.nnz;
  p.n_cols = sp.V.n_cols;
  p.C = sp.C;
  p.T = sp.T;
  p.k0 = sp.k0;
  p.it = sp.it;
  p.stages = sp.stages;
  p.rows_cap = sp.rows_cap;
  p.aligned = sp.aligned ? 1 : 0;
  p.l2pf = sp.l2pf ? 1 : 0;
  for (int i = 0; i < kEscMax; ++i) p.esc.v[i] = i < sp.n_esc ? sp.esc[i] : 0;
  return p;
}

template <int VS, typename RP, int D16, int MODE, int CW>
static int stream_prepare_t(const StreamPlan& sp, int sm_count) {
  const size_t smem = stream_smem_bytes(sp.C, sp.stages, sizeof(RP), sp.rows_cap, D16, MODE == 1);
  if (cudaFuncSetAttribute(stream_kernel<VS, RP, D16, MODE, CW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem) != cudaSuccess)
    return -1;
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, stream_kernel<VS, RP, D16, MODE, CW>, 32 * (CW + 1),
                                                    smem) != cudaSuccess ||
      per_sm < 1)
    return -1;
  if (const char* e = getenv("SPMV_STREAM_CTAS")) per_sm = std::max(1, std::min(per_sm, atoi(e)));  // experiments
  int64_t grid = (int64_t)sm_count * per_sm;
  if (grid > sp.T) grid = sp.T;
  return (int)grid;
}

template <int VS, typename RP, int D16, int MODE, int CW>
static void stream_launch_t(const StreamPlan& sp, const double* x, double* y, cudaStream_t s) {
  const size_t smem = stream_smem_bytes(sp.C, sp.stages, sizeof(RP), sp.rows_cap, D16, MODE == 1);
  launch_pdl(stream_kernel<VS, RP, D16, MODE, CW>, dim3(sp.grid), dim3(32 * (CW + 1)), smem, s,
             make_params<RP>(sp, x, y));
}

template <int VS, typename RP, int D16, int MODE, bool PREP>
static int stream_one(const StreamPlan& sp, int sm_count, const double* x, double* y, cudaStream_t s) {
  // 6 consumer warps only for the plain row-aligned one-lane-per-row kernel
  if constexpr (VS == 1 && D16 <= 1 && MODE >= 2) {
    if (sp.stages == 6) {
      if (PREP) return stream_prepare_t<VS, RP, D16, MODE, 6>(sp, sm_count);
      stream_launch_t<VS, RP, D16, MODE, 6>(sp, x, y, s);
      return 0;
    }
  }
  if (PREP) return stream_prepare_t<VS, RP, D16, MODE, kConsumerWarps>(sp, sm_count);
  stream_launch_t<VS, RP, D16, MODE, kConsumerWarps>(sp, x, y, s);
  return 0;
}

template <typename RP, int D16, int MODE, bool PREP>
static int stream_vs(const StreamPlan& sp, int smc, const double* x, double* y, cudaStream_t s) {
  switch (sp.vs) {
    case 1: return stream_one<1, RP, D16, MODE, PREP>(sp, smc, x, y, s);
    case 2: return stream_one<2, RP, D16, MODE, PREP>(sp, smc, x, y, s);
    case 4: return stream_one<4, RP, D16, MODE, PREP>(sp, smc, x, y, s);
    case 8: return stream_one<8, RP, D16, MODE, PREP>(sp, smc, x, y, s);
    case 16: return stream_one<16, RP, D16, MODE, PREP>(sp, smc, x, y, s);
    default: return stream_one<32, RP, D16, MODE, PREP>(sp, smc, x, y, s);
  }
}

template <typename RP, bool PREP>
static int stream_rp(const StreamPlan& sp, int smc, const double* x, double* y, cudaStream_t s) {
  const int d16 = sp.dcol == nullptr ? 0 : (sp.n_esc > 0 ? 2 : 1);
  if (sp.seg && !d16) return stream_one<1, RP, 0, 1, PREP>(sp, smc, x, y, s);
  if (sp.aligned) {
    // the halo-push instantiation (multi-shard iterated mode): int32 colind,
    // one lane per row only (prepare_push checks stream_push_capable)
    if (sp.vs == 1 && !d16) {
      if (PREP) {
        const int g = stream_one<1, RP, 0, 3, true>(sp, smc, x, y, s);
        if (g < 0) return g;
      } else if (sp.it.push_lo || sp.it.push_hi) {
        return stream_one<1, RP, 0, 3, false>(sp, smc, x, y, s);
      }
    }
    if (d16 == 2) return stream_vs<RP, 2, 2, PREP>(sp, smc, x, y, s);
    return d16 ? stream_vs<RP, 1, 2, PREP>(sp, smc, x, y, s) : stream_vs<RP, 0, 2, PREP>(sp, smc, x, y, s);
  }
  if (d16 == 2) return stream_vs<RP, 2, 0, PREP>(sp, smc, x, y, s);
  return d16 ? stream_vs<RP, 1, 0, PREP>(sp, smc, x, y, s) : stream_vs<RP, 0, 0, PREP>(sp, smc, x, y, s);
}

template <bool PREP>
static int stream_dispatch(const StreamPlan& sp, int smc, const double* x, double* y, cudaStream_t s) {
  if (sp.codes) {  // dictionary-coded 8-bit deltas (d8.cu)
    if (PREP) return d8_prepare(sp, smc);
    launch_d8(sp, x, y, s);
    return 0;
  }
  return sp.V.rp_bytes == 8 ? stream_rp<int64_t, PREP>(sp, smc, x, y, s) : stream_rp<int32_t, PREP>(sp, smc, x, y, s);
}

// the plan's iterated kernel has a halo-push instantiation
bool stream_push_capable(const StreamPlan& sp) {
  if (sp.codes) return d8_push_capable(sp);
  return sp.aligned && !sp.seg && !sp.rowmap && sp.vs == 1 && sp.dcol == nullptr;
}

int stream_prepare(const StreamPlan& sp, int sm_count) {
  return stream_dispatch<true>(sp, sm_count, nullptr, nullptr, nullptr);
}

int launch_stream_plan(const StreamPlan& sp, const double* x, double* y, int stage, cudaStream_t s) {
  int n = 0;
  if (stage != 2) {
    stream_dispatch<false>(sp, 0, x, y, s);
    ++n;
  }
  if (sp.need_fixup && stage != 1) {
    n += launch_fixup(sp.carry_row, sp.carry_val, sp.T, y, 0, sp.max_run, s);
  }
  return n;
}

int launch_stream(const ExecArgs& a, cudaStream_t s) { return launch_stream_plan(a.sp[0], a.x, a.y, a.stage, s); }

int launch_stream_iter(const StreamPlan& sp_in, const double* x, double* y, const IterOut& it, cudaStream_t s) {
  StreamPlan sp = sp_in;
  sp.it = it;
  stream_dispatch<false>(sp, 0, x, y, s);
  return 1;
}

int launch_stream_iter_range(const StreamPlan& sp_in, const double* x, double* y, const IterOut& it, int64_t k0,
                             int64_t k1, cudaStream_t s) {
  if (k1 <= k0) return 0;
  StreamPlan sp = sp_in;
  sp.it = it;
  sp.k0 = k0;
  sp.T = k1;
  if (sp.grid > k1 - k0) sp.grid = (int)(k1 - k0);
  stream_dispatch<false>(sp, 0, x, y, s);
  return 1;
}

// out[0] = largest j with col[j] < lo (-1 if none), out[1] = smallest j with
// col[j] >= hi (nnz if none): the nonzeros that read x outside [lo, hi)
__global__ void __launch_bounds__(kNT) halo_extent_kernel(const int32_t* __restrict__ col, int64_t nnz, int64_t lo,
                                                          int64_t hi, unsigned long long* out) {
  long long jl = -1;
  unsigned long long jh = (unsigned long long)nnz;
  for (int64_t j = (int64_t)blockIdx.x * kNT + threadIdx.x; j < nnz; j += (int64_t)gridDim.x * kNT) {
    const int64_t c = __ldg(col + j);
    if (c < lo) jl = j;
    if (c >= hi && (unsigned long long)j < jh) jh = (unsigned long long)j;
  }
  jl = warp_max(jl);
  jh = warp_min(jh);
  if ((threadIdx.x & 31) == 0) {
    if (jl >= 0) atomicMax(out, (unsigned long long)(jl + 1));  // stored +1 (0 = none)
    atomicMin(out + 1, jh);
  }
}

void launch_halo_extent(const int32_t* col, int64_t nnz, int64_t lo, int64_t hi, unsigned long long* out,
                        cudaStream_t s) {
  if (nnz <= 0) return;
  int64_t g = (nnz + kNT * 8 - 1) / (kNT * 8);
  if (g > dev_sm_count() * 8) g = dev_sm_count() * 8;
  halo_extent_kernel<<<(unsigned)g, kNT, 0, s>>>(col, nnz, lo, hi, out);
}

int launch_stream_range(const StreamPlan& sp_in, const double* x, double* y, int64_t k0, int64_t k1, cudaStream_t s) {
  if (k1 <= k0) return 0;
  StreamPlan sp = sp_in;
  sp.k0 = k0;
  sp.T = k1;
  if (sp.grid > k1 - k0) sp.grid = (int)(k1 - k0);
  stream_dispatch<false>(sp, 0, x, y, s);
  int n = 1;
  // a carry run crossing k0 is split between two ranges' fix-ups: both add
  // to y in stream order (additive), so the row is complete after the later one
  if (sp.need_fixup) n += launch_fixup_range(sp.carry_row + k0, sp.carry_val + k0, k1 - k0, y, s);
  return n;
}

__global__ void tile_rows_count_kernel(int32_t* __restrict__ tile_row, int64_t T, int64_t rpt, int64_t m) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k <= T) tile_row[k] = (int32_t)(k * rpt < m ? k * rpt : m);
}

void launch_tile_rows_count(int32_t* tile_row, int64_t T, int64_t rows_per_tile, int64_t m, cudaStream_t s) {
  tile_rows_count_kernel<<<(unsigned)((T + 1 + kNT - 1) / kNT), kNT, 0, s>>>(tile_row, T, rows_per_tile, m);
}

__global__ void __launch_bounds__(kNT) range_colmax_kernel(const int32_t* __restrict__ col, int64_t a, int64_t b,
                                                           int32_t* out) {
  int32_t mx = -1;
  for (int64_t j = a + (int64_t)blockIdx.x * kNT + threadIdx.x; j < b; j += (int64_t)gridDim.x * kNT)
    mx = max(mx, __ldg(col + j));
  mx = warp_max(mx);
  __shared__ int32_t ws[kNT / 32];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < kNT / 32; ++w) mx = max(mx, ws[w]);
    if (mx >= 0) atomicMax(out, mx);
  }
}

void launch_range_colmax(const int32_t* col, int64_t a, int64_t b, int32_t* out, cudaStream_t s) {
  if (b <= a) return;
  int64_t g = (b - a + kNT * 8 - 1) / (kNT * 8);
  if (g > dev_sm_count() * 8) g = dev_sm_count() * 8;
  range_colmax_kernel<<<(unsigned)g, kNT, 0, s>>>(col, a, b, out);
}

// Export (tests): re-decode the delta colind on the device, one thread per
// row: col = head[r] + running sum of the row's deltas (the head's placeholder
// delta skipped), escape codes through the plan's table -- the same delta
// arithmetic as the kernels (d16_delta), independent of the tiling
// (SURVEY 8(c2) D16 round trip)
template <typename RP>
__global__ void __launch_bounds__(kNT) d16_decode_rows_kernel(const RP* __restrict__ rp, int64_t m,
                                                              const uint16_t* __restrict__ dcol,
                                                              const int32_t* __restrict__ head, int32_t* __restrict__ out,
                                                              const EscTab esc) {
  __shared__ int32_t esc_s[kEscMax];
  if (threadIdx.x < kEscMax) esc_s[threadIdx.x] = esc.v[threadIdx.x];
  __syncthreads();
  const int64_t r = (int64_t)blockIdx.x * kNT + threadIdx.x;
  if (r >= m) return;
  const int64_t a = rp[r], b = rp[r + 1];
  int c = a < b ? head[r] : 0;
  for (int64_t t = a; t < b; ++t) {
    if (t > a) c += d16_delta<true>(dcol[t], esc_s);
    out[t] = c;
  }
}

void launch_d16_decode_export(const StreamPlan& sp, int32_t* out, cudaStream_t s) {
  if (sp.V.nnz == 0 || sp.V.m == 0) return;
  EscTab esc;
  for (int i = 0; i < kEscMax; ++i) esc.v[i] = i < sp.n_esc ? sp.esc[i] : 0;
  const unsigned g = (unsigned)((sp.V.m + kNT - 1) / kNT);
  if (sp.V.rp_bytes == 8)
    d16_decode_rows_kernel<int64_t><<<g, kNT, 0, s>>>((const int64_t*)sp.V.rowptr, sp.V.m, sp.dcol, sp.head, out, esc);
  else
    d16_decode_rows_kernel<int32_t><<<g, kNT, 0, s>>>((const int32_t*)sp.V.rowptr, sp.V.m, sp.dcol, sp.head, out, esc);
}

}  // namespace spmv
