// tiles.cuh -- device bodies shared by the nnz_split kernel, the column-tiled
// long-row kernel and the fused long_row_split kernel (one work unit each).
#pragma once
#include "common.cuh"
#include "internal.h"

namespace spmv {

// Streams of the nnz tiles: 256-bit non-coherent loads, L1 no-allocate (every
// 32-B sector consumed whole by one instruction). NZ_EVICT_FIRST: also an L2
// evict_first policy, so the once-read matrix streams do not push the
// gathered x out of L2 (B200: C3 267 -> 262 us, C4 117.5 -> 111 us)
#ifndef NZ_EVICT_FIRST
#define NZ_EVICT_FIRST 1
#endif
__device__ __forceinline__ void ld256_s32(const int32_t* p, int (&c)[8]) {
#if NZ_EVICT_FIRST
  asm volatile(
      "{\n.reg .b64 pol;\ncreatepolicy.fractional.L2::evict_first.b64 pol, 1.0;\n"
      "ld.global.nc.L1::no_allocate.L2::cache_hint.v8.s32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], pol;\n}"
      : "=r"(c[0]), "=r"(c[1]), "=r"(c[2]), "=r"(c[3]), "=r"(c[4]), "=r"(c[5]), "=r"(c[6]), "=r"(c[7])
      : "l"(p));
#else
  asm volatile("ld.global.nc.L1::no_allocate.v8.s32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(c[0]), "=r"(c[1]), "=r"(c[2]), "=r"(c[3]), "=r"(c[4]), "=r"(c[5]), "=r"(c[6]), "=r"(c[7])
               : "l"(p));
#endif
}
__device__ __forceinline__ void ld256_f64(const double* p, double* v) {
#if NZ_EVICT_FIRST
  asm volatile(
      "{\n.reg .b64 pol;\ncreatepolicy.fractional.L2::evict_first.b64 pol, 1.0;\n"
      "ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f64 {%0,%1,%2,%3}, [%4], pol;\n}"
      : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3])
      : "l"(p));
#else
  asm volatile("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
               : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3])
               : "l"(p));
#endif
}

// ---- nnz_split warp tile (see nzsplit.cu) -----------------------------------
template <typename RP>
struct NzP {
  const RP* rpc;
  const int32_t* col;
  const double* val;
  const double* x;
  double* y;
  const int32_t* rowmap;
  const int32_t* tile_q;
  const uint32_t* emask;  // [T][8] row-end bits: bit i of tile k set when a row ends at nonzero k*256+i
  const uint64_t* epre;   // [T]: byte w = row ends in words [0, w) of the tile's mask
  int32_t* carry_row;
  double* carry_val;
  const RP* orp;        // non-null: zero a gap row only if it is empty in this rowptr (SPLIT: long rows are not ours)
  const double* xhot;   // hot-x mode: x of the hot columns, [n_hot]
  int64_t nnz, T;  // T: end of the tile range
  int64_t k0;      // first tile of the range (pipelined host execute)
  int n_hot;
  int zero_gaps;
  int skip_wait;  // 1: no griddepcontrol.wait (launched behind a kernel whose CTAs all waited, then triggered)
};

// warp tile k = nonzeros [k*256, (k+1)*256); xh: the hot-x smem table (HOT).
// Per-tile metadata loaded with the streams (one tile ahead where the kernel
// prefetches): the lane's row-end mask word and tile_q[k], both indexed by k,
// so no load of the compute phase waits on another global load except the
// rowmap lookups of the rows it writes.
// y = 0 for the empty rows between compacted rows q and q + 1 (SPLIT: only
// those empty in orp too)
// The n_end gaps after rows q0 .. q0+n_end-1 (MASK path): a short gap
// (<= kGapLane rows) is zeroed by its own lane; long ones by the whole warp --
// their lengths scanned across the lanes, the rows dealt out 32 per step (a
// lane finds its gap by a 5-step search over the scanned lengths). A lane
// per long gap serialises long empty runs (non-empty rows 0.04 % of the
// rows: 10 ms instead of ~60 us on B200 before runs > kNzGapMax made the
// plan clear y first).
template <typename RP>
__device__ __forceinline__ void nz_zero_row(const NzP<RP>& p, int32_t r) {
  if (!p.orp || ld_ro(p.orp + r + 1) == ld_ro(p.orp + r)) p.y[r] = 0.0;
}
constexpr int32_t kGapLane = 64;  // gaps up to this many rows are zeroed by their own lane

template <typename RP>
__device__ __forceinline__ void nz_zero_gaps_warp(const NzP<RP>& p, int64_t q0, int n_end, int lane) {
  auto zero = [&](int32_t r) { nz_zero_row(p, r); };
  for (int jb = 0; jb < n_end; jb += 32) {
    const int j = jb + lane;
    int32_t ra = 0, g = 0;
    if (j < n_end) {
      ra = ld_ro(p.rowmap + q0 + j);
      g = ld_ro(p.rowmap + q0 + j + 1) - ra - 1;
    }
    const bool lng = g > kGapLane;
    if (!lng)
      for (int32_t r = ra + 1; r <= ra + g; ++r) zero(r);
    if (!__any_sync(0xffffffffu, lng)) continue;
    if (!lng) g = 0;
    int incl = g;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    for (int tb = 0; tb < total; tb += 32) {
      const int t = tb + lane;
      int lo = 0;  // first gap i with incl[i] > t
#pragma unroll
      for (int st = 16; st > 0; st >>= 1) {
        const int v = __shfl_sync(0xffffffffu, incl, lo + st - 1);
        if (v <= t) lo += st;
      }
      const int ex = __shfl_sync(0xffffffffu, incl - g, lo);
      const int32_t r = __shfl_sync(0xffffffffu, ra, lo) + 1 + (t - ex);
      if (t < total) zero(r);
    }
  }
}

struct NzMeta {
  uint32_t mw;  // emask word lane/4 of the tile
  uint32_t pw;  // row ends in the words before it (epre byte lane/4)
  int32_t q0;   // tile_q[k]: first row (compacted) ending in or after the tile
};

// the lane's 8 consecutive nonzeros of tile k (colind, values) + metadata
template <typename RP, bool MASK>
__device__ __forceinline__ void nz_tile_load(const NzP<RP>& p, int64_t k, int lane, int (&c)[8], double (&v)[8],
                                             NzMeta& m) {
  const int64_t t0 = k * kNzTile;
  const int cnt = (int)((p.nnz - t0) < kNzTile ? (p.nnz - t0) : kNzTile);
  const int e0 = lane * 8;
  if (e0 + 8 <= cnt) {
    ld256_s32(p.col + t0 + e0, c);
    ld256_f64(p.val + t0 + e0, v);
    ld256_f64(p.val + t0 + e0 + 4, v + 4);
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const bool ok = e0 + i < cnt;
      c[i] = ok ? ld_stream(p.col + t0 + e0 + i) : 0;
      v[i] = ok ? ld_stream(p.val + t0 + e0 + i) : 0.0;
    }
  }
  if constexpr (MASK) {
    m.mw = (uint32_t)ld_stream(reinterpret_cast<const int*>(p.emask) + k * 8 + (lane >> 2));
    const uint32_t* pre = reinterpret_cast<const uint32_t*>(p.epre + k);
    m.pw = (uint32_t)ld_stream(reinterpret_cast<const int*>(pre) + (lane >> 4));
    m.q0 = ld_ro(p.tile_q + k);
  }
}

template <typename RP, bool HOT, bool MASK, bool L2G>
__device__ __forceinline__ void nz_tile_compute(const NzP<RP>& p, int64_t k, int lane, const double* xh,
                                                uint32_t* em, const int (&c)[8], const double (&v)[8],
                                                const NzMeta& m);

template <typename RP, bool HOT, bool MASK, bool L2G>
__device__ __forceinline__ void nz_tile(const NzP<RP>& p, int64_t k, int lane, const double* xh, uint32_t* em) {
  int c[8];
  double v[8];
  NzMeta m;
  nz_tile_load<RP, MASK>(p, k, lane, c, v, m);
  nz_tile_compute<RP, HOT, MASK, L2G>(p, k, lane, xh, em, c, v, m);
}

// MASK: row ends from the plan's per-tile mask (emask/epre, loaded with the
// streams); else from tile_q[k..k+1] and the compacted rowptr (em: the warp's
// 8-word smem scratch mask); L2G: x gathers bypass L1 (ld_xg)
template <typename RP, bool HOT, bool MASK, bool L2G>
__device__ __forceinline__ void nz_tile_compute(const NzP<RP>& p, int64_t k, int lane, const double* xh,
                                                uint32_t* em, const int (&c)[8], const double (&v)[8],
                                                const NzMeta& m) {
  const int64_t t0 = k * kNzTile;
  const int cnt = (int)((p.nnz - t0) < kNzTile ? (p.nnz - t0) : kNzTile);
  double xv[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    if constexpr (HOT) xv[i] = c[i] < 0 ? xh[~c[i]] : ld_xg<L2G>(p.x + c[i]);
    else xv[i] = ld_xg<L2G>(p.x + c[i]);
  }

  uint32_t my;
  int before;
  int64_t q0;
  if constexpr (MASK) {
    // the lane's 8 row-end bits; rows ending before them: the word prefix
    // byte + the lower bits of the word; rows ending in the tile: q in
    // [q0, q1) (lane 31 holds the count; the gap loop broadcasts it)
    const int sh = (lane & 3) * 8;
    my = (m.mw >> sh) & 0xffu;
    before = (int)((m.pw >> (((lane >> 2) & 3) * 8)) & 0xffu) + __popc(m.mw & ((1u << sh) - 1u));
    q0 = m.q0;
    if (p.zero_gaps) nz_zero_gaps_warp(p, q0, __shfl_sync(0xffffffffu, before + __popc(my), 31), lane);
  } else {
    // rows ending in the tile: q in [q0, q1), end position rpc[q+1]-1
    q0 = ld_ro(p.tile_q + k);
    const int64_t q1 = ld_ro(p.tile_q + k + 1);
    const int n_end = (int)(q1 - q0);
    if (lane < 8) em[lane] = 0u;
    __syncwarp();
    // rows ending in the tile; the empty rows after each are zeroed by its own
    // lane (gaps are at most kNzGapMax rows: longer runs make the plan clear y
    // first). B200, C3: 264 us vs 269 us with the warp-cooperative zeroing of
    // the MASK path below, 275 us with a per-lane/warp hybrid in this loop.
    for (int j = lane; j < n_end; j += 32) {
      const int64_t q = q0 + j;
      const int e = (int)((int64_t)ld_ro(p.rpc + q + 1) - 1 - t0);
      atomicOr(&em[e >> 5], 1u << (e & 31));
      if (p.zero_gaps) {
        const int32_t ra = ld_ro(p.rowmap + q), rb = ld_ro(p.rowmap + q + 1);
        for (int32_t r = ra + 1; r < rb; ++r) nz_zero_row(p, r);
      }
    }
    __syncwarp();
    const uint4 m0 = *reinterpret_cast<const uint4*>(em);
    const uint4 m1 = *reinterpret_cast<const uint4*>(em + 4);
    const uint32_t words[8] = {m0.x, m0.y, m0.z, m0.w, m1.x, m1.y, m1.z, m1.w};
    const int wi = lane >> 2, sh = (lane & 3) * 8;
    uint32_t word = 0;
    before = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (i < wi) before += __popc(words[i]);
      if (i == wi) word = words[i];
    }
    before += __popc(word & ((1u << sh) - 1u));
    my = (word >> sh) & 0xffu;
  }
  if (k == 0 && p.zero_gaps) {
    const int32_t r0 = ld_ro(p.rowmap);
    for (int32_t r = lane; r < r0; r += 32)
      if (!p.orp || ld_ro(p.orp + r + 1) == ld_ro(p.orp + r)) p.y[r] = 0.0;
  }

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
      p.carry_row[k] = ld_ro(p.rowmap + qf + ne);  // q1: lane 31 ends the count
      p.carry_val[k] = S;
    } else {
      p.carry_row[k] = -1;
    }
  }
}

// ---- column-tiled long rows (see long_tiled.cu) -----------------------------
struct LongP {
  const int32_t* col;
  const uint16_t* col16;  // non-null: the long rows' in-block columns (colind & (kLongXB - 1))
  const double* val;
  const double* x;
  const int64_t* seg;   // [n_long][nblk+1]
  double* partial;      // [n_long][nblk]
  int64_t n_long, n_cols, nblk;
  int rg;               // row groups per x block
};

// work item it = (x block b, row group g) = (it / rg, it % rg) for the whole
// CTA of NT threads: x block b staged in xs (kLongXB doubles), then each warp
// streams the segments of long rows q = g + rg*(w + NW*i), lane l taking
// nonzeros l, l+32, ... (coalesced loads, 16 in flight per lane). Lane-strided
// order matters for the smem gather: the 32 lanes of one load read 32
// consecutive nonzeros of a sorted row, i.e. nearby columns (~2-way bank
// conflicts), where lane-contiguous chunks scatter over the whole block
// (measured ~8 wavefronts per gather on C4).
// The segment bounds of the warp's first 32 rows (lane j: row j) are loaded
// with the x block, so a row starts with its stream loads; the caller
// separates items with a barrier (xs is rewritten by the next item).
#ifndef LONG_U
#define LONG_U 16
#endif
constexpr int kLongU = LONG_U;  // nonzeros per lane per batch of the long-row stream
template <int NT, bool C16>
__device__ __forceinline__ void long_item(const LongP& p, int64_t it, double* xs) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  constexpr int NW = NT / 32;
  constexpr int XPT = (int)(kLongXB / NT);
  const int64_t b = it / p.rg, g = it % p.rg;
  const int64_t c0 = b * kLongXB;
  const int cw = (int)((p.n_cols - c0) < kLongXB ? (p.n_cols - c0) : kLongXB);
  const int64_t qs = (int64_t)p.rg * NW, q0 = g + (int64_t)p.rg * w, ld = p.nblk + 1;
  const int nq = q0 < p.n_long ? (int)((p.n_long - 1 - q0) / qs) + 1 : 0;
  long long sa = 0, sb = 0;
  if (lane < nq) {
    const int64_t q = q0 + qs * lane;
    sa = ld_ro(p.seg + q * ld + b);
    sb = ld_ro(p.seg + q * ld + b + 1);
  }
#pragma unroll
  for (int u = 0; u < XPT; ++u) {
    const int i = (int)threadIdx.x + NT * u;
    if (i < cw) xs[i] = ld_x(p.x + c0 + i);
  }
  int64_t s0 = 0, s1 = 0;
  auto bounds = [&](int j) {
    if (j < 32) {
      s0 = __shfl_sync(0xffffffffu, sa, j);
      s1 = __shfl_sync(0xffffffffu, sb, j);
    } else {
      const int64_t q = q0 + qs * j;
      s0 = ld_ro(p.seg + q * ld + b);
      s1 = ld_ro(p.seg + q * ld + b + 1);
    }
  };
  constexpr int U = kLongU;
  __syncthreads();
  for (int j = 0; j < nq; ++j) {
    bounds(j);
    double a0 = 0.0, a1 = 0.0;
    for (int64_t bb = s0; bb < s1; bb += 32 * U) {
      // one base pointer per stream + immediate offsets; slot u valid iff 32u < rem
      const int32_t* cp = p.col + bb + lane;
      const uint16_t* cp16 = p.col16 + bb + lane;
      const double* vp = p.val + bb + lane;
      const int64_t r64 = s1 - bb - lane;
      const int rem = r64 > 32 * U ? 32 * U : (int)r64;
      int c[U];
      double v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const bool ok = 32 * u < rem;
        if constexpr (C16) c[u] = ok ? ld_stream_u16(cp16 + 32 * u) : 0;
        else c[u] = ok ? ld_stream(cp + 32 * u) - (int)c0 : 0;
        v[u] = ok ? ld_stream(vp + 32 * u) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < U; u += 2) {
        a0 = fma(v[u], xs[c[u]], a0);
        a1 = fma(v[u + 1], xs[c[u + 1]], a1);
      }
    }
    const double t = warp_sum(a0 + a1);
    if (lane == 0) p.partial[(q0 + qs * j) * p.nblk + b] = t;
  }
}

// sum_b partial[b] over b < nblk for one warp (lane-strided): 8 independent
// accumulators so 8 loads are in flight per lane (a single running sum waits
// one L2 round trip per 32 partials: ~4 us for C4's 489 blocks), combined in a
// fixed order, then the fixed butterfly -- deterministic
__device__ __forceinline__ double long_row_total(const double* __restrict__ partial, int64_t nblk, int lane) {
  double a[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  int64_t b = lane;
  for (; b + 7 * 32 < nblk; b += 8 * 32) {
#pragma unroll
    for (int u = 0; u < 8; ++u) a[u] += __ldcg(partial + b + 32 * u);  // (previous kernel: L2-coherent)
  }
#pragma unroll
  for (int u = 0; u < 8; ++u)
    if (b + 32 * u < nblk) a[u] += __ldcg(partial + b + 32 * u);
  const double t = ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
  return warp_sum(t);
}

}  // namespace spmv
