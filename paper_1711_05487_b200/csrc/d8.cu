// d8.cu -- cta_stream over dictionary-coded 8-bit column deltas ("D8"): the
// MB-class optimisation of Sec. III-E ("8- or 16-bit deltas
// wherever possible, but never both"; Table II) re-designed for sm_100a.
//
// Format (reading 26):
//   delta_j = colind[j] - i              for the head j of row i (row id of
//                                        the matrix: row0 + local row)
//   delta_j = colind[j] - colind[j-1]    otherwise
//   dict    = the <= 256 distinct deltas (ascending), codes[j] = index of delta_j
//   rlen[i] = row length (<= 255)
// so the kernel reads 1 byte of index per nonzero and 1 byte per row instead
// of 4 B colind + 4/8 B rowptr: C5 (27-pt 384^3) 19.61 -> 14.66 GB per SpMV.
// The decode is a running sum per lane: c = row id; c += dict[code].
//
// Row-count tiles only (regular rows): tile k = rows [k*Rt, min((k+1)*Rt, m)),
// nonzeros [tile_nz[k], tile_nz[k+1]); no row crosses a tile, no carries.
// Persistent warp-specialised CTAs as in stream.cu: one producer lane issues
// three TMA bulk copies per tile (values, codes, row lengths; L2 evict_first)
// into the stage of the consumer warp that owns the tile; the consumer's
// lanes walk consecutive rows in step (one lane per row), 8 predicated x
// gathers in flight per lane, dictionary in shared memory.
#include <cstdlib>
#include <algorithm>
#include <type_traits>

#include "common.cuh"
#include "internal.h"
#include "iterfuse.cuh"

namespace spmv {

__host__ __device__ __forceinline__ size_t d8_al128(size_t v) { return (v + 127) & ~(size_t)127; }

struct D8Layout {
  size_t vals, codes, rl, stage, full, empty, meta, pat, total;
};

// C: nonzero capacity of a tile (Rt x longest row), Rt rows per tile, CB:
// bits per code (8, or 4 when the dictionary has <= 16 entries; 0: row-pattern
// mode -- no code stream, the per-row byte is the row's pattern, whose npofs
// column offsets live in shared memory after the barriers)
__host__ __device__ inline D8Layout d8_layout(int64_t C, int64_t Rt, int stages, int CB = 8, int64_t npofs = 0) {
  D8Layout L;
  L.vals = 0;
  // values: copy starts at the 128-B line of the first value (<= 15 before
  // t0) and is rounded up to 16 B (<= 1 after)
  L.codes = d8_al128((size_t)(C + 16) * 8);
  // codes: copy starts 16-B aligned (<= 15 before t0), rounded up to 16 B,
  // plus >= 16 readable bytes past any row end (branch-free 16-code batches)
  L.rl = L.codes + (CB == 0 ? 0 : d8_al128((size_t)(CB == 4 ? (C + 1) / 2 : C) + 64));
  L.stage = d8_al128(L.rl + (size_t)Rt + 16);
  size_t o = L.stage * stages;
  L.full = o; o += 8 * (size_t)stages;
  L.empty = o; o += 8 * (size_t)stages;
  L.meta = d8_al128(o); o = L.meta + 32 * (size_t)stages;
  // pattern offsets (+ 16 readable entries past the last: a batch past a
  // row end reads stale offsets, masked like stale codes)
  L.pat = d8_al128(o); o = L.pat + (CB == 0 ? (size_t)(npofs + 16) * 4 : 0);
  L.total = d8_al128(o);
  return L;
}

size_t d8_smem_bytes(int64_t C, int64_t Rt, int stages, int CB, int64_t npofs) {
  return d8_layout(C, Rt, stages, CB, npofs).total;
}

struct D8Meta {
  int64_t t0;
  int32_t cnt, voff;  // nonzeros; offset of t0 in the staged values
  int32_t coff, pad;  // offset of t0 in the staged codes, in codes (8-bit: t0 & 15; 4-bit: nibbles)
};

struct D8P {
  const double* val;
  const uint8_t* codes;
  const uint8_t* rlen;
  const unsigned char* tiles;  // packed tiles (PK): segment k = bytes [toff[k], toff[k+1])
  const int64_t* toff;
  const int64_t* tile_nz;
  const double* x;
  double* y;
  IterOut it;       // iterated mode: pending rescale, fused norm partials / step (iterfuse.cuh)
  int64_t m, T, k0; // rows, end of the tile range, first tile
  int64_t Rt, C;    // rows per tile, nonzero capacity
  int64_t row0;     // row id of local row 0 (the anchor of the head deltas)
  int64_t n_cols;   // (checked build only)
  int stages;
  const int32_t* pofs;  // row-pattern mode: the patterns' column offsets [n_pofs]
  int n_pofs;
  int32_t dict[256];    // dictionary; row-pattern mode: pattern p = offsets [d & 0xffff, + (d >> 16)) of pofs
};

__device__ __forceinline__ void d8_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Consumer warps' tile loop; returns the warp's sum of squares of the rows it
// wrote (its tiles in launch order; 0 outside the iterated mode).
template <int CW, bool SCALE, int UN, int CB, bool PK, bool PU>
__device__ __forceinline__ double d8_consume(const D8P& p, unsigned char* smem, const D8Layout& L, uint64_t* full,
                                             uint64_t* empty, const D8Meta* meta, const int32_t* dict_s, double f) {
  const int32_t* pat_s = reinterpret_cast<const int32_t*>(smem + L.pat);  // (row-pattern mode)
  const int S = p.stages;
  const int w = (threadIdx.x >> 5) - 1;
  const int lane = threadIdx.x & 31;
  double sqa = 0.0;  // this lane's squares over all its rows (its tiles in order): one warp sum at the end
  for (int i = w;; i += CW) {
    const int64_t kl = p.k0 + blockIdx.x + (int64_t)i * gridDim.x;
    if (kl >= p.T) break;
    const int64_t k = p.it.rev ? p.T - 1 + p.k0 - kl : kl;  // reversed launch: tiles from the end
    const int s = i % S;
    mbar_wait(&full[s], (uint32_t)((i / S) & 1));
    const D8Meta mt = meta[s];
    SPMV_CHECK(mt.cnt >= 0 && mt.cnt <= p.C && mt.voff >= 0 && mt.voff < 16 && mt.coff >= 0 && mt.coff < 32);
    const unsigned char* st = smem + L.stage * s;
    const double* vals_s;
    const uint8_t* codes_s;  // code e of the tile: unit mt.coff + e
    const uint8_t* rl_s;
    if constexpr (PK) {  // packed segment: values, codes, row lengths (16-B aligned parts)
      const int c16 = (mt.cnt + 1) & ~1;  // values padded to 16 B
      vals_s = reinterpret_cast<const double*>(st);
      codes_s = st + (size_t)c16 * 8;
      rl_s = codes_s + ((mt.cnt + 15) & ~15);
    } else {
      vals_s = reinterpret_cast<const double*>(st + L.vals) + mt.voff;
      codes_s = st + L.codes;
      rl_s = st + L.rl;
    }
    const int64_t R0 = k * p.Rt;
    const int nrows = (int)(((R0 + p.Rt) < p.m ? (R0 + p.Rt) : p.m) - R0);
    int base = 0;  // first nonzero (tile-relative) of the pass
    for (int qb = 0; qb < nrows; qb += 32) {
      const int q = qb + lane;
      // row-pattern mode: the staged byte is the row's pattern, its
      // descriptor gives the length and where its offsets start
      const int dsc = CB == 0 ? dict_s[q < nrows ? (int)rl_s[q] : 0] : 0;
      const int len = q < nrows ? (CB == 0 ? (dsc >> 16) & 0xff : (int)rl_s[q]) : 0;
      int inc = len;  // inclusive scan of the row lengths over the pass
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += v;
      }
      const int off = base + inc - len;
      base += __shfl_sync(0xffffffffu, inc, 31);
      SPMV_CHECK(off + len <= mt.cnt && len <= 255);
      int c = (int)(p.row0 + R0 + q);  // anchor of the head delta
      double a0 = 0.0, a1 = 0.0;
      for (int l0 = 0; l0 < len; l0 += UN) {
        // UN codes read unconditionally (the stage keeps >= 16 bytes of slack
        // past the tile; a stale code still indexes the 256-entry dictionary)
        // and masked by selects: no branch around the shared-memory loads;
        // UN independent x gathers in flight per lane
        int cc[UN];
        double xv[UN];
        if constexpr (CB == 0) {
          // row-pattern mode: column = row id + the pattern's offset -- no
          // running sum, every offset an independent smem read (lanes of
          // one pattern read the same word: a broadcast)
          const int32_t* po = pat_s + (dsc & 0xffff) + l0;
#pragma unroll
          for (int u = 0; u < UN; ++u) cc[u] = c + po[u];
        } else {
#pragma unroll
          for (int u = 0; u < UN; ++u) {
            const int e = mt.coff + off + l0 + u;
            const int code = CB == 8 ? (int)codes_s[e] : ((int)codes_s[e >> 1] >> ((e & 1) << 2)) & 15;
            const int d = dict_s[code];
            c += (l0 + u < len) ? d : 0;
            cc[u] = c;
          }
        }
#pragma unroll
        for (int u = 0; u < UN; ++u) SPMV_CHECK(l0 + u >= len || (cc[u] >= 0 && cc[u] < p.n_cols));
#pragma unroll
#ifdef D8_EXP_XHIT  // timing experiment only: every gather an L1 hit (wrong results)
        for (int u = 0; u < UN; ++u) xv[u] = l0 + u < len ? ld_x(p.x + (cc[u] & 2047)) : 0.0;
#else
        for (int u = 0; u < UN; ++u) xv[u] = l0 + u < len ? ld_x(p.x + cc[u]) : 0.0;
#endif
        if constexpr (UN % 2 == 0) {
#pragma unroll
          for (int u = 0; u < UN; u += 2) {
            const int l = l0 + u;
            a0 = fma(l < len ? vals_s[off + l] : 0.0, xv[u], a0);
            a1 = fma(l + 1 < len ? vals_s[off + l + 1] : 0.0, xv[u + 1], a1);
          }
        } else {  // odd batch (row patterns whose length it divides, e.g. 27 = 3 x 9)
#pragma unroll
          for (int u = 0; u < UN; ++u) {
            const double v = l0 + u < len ? vals_s[off + l0 + u] : 0.0;
            if (u & 1) a1 = fma(v, xv[u], a1);
            else a0 = fma(v, xv[u], a0);
          }
        }
      }
      double acc = a0 + a1;
      if constexpr (SCALE) acc *= f;
      if (q < nrows) {
        SPMV_CHECK(R0 + q < p.m);
        if constexpr (PU) {  // + the neighbours' replicas
          SPMV_CHECK(!p.it.push_lo || p.it.push_lo_end <= p.m);
          SPMV_CHECK(!p.it.push_hi || (p.it.push_hi_begin >= 0 && p.it.push_hi_begin <= p.m));
          iter_store(p.it, p.y, R0 + q, acc);
        }
        else p.y[R0 + q] = acc;
        sqa = fma(acc, acc, sqa);
      }
    }
    __syncwarp();
    if (lane == 0) d8_arrive(&empty[s]);
  }
  // (a per-tile warp sum before releasing the stage delayed every refill by
  // its shuffle chain: +4 % per SpMV on C5)
  return p.it.cta_part ? warp_sum(sqa) : 0.0;  // fixed butterfly: deterministic
}

// resident CTAs per SM the registers allow (launch bound): UN = 8 -> ~72
// registers, UN = 16 -> ~96
constexpr int d8_lb(int CW, int UN) { return UN <= 9 ? (CW == 4 ? 5 : (CW == 6 ? 4 : 3)) : (CW == 4 ? 4 : (CW == 6 ? 3 : 2)); }

// PU: the multi-shard halo push instantiation (IterOut::push_*; 8-bit codes or
// row patterns, unpacked tiles only -- d8_push_capable)
template <int CW, int UN, int CB, bool PK, bool PU = false>
__global__ void __launch_bounds__(32 * (CW + 1), d8_lb(CW, UN)) d8_kernel(const D8P p) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ int32_t dict_s[256];
  __shared__ double f_s;                   // iterated mode: this launch's exact factor
  __shared__ __align__(8) uint64_t fbar_s;  // ... and its hand-over barrier
  uint64_t* fbar = &fbar_s;
  const D8Layout L = d8_layout(p.C, p.Rt, p.stages, CB, p.n_pofs);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.full);
  uint64_t* empty = reinterpret_cast<uint64_t*>(smem + L.empty);
  D8Meta* meta = reinterpret_cast<D8Meta*>(smem + L.meta);
  const int S = p.stages;

  pdl_trigger();
  for (int i = threadIdx.x; i < 256; i += blockDim.x) dict_s[i] = p.dict[i];
  if constexpr (CB == 0) {
    int32_t* pat_s = reinterpret_cast<int32_t*>(smem + L.pat);
    for (int i = threadIdx.x; i < p.n_pofs + 16; i += blockDim.x) pat_s[i] = i < p.n_pofs ? p.pofs[i] : 0;
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(fbar, 1);
    fence_mbar_init();
  }
  __syncthreads();

  if (threadIdx.x < 32) {
    // ------------------------------ producer ------------------------------
    if (threadIdx.x == 0) {
      const uint64_t pol = policy_evict_first();
      int64_t nT0 = 0, nT1 = 0;
      auto fetch = [&](int64_t kk) {
        if (kk < p.T) {
          nT0 = ld_ro(p.tile_nz + kk);
          nT1 = ld_ro(p.tile_nz + kk + 1);
        }
      };
      // reversed launches (iterated mode, every other iteration) walk the
      // tiles from the end, where the previous launch last wrote its y (the
      // x read now): those lines are still in L2
      const int64_t rb = p.it.rev ? p.T - 1 + p.k0 : 0;
      auto phys = [&](int64_t kl) { return p.it.rev ? rb - kl : kl; };
      fetch(phys(p.k0 + blockIdx.x));
      int i = 0;
      for (int64_t kl = p.k0 + blockIdx.x; kl < p.T; kl += gridDim.x, ++i) {
        const int64_t k = phys(kl);
        const int s = i % S;
        const int64_t t0 = nT0, t1 = nT1;
        if (kl + gridDim.x < p.T) fetch(phys(kl + gridDim.x));
        if (i >= S) mbar_wait(&empty[s], (uint32_t)(((i / S) - 1) & 1));
        const int64_t R0 = k * p.Rt;
        const int64_t R1 = (R0 + p.Rt) < p.m ? (R0 + p.Rt) : p.m;
        // codes: 16-B aligned byte range holding codes [t0, t1) (4-bit codes:
        // two per byte, low nibble first)
        const int64_t v0 = t0 & ~15ll;
        const int64_t cb0 = (CB == 8 ? t0 : (t0 >> 1)) & ~15ll;
        const int64_t cb1 = CB == 8 ? t1 : (t1 + 1) >> 1;
        const uint32_t vb = t1 > t0 ? (uint32_t)(((t1 - v0) * 8 + 15) & ~15ll) : 0u;
        const uint32_t cb = (CB != 0 && t1 > t0) ? (uint32_t)(((cb1 - cb0) + 15) & ~15ll) : 0u;
        const uint32_t rb = (uint32_t)(((R1 - R0) + 15) & ~15ll);
        D8Meta mt;
        mt.t0 = t0;
        mt.cnt = (int32_t)(t1 - t0);
        mt.voff = PK ? 0 : (int32_t)(t0 - v0);
        mt.coff = PK ? 0 : (int32_t)(CB == 8 ? t0 - cb0 : t0 - 2 * cb0);
        mt.pad = 0;
        meta[s] = mt;
        unsigned char* st = smem + L.stage * s;
        if constexpr (PK) {
          // packed tiles: [values | codes | row lengths] of tile k contiguous
          // in one 16-B-aligned segment: ONE bulk copy per tile
          const int64_t o0 = ld_ro(p.toff + k), o1 = ld_ro(p.toff + k + 1);
          mbar_arrive_expect_tx(&full[s], (uint32_t)(o1 - o0));
          bulk_g2s(st, p.tiles + o0, (uint32_t)(o1 - o0), &full[s], pol);
        } else {
          mbar_arrive_expect_tx(&full[s], vb + cb + rb);
          if (t1 > t0) {
            bulk_g2s(st + L.vals, p.val + v0, vb, &full[s], pol);
            if constexpr (CB != 0) bulk_g2s(st + L.codes, p.codes + cb0, cb, &full[s], pol);
          }
          bulk_g2s(st + L.rl, p.rlen + R0, rb, &full[s], pol);
        }
      }
    } else if (p.it.cta_only && p.it.prev_part && blockIdx.x == gridDim.x - 1) {
      iter_lag_fold_lanes(p.it);  // lagged iteration: the previous launch's norm (lanes 1..31)
    }
    return;
  }

  // ------------------------------- consumers --------------------------------
  pdl_wait();  // x, y, the scale may be written by the previous kernel in the stream
  // iterated mode: the exact factor this launch applies (1 almost always),
  // fetched by ONE thread and handed over through an mbarrier; each warp
  // first waits for its first stage (the TMA fill hides the load), then
  // picks one of two instantiations of the tile loop, so the common path
  // carries no multiply or live factor (a live factor in the loop, or a
  // rescale pass after it, cost 7 % on C5 through code generation; a CTA
  // barrier on the load at the launch start cost ~3 % per C2 iteration)
  double f = 1.0;
  if (p.it.cta_part) {
    if (threadIdx.x == 32) {
      f_s = iter_factor(p.it);
      d8_arrive(fbar);
    }
    const int w = (threadIdx.x >> 5) - 1;
    if (p.k0 + blockIdx.x + (int64_t)w * gridDim.x < p.T) mbar_wait(&full[w % S], 0u);
    mbar_wait(fbar, 0u);
    f = f_s;
  }
  double wsq;
  if constexpr (PU) wsq = d8_consume<CW, true, UN, CB, PK, true>(p, smem, L, full, empty, meta, dict_s, f);
  else
    wsq = f == 1.0 ? d8_consume<CW, false, UN, CB, PK, false>(p, smem, L, full, empty, meta, dict_s, 1.0)
                   : d8_consume<CW, true, UN, CB, PK, false>(p, smem, L, full, empty, meta, dict_s, f);
  if constexpr (PU) __threadfence_system();  // the peer stores, before the partials / kernel end
  iter_epilogue<32 * CW>(p.it, wsq);
}

static D8P d8_params(const StreamPlan& sp, const double* x, double* y) {
  D8P p;
  p.val = sp.V.val;
  p.codes = sp.codes;
  p.rlen = sp.rlen;
  p.tiles = sp.d8_tiles;
  p.toff = sp.d8_toff;
  p.tile_nz = sp.tile_nz;
  p.x = x;
  p.y = y;
  p.it = sp.it;
  p.m = sp.V.m;
  p.T = sp.T;
  p.k0 = sp.k0;
  p.Rt = sp.rows_per_tile;
  p.C = sp.C;
  p.row0 = sp.row0;
  p.n_cols = sp.V.n_cols;
  p.stages = sp.stages;
  p.pofs = sp.pat_ofs;
  p.n_pofs = sp.n_pat_ofs;
  for (int i = 0; i < 256; ++i) p.dict[i] = i < sp.n_dict ? sp.dict[i] : 0;
  return p;
}

template <int CW, int UN, int CB, bool PK>
static int d8_prepare_t(const StreamPlan& sp, int sm_count) {
  const size_t smem = d8_smem_bytes(sp.C, sp.rows_per_tile, sp.stages, CB, sp.n_pat_ofs);
  if (cudaFuncSetAttribute(d8_kernel<CW, UN, CB, PK>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
      cudaSuccess)
    return -1;
  if constexpr ((CB == 8 || CB == 0) && !PK) {
    if (cudaFuncSetAttribute(d8_kernel<CW, UN, CB, PK, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem) != cudaSuccess)
      return -1;
  }
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, d8_kernel<CW, UN, CB, PK>, 32 * (CW + 1), smem) !=
          cudaSuccess ||
      per_sm < 1)
    return -1;
  if (const char* e = getenv("SPMV_STREAM_CTAS")) per_sm = std::max(1, std::min(per_sm, atoi(e)));  // experiments
  int64_t grid = (int64_t)sm_count * per_sm;
  if (grid > sp.T) grid = sp.T;
  return (int)std::max<int64_t>(grid, 1);
}

template <int CW, int UN, int CB, bool PK>
static int d8_per_sm_t(const StreamPlan& sp) {
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, d8_kernel<CW, UN, CB, PK>, 32 * (CW + 1),
                                                    d8_smem_bytes(sp.C, sp.rows_per_tile, sp.stages, CB, sp.n_pat_ofs)) !=
      cudaSuccess)
    return 0;
  return per_sm;
}

template <int CW, int UN, int CB, bool PK>
static void d8_launch_t(const StreamPlan& sp, const double* x, double* y, cudaStream_t s) {
  if constexpr ((CB == 8 || CB == 0) && !PK) {
    if (sp.it.push_lo || sp.it.push_hi) {
      launch_pdl(d8_kernel<CW, UN, CB, PK, true>, dim3(sp.grid), dim3(32 * (CW + 1)),
                 d8_smem_bytes(sp.C, sp.rows_per_tile, sp.stages, CB, sp.n_pat_ofs), s, d8_params(sp, x, y));
      return;
    }
  }
  launch_pdl(d8_kernel<CW, UN, CB, PK>, dim3(sp.grid), dim3(32 * (CW + 1)),
             d8_smem_bytes(sp.C, sp.rows_per_tile, sp.stages, CB, sp.n_pat_ofs), s, d8_params(sp, x, y));
}

bool d8_push_capable(const StreamPlan& sp) { return (sp.d8_bits == 8 || sp.d8_bits == 0) && !sp.d8_tiles; }

// (stages = consumer warps CW) x (batch width UN) x (code layout) -> instantiation
template <int UN, int CB, bool PK, typename F>
static int d8_cw(const StreamPlan& sp, F&& f) {
  using U = std::integral_constant<int, UN>;
  using B = std::integral_constant<int, CB>;
  using K = std::integral_constant<bool, PK>;
  switch (sp.stages) {
    case 4: return f(std::integral_constant<int, 4>{}, U{}, B{}, K{});
    case 6: return f(std::integral_constant<int, 6>{}, U{}, B{}, K{});
    case 8: return f(std::integral_constant<int, 8>{}, U{}, B{}, K{});
    default: return -1;
  }
}
template <typename F>
static int d8_dispatch(const StreamPlan& sp, F&& f) {
  if (sp.d8_bits == 0)  // row patterns
    return sp.d8_un == 16  ? d8_cw<16, 0, false>(sp, f)
           : sp.d8_un == 9 ? d8_cw<9, 0, false>(sp, f)
           : sp.d8_un == 7 ? d8_cw<7, 0, false>(sp, f)
                           : d8_cw<8, 0, false>(sp, f);
  if (sp.d8_bits == 4) return sp.d8_un == 16 ? d8_cw<16, 4, false>(sp, f) : d8_cw<8, 4, false>(sp, f);
  if (sp.d8_tiles) return d8_cw<8, 8, true>(sp, f);
  return sp.d8_un == 16 ? d8_cw<16, 8, false>(sp, f) : d8_cw<8, 8, false>(sp, f);
}

int d8_per_sm(const StreamPlan& sp) {
  const int r = d8_dispatch(
      sp, [&](auto cw, auto un, auto cb, auto pk) { return d8_per_sm_t<cw.value, un.value, cb.value, pk.value>(sp); });
  return r < 0 ? 0 : r;
}

int d8_prepare(const StreamPlan& sp, int sm_count) {
  return d8_dispatch(sp, [&](auto cw, auto un, auto cb, auto pk) {
    return d8_prepare_t<cw.value, un.value, cb.value, pk.value>(sp, sm_count);
  });
}

void launch_d8(const StreamPlan& sp, const double* x, double* y, cudaStream_t s) {
  d8_dispatch(sp, [&](auto cw, auto un, auto cb, auto pk) {
    d8_launch_t<cw.value, un.value, cb.value, pk.value>(sp, x, y, s);
    return 0;
  });
}

// packed tiles (plan time): segment k = [values (8 cnt, padded to 16 B) |
// codes (cnt, padded to 16) | row lengths (nrows, padded to 16)] at toff[k];
// one warp per tile copies the three parts
__global__ void __launch_bounds__(kNT) d8_pack_tiles_kernel(const double* __restrict__ val,
                                                            const uint8_t* __restrict__ codes,
                                                            const uint8_t* __restrict__ rlen,
                                                            const int64_t* __restrict__ tile_nz,
                                                            const int64_t* __restrict__ toff, int64_t T, int64_t Rt,
                                                            int64_t m, unsigned char* __restrict__ tiles) {
  const int64_t k = ((int64_t)blockIdx.x * kNT + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (k >= T) return;
  const int64_t t0 = tile_nz[k], cnt = tile_nz[k + 1] - t0;
  const int64_t R0 = k * Rt, nr = ((R0 + Rt) < m ? (R0 + Rt) : m) - R0;
  unsigned char* seg = tiles + toff[k];
  double* v = reinterpret_cast<double*>(seg);
  const int64_t c16 = (cnt + 1) & ~1ll;
  for (int64_t j = lane; j < c16; j += 32) v[j] = j < cnt ? val[t0 + j] : 0.0;
  uint8_t* c = seg + c16 * 8;
  const int64_t cp = (cnt + 15) & ~15ll;
  for (int64_t j = lane; j < cp; j += 32) c[j] = j < cnt ? codes[t0 + j] : 0;
  uint8_t* r = c + cp;
  const int64_t rp = (nr + 15) & ~15ll;
  for (int64_t j = lane; j < rp; j += 32) r[j] = j < nr ? rlen[R0 + j] : 0;
}

void launch_d8_pack_tiles(const StreamPlan& sp, const int64_t* toff, unsigned char* tiles, cudaStream_t s) {
  if (sp.T <= 0) return;
  const int64_t g = (sp.T * 32 + kNT - 1) / kNT;
  d8_pack_tiles_kernel<<<(unsigned)g, kNT, 0, s>>>(sp.V.val, sp.codes, sp.rlen, sp.tile_nz, toff, sp.T,
                                                   sp.rows_per_tile, sp.V.m, tiles);
}

// 4-bit codes: packed[i] = codes[2i] | codes[2i+1] << 4 (low nibble first)
__global__ void __launch_bounds__(kNT) d8_pack4_kernel(const uint8_t* __restrict__ codes, int64_t nnz,
                                                       uint8_t* __restrict__ packed) {
  const int64_t nb = (nnz + 1) / 2;
  for (int64_t i = (int64_t)blockIdx.x * kNT + threadIdx.x; i < nb; i += (int64_t)gridDim.x * kNT) {
    const uint8_t lo = codes[2 * i], hi = 2 * i + 1 < nnz ? codes[2 * i + 1] : 0;
    packed[i] = (uint8_t)(lo | (hi << 4));
  }
}

void launch_d8_pack4(const uint8_t* codes, int64_t nnz, uint8_t* packed, cudaStream_t s) {
  if (nnz <= 0) return;
  int64_t g = ((nnz + 1) / 2 + kNT - 1) / kNT;
  if (g > dev_sm_count() * 32) g = dev_sm_count() * 32;
  d8_pack4_kernel<<<(unsigned)g, kNT, 0, s>>>(codes, nnz, packed);
}

// ---- plan time ----------------------------------------------------------------
// Encode: one thread per row (rows <= 255 nonzeros): code = index of the
// row-relative delta in the sorted dictionary (binary search in smem).
template <typename RP>
__global__ void __launch_bounds__(kNT) d8_encode_kernel(const RP* __restrict__ rp, const int32_t* __restrict__ col,
                                                        int64_t m, int64_t row0, const int32_t* __restrict__ dict,
                                                        int nd, uint8_t* __restrict__ codes,
                                                        uint8_t* __restrict__ rlen) {
  __shared__ int32_t d_s[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) d_s[i] = i < nd ? dict[i] : INT32_MAX;
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += stride) {
    const int64_t a = rp[i], b = rp[i + 1];
    rlen[i] = (uint8_t)(b - a);
    int64_t prev = row0 + i;
    for (int64_t j = a; j < b; ++j) {
      const int64_t c = col[j];
      const int32_t d = (int32_t)(c - prev);
      prev = c;
      int lo = 0, hi = nd - 1;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (d_s[mid] < d) lo = mid + 1; else hi = mid;
      }
      codes[j] = (uint8_t)lo;
    }
  }
}

void launch_d8_encode(const MatView& A, int64_t row0, const int32_t* dict_dev, int nd, uint8_t* codes, uint8_t* rlen,
                      cudaStream_t s) {
  if (A.m == 0) return;
  int64_t g = (A.m + kNT - 1) / kNT;
  if (g > dev_sm_count() * 32) g = dev_sm_count() * 32;
  if (A.rp_bytes == 8)
    d8_encode_kernel<int64_t><<<(unsigned)g, kNT, 0, s>>>((const int64_t*)A.rowptr, A.col, A.m, row0, dict_dev, nd,
                                                          codes, rlen);
  else
    d8_encode_kernel<int32_t><<<(unsigned)g, kNT, 0, s>>>((const int32_t*)A.rowptr, A.col, A.m, row0, dict_dev, nd,
                                                          codes, rlen);
}

// Export (tests): colind re-decoded from codes / rlen / dict, one thread per
// row (row starts from the plan's rowptr; the SpMV itself never reads it)
template <typename RP>
__global__ void __launch_bounds__(kNT) d8_decode_kernel(const RP* __restrict__ rp, int64_t m, int64_t row0,
                                                        const uint8_t* __restrict__ codes,
                                                        const uint8_t* __restrict__ rlen,
                                                        const int32_t* __restrict__ dict, int bits,
                                                        int32_t* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * kNT + threadIdx.x;
  if (i >= m) return;
  const int64_t a = rp[i];
  int64_t c = row0 + i;
  for (int t = 0; t < rlen[i]; ++t) {
    const int64_t j = a + t;
    c += dict[bits == 8 ? codes[j] : (codes[j >> 1] >> ((j & 1) << 2)) & 15];
    out[a + t] = (int32_t)c;
  }
}

void launch_d8_decode_export(const StreamPlan& sp, const int32_t* dict_dev, int32_t* out, cudaStream_t s) {
  if (sp.V.m == 0) return;
  const unsigned g = (unsigned)((sp.V.m + kNT - 1) / kNT);
  if (sp.V.rp_bytes == 8)
    d8_decode_kernel<int64_t><<<g, kNT, 0, s>>>((const int64_t*)sp.V.rowptr, sp.V.m, sp.row0, sp.codes, sp.rlen,
                                                dict_dev, sp.d8_bits, out);
  else
    d8_decode_kernel<int32_t><<<g, kNT, 0, s>>>((const int32_t*)sp.V.rowptr, sp.V.m, sp.row0, sp.codes, sp.rlen,
                                                dict_dev, sp.d8_bits, out);
}


// ---- row patterns (plan time; reading 31) --------------------------
// Pattern of row i = its length and the offsets colind[j] - i. Pass 1 hashes
// every row and collects the distinct hashes with their first row (per-CTA
// shared-memory table, then a 1024-slot global table); the host numbers the
// patterns by first row and reads their offsets from those rows; pass 2 maps
// each row's hash to its pattern and VERIFIES the row against the pattern's
// offsets (a hash collision fails the plan over to the 8-bit codes).
constexpr int kPatLocal = 512;

__device__ __forceinline__ unsigned long long pat_hash(const int32_t* __restrict__ col, int64_t a, int64_t b,
                                                       int64_t rowid) {
  unsigned long long h = 0x9E3779B97F4A7C15ull ^ (unsigned long long)(b - a);
  for (int64_t j = a; j < b; ++j) {
    const unsigned long long o = (unsigned long long)(uint32_t)(int32_t)((int64_t)col[j] - rowid);
    h = (h ^ o) * 0x100000001B3ull;
    h ^= h >> 29;
  }
  h ^= h >> 32;
  h *= 0xD6E8FEB86659FD93ull;
  h ^= h >> 32;
  return h | 1ull;  // 0 marks an empty slot
}

template <typename RP>
__global__ void __launch_bounds__(kNT) pat_collect_kernel(const RP* __restrict__ rp, const int32_t* __restrict__ col,
                                                          int64_t m, int64_t row0, unsigned long long* __restrict__ gkey,
                                                          unsigned long long* __restrict__ gfirst, int* __restrict__ flag) {
  __shared__ unsigned long long key[kPatLocal], first[kPatLocal];
  __shared__ int cnt;
  for (int i = threadIdx.x; i < kPatLocal; i += kNT) {
    key[i] = 0ull;
    first[i] = ~0ull;
  }
  if (threadIdx.x == 0) cnt = 0;
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * kNT;
  for (int64_t i = (int64_t)blockIdx.x * kNT + threadIdx.x; i < m; i += stride) {
    const int64_t a = rp[i], b = rp[i + 1];
    if (b - a > 255) {
      atomicOr(flag, 1);
      break;
    }
    const unsigned long long h = pat_hash(col, a, b, row0 + i);
    unsigned sl = (unsigned)(h >> 40) & (kPatLocal - 1);
    for (int probe = 0; probe < kPatLocal; ++probe, sl = (sl + 1) & (kPatLocal - 1)) {
      unsigned long long k = key[sl];
      if (k == 0ull) {
        k = atomicCAS(&key[sl], 0ull, h);
        if (k == 0ull) {
          atomicAdd(&cnt, 1);
          k = h;
        }
      }
      if (k == h) {
        if ((unsigned long long)i < first[sl]) atomicMin(&first[sl], (unsigned long long)i);
        break;
      }
    }
  }
  __syncthreads();
  if (cnt > 256) {
    if (threadIdx.x == 0) atomicOr(flag, 2);
    return;
  }
  for (int t = threadIdx.x; t < kPatLocal; t += kNT) {
    const unsigned long long h = key[t];
    if (!h) continue;
    unsigned sl = (unsigned)(h >> 40) & (kPatGlobal - 1);
    for (int probe = 0; probe < kPatGlobal; ++probe, sl = (sl + 1) & (kPatGlobal - 1)) {
      const unsigned long long k = atomicCAS(&gkey[sl], 0ull, h);
      if (k == 0ull || k == h) {
        atomicMin(&gfirst[sl], first[t]);
        break;
      }
    }
  }
}

// pass 2: ids[i] = the pattern of row i (skey: the patterns' hashes sorted,
// sid: their ids); flag |= 4 when a hash is not found, 8 when a row differs
// from its pattern (collision)
template <typename RP>
__global__ void __launch_bounds__(kNT) pat_assign_kernel(const RP* __restrict__ rp, const int32_t* __restrict__ col,
                                                         int64_t m, int64_t row0,
                                                         const unsigned long long* __restrict__ skey,
                                                         const int32_t* __restrict__ sid, int np,
                                                         const int32_t* __restrict__ desc,
                                                         const int32_t* __restrict__ pofs, int npofs,
                                                         uint8_t* __restrict__ ids, int* __restrict__ flag) {
  __shared__ unsigned long long k_s[256];
  __shared__ int32_t id_s[256], d_s[256];
  __shared__ int32_t o_s[kPatMaxOfs];
  for (int i = threadIdx.x; i < 256; i += kNT) {
    k_s[i] = i < np ? skey[i] : ~0ull;
    id_s[i] = i < np ? sid[i] : 0;
    d_s[i] = i < np ? desc[i] : 0;
  }
  for (int i = threadIdx.x; i < npofs; i += kNT) o_s[i] = pofs[i];
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * kNT;
  for (int64_t i = (int64_t)blockIdx.x * kNT + threadIdx.x; i < m; i += stride) {
    const int64_t a = rp[i], b = rp[i + 1];
    const unsigned long long h = pat_hash(col, a, b, row0 + i);
    int lo = 0, hi = np - 1;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (k_s[mid] < h) lo = mid + 1; else hi = mid;
    }
    if (np == 0 || k_s[lo] != h) {
      atomicOr(flag, 4);
      continue;
    }
    const int pid = id_s[lo], d = d_s[pid];
    bool same = ((d >> 16) & 0xff) == (int)(b - a);
    for (int64_t j = a; same && j < b; ++j) same = o_s[(d & 0xffff) + (j - a)] == (int32_t)((int64_t)col[j] - (row0 + i));
    if (!same) atomicOr(flag, 8);
    ids[i] = (uint8_t)pid;
  }
}

void launch_pat_collect(const MatView& A, int64_t row0, unsigned long long* gkey, unsigned long long* gfirst,
                        int* flag, cudaStream_t s) {
  if (A.m == 0) return;
  int64_t g = (A.m + kNT - 1) / kNT;
  if (g > dev_sm_count() * 8) g = dev_sm_count() * 8;
  if (A.rp_bytes == 8)
    pat_collect_kernel<int64_t><<<(unsigned)g, kNT, 0, s>>>((const int64_t*)A.rowptr, A.col, A.m, row0, gkey,
                                                            gfirst, flag);
  else
    pat_collect_kernel<int32_t><<<(unsigned)g, kNT, 0, s>>>((const int32_t*)A.rowptr, A.col, A.m, row0, gkey,
                                                            gfirst, flag);
}

void launch_pat_assign(const MatView& A, int64_t row0, const unsigned long long* skey, const int32_t* sid, int np,
                       const int32_t* desc, const int32_t* pofs, int npofs, uint8_t* ids, int* flag, cudaStream_t s) {
  if (A.m == 0) return;
  int64_t g = (A.m + kNT - 1) / kNT;
  if (g > dev_sm_count() * 8) g = dev_sm_count() * 8;
  if (A.rp_bytes == 8)
    pat_assign_kernel<int64_t><<<(unsigned)g, kNT, 0, s>>>((const int64_t*)A.rowptr, A.col, A.m, row0, skey, sid,
                                                           np, desc, pofs, npofs, ids, flag);
  else
    pat_assign_kernel<int32_t><<<(unsigned)g, kNT, 0, s>>>((const int32_t*)A.rowptr, A.col, A.m, row0, skey, sid,
                                                           np, desc, pofs, npofs, ids, flag);
}

// Export (tests): colind re-decoded from the row patterns (one thread per row)
template <typename RP>
__global__ void __launch_bounds__(kNT) pat_decode_kernel(const RP* __restrict__ rp, int64_t m, int64_t row0,
                                                         const uint8_t* __restrict__ ids,
                                                         const int32_t* __restrict__ desc,
                                                         const int32_t* __restrict__ pofs, int32_t* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * kNT + threadIdx.x;
  if (i >= m) return;
  const int d = desc[ids[i]];
  for (int t = 0; t < ((d >> 16) & 0xff); ++t) out[(int64_t)rp[i] + t] = (int32_t)(row0 + i + pofs[(d & 0xffff) + t]);
}

void launch_pat_decode_export(const StreamPlan& sp, int32_t* out, cudaStream_t s) {
  if (sp.V.m == 0) return;
  const unsigned g = (unsigned)((sp.V.m + kNT - 1) / kNT);
  if (sp.V.rp_bytes == 8)
    pat_decode_kernel<int64_t><<<g, kNT, 0, s>>>((const int64_t*)sp.V.rowptr, sp.V.m, sp.row0, sp.rlen,
                                                 sp.d8_dict_dev, sp.pat_ofs, out);
  else
    pat_decode_kernel<int32_t><<<g, kNT, 0, s>>>((const int32_t*)sp.V.rowptr, sp.V.m, sp.row0, sp.rlen,
                                                 sp.d8_dict_dev, sp.pat_ofs, out);
}

}  // namespace spmv
