// long_tma.cu -- TMA-staged column-tiled long rows for long_row_split
// (IMB decomposition: "every row is computed by all threads and a
// reduction of partial results follows"), the long_mode 3 variant of
// long_tiled.cu, run on the plan's side stream CONCURRENTLY with the short
// rows' nnz_split bin.
//
// Same work decomposition as long_tiled.cu: the columns are cut into x
// blocks of kLongXB columns, item (b, g) is x block b and the long rows
// q = g (mod rg), and each (row, block) segment [seg[q][b], seg[q][b+1])
// gives one partial[q][b], reduced per row in block order afterwards. What
// changes is how the bytes move:
//  * one persistent CTA per SM (grid = SM count), so the short-row bin's
//    CTAs fill the rest of every SM: the bin is bound by the L1 miss path
//    (random x gathers), this kernel by HBM streams, and they overlap;
//  * the x block is bulk-copied (cp.async.bulk) into one of two smem
//    buffers one item ahead (mbarrier xs_full): the last warp to leave item
//    k (a shared counter) refills its buffer with item k + 2;
//  * each warp is its own producer: lane 0 bulk-copies the next chunks
//    (<= kLtCH nonzeros of one row segment, colind and values, 16-B-aligned
//    windows around them) into the warp's kLtD-stage ring, the chunk's
//    metadata next to it, and the warp consumes them in order from smem
//    (colind, values, x all from shared memory), so kLtD chunks per warp are
//    in flight without holding them in registers (the register-prefetched
//    variant of long_tiled.cu spilled);
//  * the chunk stream continues across items: only the x buffers
//    synchronise the warps, never a CTA barrier.
//
// Measured on B200 and NOT auto-selected (long_mode = 3 forces it): C4's long
// rows alone 129 us vs 59 us for long_tiled.cu, C4 whole 195 vs 111 us with
// the fused grid. ncu: 8 warps per SM issue 33 % of cycles on the smem
// consumer loop (39 M instructions, stalls wait 39 % / short_scoreboard 20 %)
// while DRAM runs at 26 %; time scales with the chunk count, not the ring
// depth (256-nnz chunks 129 us, 512: 91 us, 128: 209 us; 4 or 6 stages
// equal), and the PDL-launched short-row bin claims the SMs before this
// side-stream grid starts, so the two hardly overlap. DESIGN.md section 6.
#include "tiles.cuh"

namespace spmv {

#ifndef LT_CH
#define LT_CH 256
#endif
#ifndef LT_D
#define LT_D 4
#endif
#ifndef LT_MINB
#define LT_MINB 4  // register cap 64: the short-row bin needs the rest of the register file
#endif
#ifndef LT_NW
#define LT_NW 8
#endif
constexpr int kLtCH = LT_CH;                  // nonzeros per chunk
constexpr int kLtD = LT_D;                    // ring stages per warp
constexpr int kLtNW = LT_NW;                  // warps per CTA
constexpr int kLtColB = (kLtCH + 8) * 4;      // colind window [e0 & ~3, (e1 + 3) & ~3)
constexpr int kLtValB = (kLtCH + 2) * 8;      // values window [e0 & ~1, (e1 + 1) & ~1)
constexpr int kLtStageB = kLtColB + kLtValB;  // multiple of 16
static_assert(kLtColB % 16 == 0 && kLtValB % 16 == 0, "bulk-copy windows must stay 16-B aligned");

struct LtMeta {        // one ring stage's chunk (written by lane 0 before its arrive)
  int64_t e0;          // first nonzero
  int32_t len;         // nonzeros
  int32_t q;           // long row (index into long_rows / partial)
  int32_t kk;          // the CTA's item sequence number (x buffer kk & 1)
  int32_t last;        // 1: the chunk ends the row's segment
};

constexpr size_t kLtXsB = (size_t)kLongXB * 8;
constexpr size_t kLtRingB = (size_t)kLtNW * kLtD * kLtStageB;
constexpr size_t kLtMetaB = (size_t)kLtNW * kLtD * sizeof(LtMeta);
constexpr size_t kLtBarB = (size_t)(kLtNW * kLtD + 4) * 8;

size_t long_tma_smem_bytes() { return 2 * kLtXsB + kLtRingB + kLtMetaB + kLtBarB; }

// x block of item kk into xs buffer kk & 1 (thread 0): a bulk copy of the
// even part, the odd last column of the last block by a plain store before
// the arrive (the buffer's readers acquire it through xs_full)
__device__ __forceinline__ void lt_stage_x(const LongP& p, int64_t it, double* xs, uint64_t* full, uint64_t pol) {
  const int64_t b = it / p.rg, c0 = b * kLongXB;
  const int cw = (int)((p.n_cols - c0) < kLongXB ? (p.n_cols - c0) : kLongXB);
  const int ce = cw & ~1;
  if (cw & 1) xs[cw - 1] = __ldg(p.x + c0 + cw - 1);
  fence_proxy_async();  // the buffer's earlier generic reads before the async writes
  mbar_arrive_expect_tx(full, (uint32_t)ce * 8);
  if (ce > 0) bulk_g2s(xs, p.x + c0, (uint32_t)ce * 8, full, pol);
  (void)pol;
}

__global__ void __launch_bounds__(kLtNW * 32, LT_MINB) long_tma_kernel(const LongP p, int64_t n_items) {
  extern __shared__ __align__(128) unsigned char sm[];
  double* xsb = reinterpret_cast<double*>(sm);  // 2 x kLongXB
  unsigned char* ring_all = sm + 2 * kLtXsB;
  LtMeta* meta_all = reinterpret_cast<LtMeta*>(ring_all + kLtRingB);
  uint64_t* bars = reinterpret_cast<uint64_t*>(ring_all + kLtRingB + kLtMetaB);
  uint64_t* xs_full = bars;                                      // [2], count 1 (+ tx)
  uint32_t* xs_left = reinterpret_cast<uint32_t*>(bars + 2);     // [2]: warps done with the buffer's item
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* ring = ring_all + (size_t)w * kLtD * kLtStageB;
  LtMeta* meta = meta_all + w * kLtD;
  uint64_t* bar = bars + 4 + w * kLtD;
  const int64_t my_items = (int64_t)blockIdx.x < n_items ? (n_items - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const uint64_t pol = policy_evict_first();
  if (threadIdx.x == 0) {
    mbar_init(&xs_full[0], 1);
    mbar_init(&xs_full[1], 1);
    xs_left[0] = xs_left[1] = 0;
  }
  if (lane == 0)
    for (int s = 0; s < kLtD; ++s) mbar_init(&bar[s], 1);
  fence_mbar_init();
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int64_t kk = 0; kk < 2 && kk < my_items; ++kk)
      lt_stage_x(p, blockIdx.x + kk * gridDim.x, xsb + (kk & 1) * kLongXB, &xs_full[kk & 1], pol);
  }
  const int64_t ld = p.nblk + 1;
  const int64_t qs = (int64_t)p.rg * kLtNW;  // row stride of a warp inside an item

  // producer cursor: item kp (its rows' segment bounds in lane j = row j of
  // the warp), row ji, offset pi inside the row's segment
  int64_t kp = -1;
  int nq = 0, ji = 0, nq_n = 0;
  int64_t pi = 0, sa = 0, sb = 0, sa_n = 0, sb_n = 0;
  bool pdone = my_items == 0;
  // lane j: the segment bounds of the warp's row j in item k (loads in flight
  // until used: the next item's bounds are fetched when an item starts)
  auto load_bounds = [&](int64_t k, int& n_, int64_t& a_, int64_t& b_) {
    n_ = 0;
    a_ = b_ = 0;
    if (k >= my_items) return;
    const int64_t it = blockIdx.x + k * gridDim.x, b = it / p.rg, g = it % p.rg;
    const int64_t q0 = g + (int64_t)p.rg * w;
    n_ = q0 < p.n_long ? (int)((p.n_long - 1 - q0) / qs) + 1 : 0;  // <= 32 (plan: rg)
    if (lane < n_) {
      const int64_t q = q0 + qs * lane;
      a_ = __ldg(p.seg + q * ld + b);
      b_ = __ldg(p.seg + q * ld + b + 1);
    }
  };
  auto next_item = [&]() {  // move the producer to item kp + 1 (warp-uniform)
    ++kp;
    ji = 0;
    pi = 0;
    nq = nq_n;
    sa = sa_n;
    sb = sb_n;
    if (kp >= my_items) {
      pdone = true;
      return;
    }
    if (lane < nq && sa == sb) {  // empty segment
      const int64_t it = blockIdx.x + kp * gridDim.x, g = it % p.rg;
      p.partial[(g + (int64_t)p.rg * w + qs * lane) * p.nblk + it / p.rg] = 0.0;
    }
    load_bounds(kp + 1, nq_n, sa_n, sb_n);
  };
  int tail = 0, head = 0, inflight = 0;
  uint32_t ph = 0;  // bit s: parity of stage s's next completion
  // issue the next chunk of this warp into stage `tail`; false when none is left
  auto issue = [&]() -> bool {
    while (!pdone) {
      if (ji < nq) {
        const int64_t s0 = __shfl_sync(0xffffffffu, sa, ji), s1 = __shfl_sync(0xffffffffu, sb, ji);
        if (s0 + pi < s1) {
          const int64_t e0 = s0 + pi, e1 = (s1 - e0) > kLtCH ? e0 + kLtCH : s1;
          if (lane == 0) {
            const int64_t it = blockIdx.x + kp * gridDim.x, g = it % p.rg;
            LtMeta& m = meta[tail];
            m.e0 = e0;
            m.len = (int32_t)(e1 - e0);
            m.q = (int32_t)(g + (int64_t)p.rg * w + qs * ji);
            m.kk = (int32_t)kp;
            m.last = e1 == s1;
            const int64_t a0 = e0 & ~(int64_t)3, a1 = (e1 + 3) & ~(int64_t)3;
            const int64_t v0 = e0 & ~(int64_t)1, v1 = (e1 + 1) & ~(int64_t)1;
            unsigned char* st = ring + (size_t)tail * kLtStageB;
            // (the stage's previous reads are ordered by the warp's __syncwarp
            // before this issue, as the empty-barrier handshake of the stream
            // kernels orders them)
            mbar_arrive_expect_tx(&bar[tail], (uint32_t)((a1 - a0) * 4 + (v1 - v0) * 8));
            bulk_g2s(st, p.col + a0, (uint32_t)((a1 - a0) * 4), &bar[tail], pol);
            bulk_g2s(st + kLtColB, p.val + v0, (uint32_t)((v1 - v0) * 8), &bar[tail], pol);
          }
          pi = e1 - s0;
          tail = tail + 1 == kLtD ? 0 : tail + 1;
          ++inflight;
          return true;
        }
        ++ji;
        pi = 0;
        continue;
      }
      next_item();
    }
    return false;
  };

  // consumer: every warp enters every item of its CTA in order (waits for
  // the item's x block, even with no chunk in it) and leaves it by counting
  // itself out; the last warp to leave item kc refills that buffer with item
  // kc + 2 (so no warp can count itself out of kc + 2 before the counter is
  // reset, and no buffer is rewritten while read)
  int64_t kc = -1;  // the item this warp is in
  auto advance_to = [&](int64_t k) {  // leave items up to k - 1, enter k (k = my_items: the end)
    while (kc < k) {
      if (kc >= 0) {
        __syncwarp();
        if (lane == 0) {
          const uint32_t B = (uint32_t)(kc & 1);
          if (atomicAdd(&xs_left[B], 1u) == kLtNW - 1) {
            xs_left[B] = 0;
            if (kc + 2 < my_items)
              lt_stage_x(p, blockIdx.x + (kc + 2) * gridDim.x, xsb + B * kLongXB, &xs_full[B], pol);
          }
        }
      }
      ++kc;
      if (kc < my_items) mbar_wait(&xs_full[kc & 1], (uint32_t)((kc >> 1) & 1));
    }
  };

  load_bounds(0, nq_n, sa_n, sb_n);
  next_item();
  double a0 = 0.0, a1 = 0.0;
  for (;;) {
    while (inflight < kLtD && issue()) {
    }
    if (inflight == 0) break;
    mbar_wait(&bar[head], (ph >> head) & 1u);
    ph ^= 1u << head;
    const LtMeta m = meta[head];
    if (m.kk != kc) advance_to(m.kk);
    const int64_t it = blockIdx.x + (int64_t)m.kk * gridDim.x, b = it / p.rg;
    const int c0 = (int)(b * kLongXB);
    const double* xs = xsb + (m.kk & 1) * kLongXB;
    const unsigned char* st = ring + (size_t)head * kLtStageB;
    const int32_t* cs = reinterpret_cast<const int32_t*>(st) + (m.e0 & 3);
    const double* vs = reinterpret_cast<const double*>(st + kLtColB) + (m.e0 & 1);
    SPMV_CHECK(m.len > 0 && m.len <= kLtCH && m.q >= 0 && m.q < p.n_long && b < p.nblk);
#ifdef SPMV_CHECKS
    for (int i = lane; i < m.len; i += 32) SPMV_CHECK(cs[i] - c0 >= 0 && cs[i] - c0 < kLongXB);
#endif
    int i = lane;
    for (; i + 32 < m.len; i += 64) {
      a0 = fma(vs[i], xs[cs[i] - c0], a0);
      a1 = fma(vs[i + 32], xs[cs[i + 32] - c0], a1);
    }
    if (i < m.len) a0 = fma(vs[i], xs[cs[i] - c0], a0);
    __syncwarp();
    head = head + 1 == kLtD ? 0 : head + 1;
    --inflight;
    if (m.last) {
      const double t = warp_sum(a0 + a1);
      if (lane == 0) p.partial[(int64_t)m.q * p.nblk + b] = t;
      a0 = a1 = 0.0;
    }
  }
  advance_to(my_items);  // every item entered (its x copy landed) and left
}

LongP long_params(const ExecArgs& a);

// rows of one warp inside an item must fit the 32 lanes: rg >= n_long / (32 NW)
int long_tma_rg(int64_t n_long, int64_t nblk, int sm_count) {
  int64_t rg = (n_long + 32 * kLtNW - 1) / (32 * kLtNW);
  const int64_t bal = (4 * (int64_t)sm_count + nblk - 1) / std::max<int64_t>(nblk, 1);  // >= 4 items per CTA
  if (bal > rg) rg = bal;
  if (rg > n_long) rg = std::max<int64_t>(n_long, 1);
  return (int)std::max<int64_t>(rg, 1);
}

int long_tma_prepare() {
  return cudaFuncSetAttribute(long_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)long_tma_smem_bytes()) == cudaSuccess
             ? 0
             : -1;
}

void launch_long_tma(const ExecArgs& a, int sm_count, cudaStream_t s) {
  LongP p = long_params(a);
  p.rg = a.long_rg;
  const int64_t items = a.nblk * p.rg;
  const int grid = (int)std::min<int64_t>(items, sm_count);
  long_tma_kernel<<<grid, kLtNW * 32, long_tma_smem_bytes(), s>>>(p, items);
}

}  // namespace spmv
