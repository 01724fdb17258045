// internal.h -- host-side declarations shared by api.cu and the kernel files.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace spmv {

constexpr int kNT = 256;  // threads per CTA for every SpMV kernel
constexpr int kNormPartials = 512;  // fixed row chunking of the norm reduction
#ifndef STREAM_CW
#define STREAM_CW 4
#endif
constexpr int kStreamConsumerWarps = STREAM_CW;  // cta_stream consumer warps per CTA (stages: multiple of this)
constexpr int64_t kShortRowMax = 32;  // SPLIT: rows up to this length form the one-lane-per-row bin

// Device-side inspector accumulators (integers only => order-independent).
struct DevStats {
  unsigned long long s1, s2, s1_short, s2_short;
  long long nnz_min, nnz_max, n_empty, n_long, nnz_long, n_short, max_short;
  long long maxgap, misses;
  long long rp_err;   // smallest row i with rowptr[i+1] < rowptr[i] (LLONG_MAX if none)
  long long col_err;  // min over nonzeros of 2*j + (order violation ? 1 : 0) (LLONG_MAX if none)
  long long n_incoming;  // STREAM tiles with an incoming row (carry fix-up needed)
  long long col_min, col_max;  // column range touched (LLONG_MAX / -1 if no nonzero)
  // distinct in-row gaps >= kEsc0 (escape-coded D16): open-addressing set,
  // 0 = empty slot; big_over = 1 when more than kBigTab distinct values
  int32_t bigtab[128];
  int32_t big_over;
  // x-line reuse probe: sampled rows r, nonzeros of r whose 128-B x line row
  // r-1 also reads (hits) out of the sampled nonzeros (tot)
  unsigned long long reuse_hit, reuse_tot;
  // distinct row-relative deltas (D8, reading 26): head deltas
  // colind[rowptr[i]] - (row0 + i) and in-row gaps; open-addressing set,
  // INT32_MIN = empty slot; d_over = 1 once more than kD8Max distinct values
  int32_t dtab[1024];
  int32_t d_count, d_over;
};
constexpr int kDTab = 1024;  // global distinct-delta table slots
constexpr int kD8Max = 256;  // dictionary entries (one byte per code)
constexpr int kD8MaxRow = 255;  // row lengths stored in one byte
// escape-coded 16-bit deltas (SURVEY 8(f) f3 reading; reading 21):
// a delta d < kEsc0 is stored as d, a delta d >= kEsc0 as kEsc0 + (index of d
// in the plan's sorted table of distinct large deltas, at most kEscMax)
constexpr int kEsc0 = 65536 - 64;
constexpr int kEscMax = 64;
constexpr int kBigTab = 128;

// iterated-mode epilogue fused into the row-aligned persistent SpMV kernels
// (iterfuse.cuh): pending exact rescale of the previous step, per-CTA sums of
// squares folded into kNormPartials rank partials by the last CTA, and for a
// single rank the norm step itself
struct IterOut {
  const double* scale = nullptr;  // pending factor of the previous step (nn + 1; 0 = none), or null
  double* cta_part = nullptr;     // [grid] per-CTA sums of squares (null: no partials)
  unsigned int* done = nullptr;   // ticket counter (zero between launches)
  double* partials = nullptr;     // [kNormPartials] rank partials
  double* nn = nullptr;           // non-null: fused norm step (single rank), nn[0..1]
  double* nu_k = nullptr;
  // single-rank iteration, nothing between two SpMVs ("lagged" mode): every
  // CTA stores its sum of squares; the LAST CTA (the one with the fewest
  // tiles) then folds the PREVIOUS launch's sums (prev_part[0..prev_grid))
  // into ||yh_{k-1}||, writes nu_{k-1} (*nu_k) and decides the exact factor
  // the NEXT launch applies, from ||yh_{k-1}|| and this launch's factor
  // (state st[0..3] = N_{k-1}, F_k, and the factors by launch parity
  // st[2 + par]; reading 27)
  const double* prev_part = nullptr;
  int prev_grid = 0;
  int par = 0;  // launch parity (k & 1)
  int rev = 0;  // D8: walk the tiles from the end (every other iteration: x lines still in L2)
  double* st = nullptr;
  bool cta_only = false;
  // multi-shard iteration, halo push: the kernel also stores
  // its rows [0, push_lo_end) into push_lo and [push_hi_begin, m) into
  // push_hi -- a neighbour shard's next replica (peer memory over NVLink, or
  // the same device when emulated), pre-offset so index r is local row r
  double* push_lo = nullptr;
  int64_t push_lo_end = 0;
  double* push_hi = nullptr;
  int64_t push_hi_begin = 0;
};

// the y store of the iterated kernels: own block + the neighbours' replicas
__device__ __forceinline__ void iter_store(const IterOut& it, double* y, int64_t r, double v) {
  y[r] = v;
  if (it.push_lo && r < it.push_lo_end) it.push_lo[r] = v;
  if (it.push_hi && r >= it.push_hi_begin) it.push_hi[r] = v;
}

struct MatView {
  int rp_bytes;
  const void* rowptr;   // int32 or int64 [m+1]
  const int32_t* col;   // [nnz]
  const double* val;    // [nnz]
  int64_t m, n_cols, nnz;
};

// One cta_stream pass over the CSR view V (the whole shard, or one compacted
// length bin of long_row_split whose row q is row rowmap[q] of y).
struct StreamPlan {
  MatView V{};
  const int32_t* rowmap = nullptr;  // nullptr = identity
  int64_t C = 0, T = 0;
  int32_t* tile_row = nullptr;
  int32_t* carry_row = nullptr;
  double* carry_val = nullptr;
  bool need_fixup = false;
  const uint16_t* dcol = nullptr;  // D16 stream (nullptr = int32 colind)
  int n_esc = 0;                   // escape-coded large deltas (<= kEscMax)
  int32_t esc[kEscMax] = {};       // sorted distinct deltas >= kEsc0
  const int32_t* head = nullptr;
  const int32_t* anchor = nullptr;
  int stages = 0, grid = 0, vs = 1, rows_cap = 0;
  bool seg = false;  // segmented consumer mode (random-gather tiles)
  bool aligned = false;  // row-aligned tiles: tile k = rows starting in [k*stride, (k+1)*stride)
  int64_t stride = 0;    // tile stride in nonzeros (C, or C - longest row when aligned)
  int64_t* tile_nz = nullptr;  // aligned: tile_nz[k] = rowptr[tile_row[k]], k = 0..T
  int64_t max_run = 1;         // longest run of equal carry rows (fix-up choice)
  bool l2pf = false;           // producer L2-prefetches each stage's next tile (measured slower: C2 53.7 vs 47.0 us)
  int64_t k0 = 0;              // first tile of the launch (tile-range launches: pipelined host execute)
  int64_t rows_per_tile = 0;   // > 0: row-count tiles (tile k = rows [k*rpt, (k+1)*rpt), aligned)
  IterOut it{};                // launch-time: iterated-mode epilogue (row-aligned tiles; iterfuse.cuh)
  // D8 (dictionary-coded 8-bit deltas, d8.cu): codes[nnz], rlen[m], dict; row-count tiles only
  const uint8_t* codes = nullptr;
  const uint8_t* rlen = nullptr;
  int n_dict = 0;
  int32_t dict[256] = {};
  int64_t row0 = 0;            // row id of local row 0 (anchor of the head deltas)
  const int32_t* d8_dict_dev = nullptr;  // the dictionary on the device (export decode)
  int d8_un = 8;               // D8 codes decoded + x gathers in flight per lane per batch (8 or 16)
  int d8_bits = 8;             // D8 bits per code: 8, or 4 (two per byte) when the dictionary has <= 16 entries;
                               // 0: row-pattern mode (rlen holds each row's pattern id; dict = pattern descriptors
                               // len << 16 | first offset; pat_ofs = the patterns' column offsets from the row id)
  const int32_t* pat_ofs = nullptr;
  int n_pat_ofs = 0;
  const unsigned char* d8_tiles = nullptr;  // packed tiles: [values | codes | row lengths] per tile (one TMA copy)
  const int64_t* d8_toff = nullptr;         // their byte offsets [T+1]
};
size_t d8_smem_bytes(int64_t C, int64_t Rt, int stages, int CB = 8, int64_t npofs = 0);
// row patterns (reading 31): <= 256 patterns, <= kPatMaxOfs offsets in total
constexpr int kPatGlobal = 1024;   // slots of the plan-time hash table
constexpr int kPatMaxOfs = 4096;
void launch_pat_collect(const MatView& A, int64_t row0, unsigned long long* gkey, unsigned long long* gfirst,
                        int* flag, cudaStream_t s);
void launch_pat_assign(const MatView& A, int64_t row0, const unsigned long long* skey, const int32_t* sid, int np,
                       const int32_t* desc, const int32_t* pofs, int npofs, uint8_t* ids, int* flag, cudaStream_t s);
void launch_pat_decode_export(const StreamPlan& sp, int32_t* out, cudaStream_t s);
int d8_prepare(const StreamPlan& sp, int sm_count);  // stages = consumer warps (4, 6, 8)
bool d8_push_capable(const StreamPlan& sp);           // has the halo-push instantiation
bool stream_push_capable(const StreamPlan& sp);       // STREAM / D8 iterated kernel with the halo push
int d8_per_sm(const StreamPlan& sp);                 // resident CTAs per SM (after d8_prepare)
void launch_d8(const StreamPlan& sp, const double* x, double* y, cudaStream_t s);
void launch_d8_encode(const MatView& A, int64_t row0, const int32_t* dict_dev, int nd, uint8_t* codes, uint8_t* rlen,
                      cudaStream_t s);
void launch_d8_pack4(const uint8_t* codes, int64_t nnz, uint8_t* packed, cudaStream_t s);
void launch_d8_pack_tiles(const StreamPlan& sp, const int64_t* toff, unsigned char* tiles, cudaStream_t s);
void launch_d8_decode_export(const StreamPlan& sp, const int32_t* dict_dev, int32_t* out, cudaStream_t s);
// row-aligned STREAM / D8 plan (no fix-up) with the iterated-mode epilogue
int launch_stream_iter(const StreamPlan& sp, const double* x, double* y, const IterOut& it, cudaStream_t s);
// the same over tiles [k0, k1) (the epilogue folds this launch's CTAs only)
int launch_stream_iter_range(const StreamPlan& sp, const double* x, double* y, const IterOut& it, int64_t k0,
                             int64_t k1, cudaStream_t s);
// out[0] = 1 + largest nonzero index with col < lo (0: none), out[1] = smallest
// with col >= hi (nnz: none); out preset to {0, nnz} by the caller
void launch_halo_extent(const int32_t* col, int64_t nnz, int64_t lo, int64_t hi, unsigned long long* out,
                        cudaStream_t s);
void launch_tile_rows_count(int32_t* tile_row, int64_t T, int64_t rows_per_tile, int64_t m, cudaStream_t s);
// tiles [k0, k1) of a STREAM plan (+ the fix-up of their carries); the rows
// cut at k0 / k1 are completed by the neighbouring ranges' fix-ups
int launch_stream_range(const StreamPlan& sp, const double* x, double* y, int64_t k0, int64_t k1, cudaStream_t s);
// out[0] = max colind over nonzeros [a, b) (atomicMax; out zeroed by the caller)
void launch_range_colmax(const int32_t* col, int64_t a, int64_t b, int32_t* out, cudaStream_t s);
void launch_tile_nz(const MatView& A, const int32_t* tile_row, int64_t T, int64_t* tile_nz, cudaStream_t s);

// One nnz_split pass (nzsplit.cu) over the CSR view V restricted to its
// non-empty rows: rpc[mc+1] (rowptr of the non-empty rows, V's rowptr type),
// rowmap[mc+1] (y row of each, rowmap[mc] = m_out), warp tiles of kNzTile
// nonzeros with tile_q[k] = the non-empty row holding nonzero k*kNzTile.
constexpr int64_t kNzTile = 256;
struct NzPlan {
  MatView V{};                      // colind / values / nnz (V.rowptr unused by the kernel)
  const void* rpc = nullptr;
  const int32_t* rowmap = nullptr;
  int32_t* tile_q = nullptr;
  uint32_t* emask = nullptr;  // [T][8] row-end bits of each 256-nonzero tile
  uint64_t* epre = nullptr;   // [T] per-word prefix counts of emask (bytes)
  bool gather_l2 = false;     // x gathers bypass L1 (.cg): rows share no x lines with their neighbours
  int32_t* carry_row = nullptr;
  double* carry_val = nullptr;
  int64_t mc = 0, T = 0, m_out = 0;
  int grid = 0;
  int64_t max_run = 1;    // longest run of equal carry rows (fix-up choice)
  // hot-x mode: colind of the n_hot most frequent columns re-encoded as ~slot;
  // xhot[slot] = x[hot_cols[slot]] is refreshed per SpMV and staged in smem
  int n_hot = 0;
  const int32_t* hot_cols = nullptr;
  double* xhot = nullptr;
  bool zero_gaps = true;  // write y = 0 for the rows of [0, m_out) not in rowmap
  bool persistent = true;  // grid = resident CTAs (else one tile per warp: lets a concurrent kernel share the SMs)
  const void* skip_rp = nullptr;  // SPLIT: zero only the gap rows empty in this rowptr (long rows are written
                                  // concurrently by the long-row reduction)
  bool memset_y = false;  // a gap of more than kNzGapMax empty rows: y cleared before the pass, no gap zeroing
  bool skip_wait = false; // launched with PDL behind the long-row kernel, which waited for the previous SpMV
};
constexpr int32_t kNzGapMax = 4096;  // longest empty-row run a warp zeroes in-kernel
void launch_nz_tiles(const NzPlan& z, cudaStream_t s);  // tile_q and rowmap[mc] = m_out
void launch_nz_max_gap(const NzPlan& z, int32_t* out, cudaStream_t s);  // *out = longest run of rows not in rowmap
int nz_prepare(NzPlan& z, int sm_count);  // persistent grid (<0 on error)
// hot-x set (plan time): column counts + a count histogram of kHotBuckets,
// then the ordered compaction of the columns with count >= t (first K)
constexpr int kHotBuckets = 4096;
#ifndef SPMV_HOT_MAX
#define SPMV_HOT_MAX 16384
#endif
constexpr int kHotMax = SPMV_HOT_MAX;  // hot columns staged in smem (128 KB; B200 sweep on C3: 8K 283, 16K 275, 20K 285, 24K 322 us)
void launch_col_counts(const int32_t* col, int64_t nnz, int64_t n_cols, int32_t* cnt, int32_t* H, cudaStream_t s);
void launch_hot_flags(const int32_t* cnt, int64_t n_cols, int32_t t, int32_t* bsum, cudaStream_t s);
void launch_hot_write(const int32_t* cnt, int64_t n_cols, int32_t t, const int32_t* boff, int K, int32_t* hot_cols,
                      int32_t* slot, cudaStream_t s);
void launch_hot_encode(int32_t* col, int64_t nnz, const int32_t* slot, cudaStream_t s);
int launch_nz_plan(const NzPlan& z, const double* x, double* y, int stage, cudaStream_t s);
int launch_nz_prologue(const NzPlan& z, const double* x, double* y, cudaStream_t s);
int launch_nz_range(const NzPlan& z, const double* x, double* y, int64_t k0, int64_t k1, cudaStream_t s);
int launch_nz_fixup_range(const NzPlan& z, double* y, int64_t k0, int64_t k1, cudaStream_t s);

// ---- inspector ------------------------------------------------------------
void launch_rowstats(const MatView& A, int64_t l_split, int64_t row0, uint32_t* headbits, DevStats* st,
                     cudaStream_t s);
void launch_validate_gaps(const MatView& A, const uint32_t* headbits, DevStats* st, cudaStream_t s);
void launch_x_reuse(const MatView& A, DevStats* st, cudaStream_t s);  // DevStats reuse_hit / reuse_tot
void launch_tile_rows(const MatView& A, int64_t C, int64_t T, int32_t* tile_row, DevStats* st, cudaStream_t s);
void launch_merge_splits(const MatView& A, int64_t items, int64_t T, int32_t* mrow, int64_t* mnnz, cudaStream_t s);
// ordered list of rows with len > l_split and exclusive prefix of their chunk counts
void launch_long_rows(const MatView& A, int64_t l_split, int64_t chunk, int32_t* long_rows, int64_t n_long,
                      int64_t* chunk_start, int32_t* scratch_counts, int nblocks_scratch, cudaStream_t s);
void launch_d16_encode(const MatView& A, const uint32_t* headbits, int64_t C, int64_t T, uint16_t* dcol,
                       int32_t* head, int32_t* anchor, const int32_t* esc_dev, int n_esc, cudaStream_t s);
void launch_d16_decode_export(const StreamPlan& sp, int32_t* out, cudaStream_t s);
// ordered carry fix-up (vector.cu); the carry arrays must hold fixup_capacity(T)
// entries (levels of the hierarchical reduce-by-key live after the T carries)
int64_t fixup_capacity(int64_t T);
int launch_fixup(int32_t* crow, double* cval, int64_t T, double* y, int set, int64_t max_run, cudaStream_t s);
// fix-up of the carries of one tile range (crow/cval offset to the range start,
// T = its length): adds to y, uses no scratch, any run length
int launch_fixup_range(const int32_t* crow, const double* cval, int64_t T, double* y, cudaStream_t s);
void launch_rebase(void* rowptr, int rp_bytes, int64_t count, int64_t base, cudaStream_t s);

// ---- length bins (bins.cu) ----------------------------------------------------
int64_t scan_blocks(int64_t m);
// rowptr (and colind/values when out_col != null) of the rows with lo <= len <= hi,
// every other row empty (same row count)
void launch_filtered_csr(const MatView& A, int64_t lo, int64_t hi, void* out_rp, int32_t* out_col, double* out_val,
                         int64_t* scratch, cudaStream_t s);
// ordered list of the rows with lo <= len <= hi (count in scratch[scan_blocks(m)]; out may be null)
void launch_filtered_vals(const MatView& A, int64_t lo, int64_t hi, const void* out_rp, double* out_val,
                          cudaStream_t s);
void launch_row_list(const MatView& A, int64_t lo, int64_t hi, int32_t* out, int64_t* scratch, cudaStream_t s);
// compacted rowptr: out[q] = frp[rows[q]] (q < n), out[n] = frp[m]
void launch_gather_rowptr(const void* frp, int rp_bytes, const int32_t* rows, int64_t n, int64_t m, void* out,
                          cudaStream_t s);

// ---- SpMV variants ----------------------------------------------------------
struct ExecArgs {
  MatView A;
  const double* x;
  double* y;
  int vs;
  int sm_count;
  int64_t nnz_max;  // longest row (bounds the carry runs of the fix-ups)
  int stage;  // 0 = whole SpMV, 1 = main kernel(s) only, 2 = epilogue (fix-up) only
  // STREAM (sp[0]) / SPLIT bins (sp[0] short, sp[1] medium)
  StreamPlan sp[2];
  int n_sp;
  bool zero_y;  // SPLIT over compacted bins: y = 0 before the bin kernels
  // NNZSPLIT (whole shard) / SPLIT short+medium rows as one nnz_split bin
  NzPlan nz;
  bool use_nz;
  // SPLIT: long rows run on a side stream concurrently with the bins
  cudaStream_t side;
  cudaEvent_t ev_fork, ev_join;
  // MERGE
  int64_t items, Tm;
  const int32_t* mrow;
  const int64_t* mnnz;
  int32_t* mcarry_row;
  double* mcarry_val;
  // SPLIT long rows: nonzero chunks, or column-tiled (x block in smem)
  int64_t l_split, chunk, n_long, n_chunks;
  const int32_t* long_rows;
  const int64_t* chunk_start;
  int32_t* chunk_row;
  double* chunk_val;
  bool long_tiled;
  int64_t nblk;               // x blocks of kLongXB columns
  const int64_t* long_seg;    // [n_long][nblk+1] segment starts
  const uint16_t* long_c16;   // [nnz] (long rows' entries only): colind & (kLongXB - 1), or null
  double* long_partial;       // [n_long][nblk]
  int long_grid;              // persistent grid of the column-tiled kernel
  bool split_fused;           // SPLIT: nz bin + tiled long rows interleaved in one grid
  bool long_tma;              // SPLIT long_mode 3: TMA-staged tiled long rows (long_tma.cu) on the side stream
  int long_rg;                // its row groups per x block
};

#ifndef LONG_XB
#define LONG_XB 2048
#endif
constexpr int64_t kLongXB = LONG_XB;  // columns per x block staged in smem by the column-tiled long-row kernel
void launch_long_seg(const MatView& A, const int32_t* long_rows, int64_t n_long, int64_t nblk, int64_t* seg,
                     cudaStream_t s);
void launch_long_tiled(const ExecArgs& a, int part, cudaStream_t s);
void launch_long_c16(const MatView& A, const int32_t* long_rows, int64_t n_long, uint16_t* c16, cudaStream_t s);
int long_tiled_grid(int64_t nblk, int sm_count, int per_sm);
size_t long_tma_smem_bytes();
int long_tma_prepare();                                        // smem attribute (< 0 on error)
int long_tma_rg(int64_t n_long, int64_t nblk, int sm_count);   // row groups per x block (<= 32 rows per warp)
void launch_long_tma(const ExecArgs& a, int sm_count, cudaStream_t s);

int launch_vector(const ExecArgs& a, bool skip_long, cudaStream_t s);  // returns #launches
int launch_stream_plan(const StreamPlan& sp, const double* x, double* y, int stage, cudaStream_t s);
int launch_stream(const ExecArgs& a, cudaStream_t s);
int launch_merge(const ExecArgs& a, cudaStream_t s);
int launch_split(const ExecArgs& a, cudaStream_t s);
int launch_nzsplit(const ExecArgs& a, cudaStream_t s);
int launch_split_fused(const ExecArgs& a, cudaStream_t s);  // nz bin + column-tiled long rows, one grid
size_t stream_smem_bytes(int64_t C, int stages, int rp_bytes, int rows_cap, bool d16, bool seg);
int stream_prepare(const StreamPlan& sp, int sm_count);  // smem attribute + persistent grid (<0 on error)
void launch_chunk_export(const ExecArgs& a, int64_t* out, cudaStream_t s);  // [row|begin|end] x n_chunks

// ---- profile-guided selection (profile.cu; Sec. III-B bounds, Fig. 4) -----------
struct ProfileBounds {
  double p_csr = 0, p_mb = 0, p_ml = 0, p_imb = 0, p_cmp = 0, p_peak = 0, bmax = 0;
  double p_stream = 0;  // second stage: the plain cta_stream kernel's rate (reading 30; 0 = not run)
  int ws_fits_l2 = 0, vs = 0, ctas = 0;
};
int run_profile_probes(const MatView& A, int vs, int sm_count, int64_t l2_bytes, double* x, double* y,
                       ProfileBounds& out, cudaStream_t s);

// ---- full Table I features (table1.cu; f4) ------------------------------------
struct Table1 {
  double bw_min = 0, bw_max = 0, bw_avg = 0, bw_sd = 0, scatter_avg = 0, scatter_sd = 0, clustering_avg = 0;
  int64_t n_nonempty = 0, misses_total = 0;
};
// hot_cols: the plan's hot-x column list when its colind copy is re-encoded (else null)
int compute_table1(const MatView& A, const int32_t* hot_cols, int sm_count, Table1& out, cudaStream_t s);

// ---- iterated mode -------------------------------------------------------------
int launch_norm_partials(const double* y, int64_t m, double* partials, cudaStream_t s);
// partials[q] = sum of v over the fixed chunk q of v[0..n) (no squares)
int launch_sum_partials(const double* v, int64_t n, double* partials, cudaStream_t s);
// deferred normalisation (norm.cu): nn[0..1] running norm / pending exact
// rescale factor (applied by the next SpMV or the final unit, never in place)
int launch_norm_step(const double* partials, int count, double* nn, double* nu_k, cudaStream_t s);
// non-fused variants: y *= nn[1] (pending factor; nn may be null) + partials of y^2
int launch_scale_partials(double* y, int64_t m, const double* nn, double* partials, cudaStream_t s);
// final step of the lagged iteration: n = fold of the last launch's per-CTA
// sums, *nu_last = n / (st[1] st[0]) (n when st[0] == 0), x_out = y / n
int launch_unit_fold(const double* y, int64_t m, const double* cta_part, int grid, const double* st, double* nu_last,
                     double* x_out, cudaStream_t s);
int launch_unit(const double* y, int64_t m, const double* nn, double* x_out, cudaStream_t s);
int launch_normalize(const double* y, int64_t m, const double* partials, int count, double* x_out,
                     double* nu_dev, cudaStream_t s);

}  // namespace spmv
