// internal.h -- host-side declarations shared by api.cu and kernels.cu.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace spmv {

constexpr int kNT = 256;  // threads per CTA for every SpMV kernel
constexpr int kNormPartials = 512;  // fixed row chunking of the norm reduction
constexpr int kStreamConsumerWarps = 4;  // cta_stream consumer warps per CTA (stages: multiple of this)

// Device-side inspector accumulators (integers only => order-independent).
struct DevStats {
  unsigned long long s1, s2, s1_short, s2_short;
  long long nnz_min, nnz_max, n_empty, n_long, nnz_long, n_short, max_short;
  long long maxgap, misses;
  long long rp_err;   // smallest row i with rowptr[i+1] < rowptr[i] (LLONG_MAX if none)
  long long col_err;  // min over nonzeros of 2*j + (order violation ? 1 : 0) (LLONG_MAX if none)
  long long n_incoming;  // STREAM tiles with an incoming row (carry fix-up needed)
};

struct MatView {
  int rp_bytes;
  const void* rowptr;   // int32 or int64 [m+1]
  const int32_t* col;   // [nnz]
  const double* val;    // [nnz]
  int64_t m, n_cols, nnz;
};

// ---- inspector ------------------------------------------------------------
void launch_rowstats(const MatView& A, int64_t l_split, uint32_t* headbits, DevStats* st, cudaStream_t s);
void launch_validate_gaps(const MatView& A, const uint32_t* headbits, DevStats* st, cudaStream_t s);
void launch_tile_rows(const MatView& A, int64_t C, int64_t T, int32_t* tile_row, DevStats* st, cudaStream_t s);
void launch_merge_splits(const MatView& A, int64_t items, int64_t T, int32_t* mrow, int64_t* mnnz, cudaStream_t s);
// ordered list of rows with len > l_split and exclusive prefix of their chunk counts
void launch_long_rows(const MatView& A, int64_t l_split, int64_t chunk, int32_t* long_rows, int64_t n_long,
                      int64_t* chunk_start, int32_t* scratch_counts, int nblocks_scratch, cudaStream_t s);
void launch_d16_encode(const MatView& A, const uint32_t* headbits, int64_t C, int64_t T, uint16_t* dcol,
                       int32_t* head, int32_t* anchor, cudaStream_t s);
void launch_d16_decode_export(const MatView& A, const uint16_t* dcol, const int32_t* head, const int32_t* anchor,
                              const int32_t* tile_row, int64_t C, int64_t T, int vs, int32_t* out, cudaStream_t s);
void launch_fixup(const int32_t* crow, const double* cval, int64_t T, double* y, int set, cudaStream_t s);

// ---- SpMV variants ----------------------------------------------------------
struct ExecArgs {
  MatView A;
  const double* x;
  double* y;
  int vs;
  int sm_count;
  int stage;  // 0 = whole SpMV, 1 = main kernel(s) only, 2 = epilogue (fix-up) only
  // STREAM
  int64_t C, T;
  const int32_t* tile_row;
  int32_t* carry_row;
  double* carry_val;
  bool need_fixup;
  const uint16_t* dcol;
  const int32_t* head;
  const int32_t* anchor;
  int stages;
  int stream_grid;
  bool seg;  // cta_stream segmented mode (random-gather tiles)
  // MERGE
  int64_t items, Tm;
  const int32_t* mrow;
  const int64_t* mnnz;
  int32_t* mcarry_row;
  double* mcarry_val;
  // SPLIT
  int64_t l_split, chunk, n_long, n_chunks;
  const int32_t* long_rows;
  const int64_t* chunk_start;
  int32_t* chunk_row;
  double* chunk_val;
  MatView S;                 // SPLIT: compacted short-row CSR (other rows empty)
  const int32_t* mid_rows;   // SPLIT: medium rows, one warp each
  int64_t n_mid;
};

constexpr int64_t kShortRowMax = 32;  // SPLIT: rows up to this length go to cta_stream (one lane per row)
int64_t scan_blocks(int64_t m);
void launch_filtered_csr(const MatView& A, int64_t lo, int64_t hi, void* out_rp, int32_t* out_col, double* out_val,
                         int64_t* scratch, cudaStream_t s);
void launch_row_list(const MatView& A, int64_t lo, int64_t hi, int32_t* out, int64_t* scratch, cudaStream_t s);
void launch_rowlist(const ExecArgs& a, const int32_t* rows, int64_t nrows, cudaStream_t s);

int launch_vector(const ExecArgs& a, bool skip_long, cudaStream_t s);  // returns #launches
int launch_stream(const ExecArgs& a, cudaStream_t s);
int launch_merge(const ExecArgs& a, cudaStream_t s);
int launch_split(const ExecArgs& a, cudaStream_t s);
size_t stream_smem_bytes(int64_t C, int stages, int rp_bytes, bool d16, bool seg);
int stream_prepare(const ExecArgs& a);  // smem attribute + persistent grid (<0 on error)
void launch_chunk_export(const ExecArgs& a, int64_t* out, cudaStream_t s);  // [row|begin|end] x n_chunks
void launch_rebase(void* rowptr, int rp_bytes, int64_t count, int64_t base, cudaStream_t s);

// ---- iterated mode -------------------------------------------------------------
int launch_norm_partials(const double* y, int64_t m, double* partials, cudaStream_t s);
int launch_normalize(const double* y, int64_t m, const double* partials, int count, double* x_out,
                     double* nu_dev, cudaStream_t s);

}  // namespace spmv
