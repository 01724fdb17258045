/* spmv.h -- C ABI of the B200-native adaptive fp64 CSR SpMV library (libspmv.so).
 *
 * The method is Elafrou, Goumas, Koziris, arXiv 1711.05487 ("the paper";
 * P:n = /root/reference/PAPER.md line n, S:n = SPEC.md line n). The library
 * computes y = A*x for A in CSR (Sec. II, Fig. 2) after a cheap
 * inspector that extracts Theta(N) features (Table I), builds
 * nnz-balanced partitions (Sec. IV-A), optionally delta-encodes
 * the column indices (MB class, Sec. III-E) and selects one of the
 * optimisations of Table II re-designed for sm_100a.
 *
 * No C++ types, exceptions or torch types cross this boundary. Every call
 * returns a status (or NULL) and never throws. Failing calls set a
 * thread-local status/message readable with spmv_last_status()/_error().
 *
 * Conventions
 *  - Ownership: plan-creation calls read the caller's arrays synchronously and
 *    copy what they need; the caller keeps ownership and may free them on
 *    return. Array pointers may be host (pageable or pinned) or device
 *    memory of the plan's device; the library detects which.
 *  - Failure leaves no plan: on error *out is NULL and nothing leaks.
 *  - A plan is not reentrant (one call at a time per plan); distinct plans
 *    are independent. All floating-point data is IEEE fp64.
 *  - CSR invariants: rowptr[0] = 0, rowptr[n_rows] = nnz,
 *    nondecreasing; 0 <= colind < n_cols and strictly increasing inside a
 *    row (no duplicates). Empty rows are legal and give y_i = 0.0.
 */
#ifndef SPMV_H_
#define SPMV_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct spmv_plan_s* spmv_plan;

typedef enum {
  SPMV_OK = 0,
  SPMV_E_ARG = -1,          /* null pointer, negative size, bad option, ngpus out of range */
  SPMV_E_CSR = -2,          /* CSR invariant violated; spmv_last_error() names it and where */
  SPMV_E_CUDA = -3,         /* CUDA runtime error (message carries cudaGetErrorString) */
  SPMV_E_NCCL = -4,         /* reserved for the fused NVLink exchange */
  SPMV_E_NOMEM = -5,        /* device or host allocation failed */
  SPMV_E_UNSUPPORTED = -6,  /* n >= 2^31 (int32 colind) or nnz >= 2^31 with 32-bit rowptr */
  SPMV_E_ZERO_NORM = -7     /* iterated mode hit ||y|| == 0 */
} spmv_status;

/* Kernel variants (Table II re-designed for sm_100a). */
typedef enum {
  SPMV_VARIANT_AUTO = 0,    /* feature-guided selection (P:492-521 reading) */
  SPMV_VARIANT_VECTOR = 1,  /* csr_vector<VS>: VS lanes per row (CMP: unroll+vectorise) */
  SPMV_VARIANT_STREAM = 2,  /* cta_stream: TMA-staged fixed nnz tiles (MB: vectorised streaming) */
  SPMV_VARIANT_MERGE = 3,   /* merge_path: rows+nnz balanced (IMB "auto" schedule) */
  SPMV_VARIANT_SPLIT = 4,   /* long_row_split: long rows by column-tiled CTAs + the other rows (IMB decomposition, Fig. 7) */
  SPMV_VARIANT_NNZSPLIT = 5 /* nnz_split: equal-nonzero warp tiles over the non-empty rows, rows cut at tile edges
                               (nnz-balanced partition P:708-711 + decomposition P:608-621 at warp granularity) */
} spmv_variant;

/* Bottleneck classes (Sec. III-A) recorded by the selection. */
enum { SPMV_CLASS_MB = 1, SPMV_CLASS_ML = 2, SPMV_CLASS_IMB = 4, SPMV_CLASS_CMP = 8 };

typedef struct spmv_options {
  int32_t struct_size;     /* = sizeof(spmv_options); set by spmv_options_default */
  int32_t force_variant;   /* spmv_variant; 0 = feature-guided selection */
  int32_t force_vs;        /* lanes per row for VECTOR/STREAM/SPLIT reductions: 0 = auto, else 1,2,4,8,16,32 */
  int32_t d16;             /* delta colind (STREAM only): -1 auto, 0 off, 1 = 16-bit deltas when
                              encodable, 2 = dictionary-coded 8-bit deltas (D8) when codable (<= 256 distinct
                              row-relative deltas, rows <= 255 nonzeros; reading 26); a D8 plan whose
                              rows follow <= 256 (length, column offsets) patterns with <= 4096 offsets stores
                              one pattern byte per row instead (row-pattern mode, reading 31) */
  int32_t xwin;            /* L2 persistence window on x (ML analogue of P:599-606): -1 auto, 0 off, 1 on */
  int32_t validate;        /* 1 = check CSR invariants on the device (default), 0 = trust the input */
  int64_t l_split;         /* long-row threshold in nnz (0 = 4096) */
  int64_t k_long;          /* long rows trigger SPLIT when nnz_max > k_long * nnz_avg (0 = 100) */
  int64_t tile_nnz;        /* STREAM tile size C in nonzeros (0 = 512; multiple of 128, <= 16384) */
  int64_t merge_items;     /* MERGE items (rows + nnz) per CTA (0 = 2048; multiple of 256) */
  int64_t long_chunk;      /* SPLIT chunk size in nonzeros (0 = 8192; multiple of 256) */
  int32_t emulate_devices; /* ngpus > 1: 1 = place every shard on the current device (tests) */
  int32_t stages;          /* STREAM smem ring depth: 0 = auto (one stage per consumer warp), else a multiple of 4 <= 32 */
  int32_t seg;             /* STREAM / SPLIT short part, segmented consumer mode: -1 auto, 0 off, 1 on */
  int32_t long_mode;       /* SPLIT long rows: 0 auto, 1 nonzero chunks, 2 column-tiled (x block in smem),
                              3 column-tiled with TMA-staged chunks on the side stream (experiment, measured slower;
                              needs the nnz_split bin, split_bins != 0) */
  int32_t split_bins;      /* SPLIT non-long rows: -1 auto (one nnz_split bin), 0 cta_stream length bins, 1 nnz_split bin */
  int32_t hot_x;           /* NNZSPLIT hot-x table in smem: -1 auto (top columns cover >= 20 % of nnz), 0 off,
                              K > 0 = force, at most K (<= 16384) columns */
  int32_t select_mode;     /* 0 feature-guided (Table I features, default), 1 profile-guided (Sec. III-B bounds from
                              three timed micro-benchmarks + Fig. 4 rules; reading 22) */
  int32_t reserved[1];     /* reserved[0] = 1 disables row-aligned tiles (tests) */
  /* Fig. 4 hyperparameters of the profile-guided classifier. The paper tunes T_IMB and T_ML per
   * platform by grid search (1.24 / 1.25 on KNC); 0 selects the values of this library's
   * grid search on B200 (tools/tune_profile.py, profiles/r02_profile_tuning.json, reading 29);
   * pass 1.24 / 1.25 / 0.10 for the paper's. approx_tol: "P_CSR ~ P_MB" read as P_CSR >= (1 - tol) P_MB. */
  double t_imb, t_ml, approx_tol;
  int32_t force_classes;   /* profile-guided mode: -1 measure and classify (default); 0..15 = skip the probes and
                              apply Table II's mapping to this SPMV_CLASS_* set (the grid search times it) */
  int32_t pad_;
} spmv_options;

/* Theta(N) features (Table I) + counts used by the selection.
 * Integers are exact; nnz_sd = sqrt((double)(N*S2 - S1^2)) / N (128-bit difference). */
typedef struct spmv_features {
  int64_t n, nnz, nnz_min, nnz_max, n_empty, n_long, nnz_long, n_short, max_short;
  uint64_t s1, s2, s1_short, s2_short;
  int64_t maxgap;          /* max in-row column gap over non-head nonzeros (0 if none) */
  int64_t misses;          /* non-head nonzeros with gap > 16 (Table I misses_i, 128-B line) */
  double nnz_avg, nnz_sd, avg_short, sd_short;
  int64_t n_cols;          /* columns (x length); the long-row density test uses it */
  int64_t n_big_gaps;      /* distinct in-row gaps >= 65472 (129 = more than 128): escape-coded D16 needs <= 64 */
  int64_t col_min, col_max;/* smallest / largest column index (x range the rows read; 0 / -1 when nnz = 0):
                              the halo of a row block in the distributed iterated mode */
  int64_t n_deltas;        /* distinct row-relative deltas (head: colind[rowptr[i]] - i, else the in-row gap;
                              257 = more than 256): the D8 dictionary size (reading 26) */
} spmv_features;

typedef struct spmv_device_props {
  int32_t sm_count;
  int32_t cc_major, cc_minor;
  int32_t pad_;
  int64_t l2_bytes;              /* cudaDeviceProp::l2CacheSize */
  int64_t persisting_l2_max;     /* cudaDeviceProp::persistingL2CacheMaxSize */
  int64_t access_window_max;     /* cudaDeviceProp::accessPolicyMaxWindowSize */
  int64_t global_mem_bytes;
} spmv_device_props;

typedef struct spmv_selection {
  int32_t variant;   /* spmv_variant (never AUTO) */
  int32_t vs;        /* lanes per row */
  int32_t d16;       /* index stream: 0 int32 colind, 1 16-bit deltas, 2 dictionary-coded 8-bit deltas (D8) */
  int32_t xwin;      /* 1 when the x persistence window is set */
  int32_t classes;   /* SPMV_CLASS_* bitmask */
  int32_t seg;       /* 1: cta_stream runs in segmented mode (random gathers: products first, balanced row walk) */
} spmv_selection;

typedef struct spmv_plan_info {
  int64_t n_rows, n_cols, nnz;
  int32_t rowptr_bytes, ngpus;
  spmv_selection sel;
  spmv_features feat;
  int32_t d16_width;          /* 0, 8 or 16 (matrix-global, "never both") */
  int32_t d16_n_esc;          /* escape-coded large deltas (16-bit codes >= 65472, reading 21) */
  int64_t tile_nnz, n_tiles;  /* STREAM tiling */
  int64_t merge_items, n_merge_tiles;
  int64_t l_split, long_chunk, n_long_chunks;
  double upload_ms, inspect_ms, select_ms, encode_ms; /* plan-time breakdown */
  int64_t device_bytes;       /* device memory held by the plan (all shards) */
  int64_t shard_bounds[9];    /* b_0..b_G for G <= 8 (rows) */
  int64_t tile_stride;        /* STREAM tile stride in nonzeros (= tile_nnz, or tile_nnz - longest row) */
  int32_t tiles_row_aligned;  /* 1: tile k = rows starting in [k*stride, (k+1)*stride); no carries */
  int32_t rows_per_tile;      /* > 0: row-count tiles, tile k = rows [k*rows_per_tile, (k+1)*rows_per_tile) */
  int64_t n_nz_rows;          /* nnz_split: non-empty rows of the pass (mc) */
  int64_t n_nz_tiles;         /* nnz_split: warp tiles of 256 nonzeros */
  int64_t n_hot;              /* nnz_split: hot columns served from shared memory (0 = off) */
  double hot_cover;           /* fraction of nonzeros in the (candidate) hot columns */
  /* profile-guided mode (select_mode = 1): Sec. III-B bounds in flop/s and B_max in bytes/s; the Fig. 4
   * classes are sel.classes. p_csr/p_ml/p_cmp measured, p_imb from the median CTA busy time of the
   * static nnz-balanced baseline, p_mb/p_peak analytic. Zero in feature mode. */
  double p_csr, p_mb, p_ml, p_imb, p_cmp, p_peak, bmax;
  int32_t profile_vs, profile_ctas; /* baseline lanes per row, CTAs of its static partition */
  double profile_ms;          /* micro-benchmark time (part of select_ms: the classifier's t_pre) */
  double x_reuse;             /* sampled fraction of nonzeros whose 128-B x line the previous row also reads */
  int32_t nz_gather_l2;       /* nnz_split / split tiles gather x through L2 only (x_reuse < 0.5, x > 1 MB) */
  int32_t stream_stages;      /* STREAM: smem stages (= consumer warps per CTA) */
  int32_t d8_n_dict;          /* D8: dictionary entries (0 when D8 is not used) */
  int32_t stream_grid;        /* STREAM: persistent CTAs of shard 0's main kernel */
  int64_t kernel_bytes;       /* compulsory DRAM bytes of one SpMV in the plan's own format (all shards):
                                 values + the index streams the kernel reads + x (n_cols) + y (n_rows) */
  int32_t long_mode;          /* SPLIT long rows: 0 none, 1 nonzero chunks, 2 column-tiled (fused grid or side
                                 stream), 3 column-tiled TMA-staged on the side stream (long_tma.cu) */
  int32_t long_rg;            /* long_mode 2/3: row groups per x block */
  int32_t iter_push;          /* 1: the multi-shard iterated mode pushes each shard's halo rows into its
                                 neighbours' replicas from the SpMV kernel (banded row blocks; 0 = halo copies,
                                 or no spmv_iterate yet: decided at the first one) */
  int32_t long_c16;           /* 1: SPLIT's column-tiled long rows read 16-bit in-block columns (colind mod the
                                 2048-column x block) instead of int32 colind: 10 instead of 12 B per nonzero */
  double p_stream;            /* profile mode, second stage: flop/s of the plain cta_stream kernel when Fig. 4
                                 mapped the matrix to it and its indices are D8-codable; >= (1 - tol) P_MB adds
                                 MB and D8 (reading 30); 0 when not run */
  int32_t d8_patterns;        /* D8 row-pattern mode (reading 31): the rows' patterns (<= 256; one byte
                                 per row names its pattern, no per-nonzero index is read); 0 when not used */
  int32_t pad3_;
} spmv_plan_info;

/* ---- plan lifecycle ---------------------------------------------------- */

/* Fill *opt with defaults (auto selection, validation on). */
void spmv_options_default(spmv_options* opt);

/* Core call named by BJ.north_star. Square n x n matrix, int64 rowptr.
 * ngpus >= 1 shards rows nnz-balanced over devices 0..ngpus-1 of this
 * process (SURVEY 8(c2) bound rule) with x replicated.
 * Returns NULL on failure (see spmv_last_status / spmv_last_error). */
spmv_plan spmv_plan_create(int64_t n, int64_t nnz, const int64_t* rowptr, const int32_t* colind,
                           const double* values, int ngpus);

/* Extended creation: rectangular row blocks (n_rows x n_cols, e.g. one rank's
 * shard of a square matrix; colind are global column ids), rowptr of 4 or 8
 * bytes per entry, options (nullable). *out = NULL on failure. */
spmv_status spmv_plan_create_ex(spmv_plan* out, int64_t n_rows, int64_t n_cols, int64_t nnz,
                                const void* rowptr, int rowptr_bytes, const int32_t* colind,
                                const double* values, int ngpus, const spmv_options* opt);

/* NULL-safe; frees device memory and streams of every shard. */
void spmv_plan_destroy(spmv_plan p);

/* New values for the plan's matrix, same sparsity pattern (iterative solvers re-assemble values without
 * re-planning): values[nnz] in the CSR order given at creation, host or device memory, not retained.
 * Every value-derived copy the plan made (SPLIT bins, packed D8 tiles) is refreshed; the selection,
 * partitions and index encodings depend on the pattern only and are kept. Synchronous: waits for the
 * plan's earlier work. SPMV_E_ARG on a NULL plan or values. */
spmv_status spmv_plan_update_values(spmv_plan p, const double* values);

/* ---- execution ----------------------------------------------------------- */

/* y = A x (overwrite, Fig. 2 read as accumulation).
 * x: n_cols doubles, y: n_rows doubles, host or device. Synchronous. */
int spmv_execute(spmv_plan p, const double* x, double* y);

/* Same, enqueued on the plan's stream of shard 0 without a host sync.
 * Single-shard plans only; x and y must be device pointers of that device. */
int spmv_execute_async(spmv_plan p, const double* x, double* y);

/* As spmv_execute_async, restricted to one stage for per-kernel timing:
 * stage 0 = the whole SpMV, 1 = the main kernel(s) only, 2 = the carry
 * fix-up epilogue only (y is complete only after stages 1 and 2). */
int spmv_execute_stage(spmv_plan p, const double* x, double* y, int stage);

/* Iterated mode (BJ.configs[5]): x_0 = x0; for k < iters: y = A x_k,
 * nu_k = ||y||_2, x_{k+1} = y / nu_k. Writes x_iters to x_out (host or
 * device), nu_{iters-1} to *last_norm (nullable) and nu_0..nu_{iters-1} to
 * nu_out (nullable, host). Square plans only. Synchronous. Computed with
 * deferred normalisation (reading 25): yh_k = A yh_{k-1}
 * (yh_{-1} = x0), nu_k = ||yh_k|| / ||yh_{k-1}||, x_iters = yh_{iters-1} /
 * ||yh_{iters-1}||, magnitudes kept in range by exact power-of-two rescales;
 * equal to the per-step form up to rounding (SURVEY 8(c3) #21 tolerances).
 * SPMV_E_ZERO_NORM when some ||y|| is 0. */
spmv_status spmv_iterate(spmv_plan p, const double* x0, double* x_out, int iters, double* last_norm,
                         double* nu_out);

/* Building blocks of the distributed iterated mode (one process per GPU;
 * the exchange runs in the caller's NCCL process group). Single-shard
 * plans, device pointers, enqueued on the plan stream:
 *   spmv_norm_partials: partials[0..spmv_norm_partial_count()) = sums of
 *     y_i^2 over fixed contiguous row chunks of y (n_rows entries).
 *   spmv_normalize: nu = sqrt(sum_{q ascending} partials[q]) over `count`
 *     partials (all ranks' partials in rank order), x_out[i] = y[i] / nu,
 *     *nu_dev = nu. Every rank computes the identical nu. */
int32_t spmv_norm_partial_count(void);
int spmv_norm_partials(spmv_plan p, const double* y, double* partials);
int spmv_normalize(spmv_plan p, const double* y, const double* partials, int count, double* x_out,
                   double* nu_dev);
/* Deferred-normalisation steps (what spmv_iterate runs per shard; DESIGN.md
 * reading 25). nn: 2 device doubles of state, zeroed by the caller before
 * the first step; nn[0] = the running norm, nn[1] = a PENDING exact
 * power-of-two rescale factor (0 or 1: none) that the next spmv_iter_step
 * applies to its output and spmv_unit to the final x -- no pass ever
 * rescales a block in place.
 *   spmv_iter_step: y = s * (A x) with s = nn[1] (1 when 0), partials[0..
 *     spmv_norm_partial_count()) = sums of y_i^2 over fixed chunks (row-
 *     aligned STREAM / D8 plans: fixed per-CTA sums folded into the chunks by
 *     the kernel's last CTA), and, when nu_k is non-NULL, the norm step below
 *     on these partials alone (a single rank: one launch per iteration for
 *     fused plans). Device pointers of the plan's device, plan stream.
 *   spmv_norm_step: n = sqrt(sum of `count` partials, fixed order); *nu_k =
 *     n / nn[0] (n when nn[0] == 0, the first step); nn[0] = n scaled into
 *     [2^-256, 2^256] by an exact power of two, nn[1] = that factor (else 1).
 *     Every rank computes identical values from the gathered partials.
 *   spmv_unit: x_out[i] = y[i] * nn[1] / nn[0] for i < n (the final x =
 *     yh/||yh||; x_out may equal y). */
int spmv_iter_step(spmv_plan p, const double* x, double* y, double* partials, double* nn, double* nu_k);
int spmv_norm_step(spmv_plan p, const double* partials, int count, double* nn, double* nu_k);
/* spmv_execute_async(p, x, y) followed by the partials of y (as spmv_iter_step
 * with no pending factor and no norm step). */
int spmv_execute_norm(spmv_plan p, const double* x, double* y, double* partials);
int spmv_unit(spmv_plan p, const double* y, int64_t n, const double* nn, double* x_out);

/* Halo push across processes: the
 * one-process-per-GPU form of the exchange fused into the SpMV. For banded
 * row blocks the rows a neighbour rank reads from this rank's block are a
 * prefix (lower neighbour) and/or a suffix (upper neighbour) of it; the
 * iterated kernel stores those rows straight into the neighbours' next x
 * replicas (NVLink peer stores, CUDA IPC mappings) while it computes them,
 * so no separate exchange runs. Single-shard plans only.
 *   spmv_plan_replicas: the plan's two x replicas (n_cols doubles each,
 *     plan-owned, freed by spmv_plan_destroy; the second is allocated on the
 *     first call). The iterated mode ping-pongs between them; only these two
 *     buffers can be exported.
 *   spmv_iter_push_capable: 1 when the plan's iterated kernel (row-aligned
 *     STREAM / D8) has the halo-push instantiation, else 0 (NULL plan: 0).
 *   spmv_ipc_export: writes the SPMV_IPC_HANDLE_BYTES-byte CUDA IPC handle
 *     of `replica` (one of the two pointers above; else SPMV_E_ARG) to
 *     `handle` (host memory). The handle is sent to the peers by the caller.
 *   spmv_ipc_open: maps a peer's exported replica into this process on the
 *     plan's device (*ptr: its base, device memory of the peer's GPU;
 *     another process only: CUDA refuses a handle of the same process,
 *     SPMV_E_CUDA); unmapped by spmv_plan_destroy.
 *   spmv_iter_step_push: spmv_iter_step (no norm step) whose kernel also
 *     stores local rows [0, push_lo_end) into push_lo[r] and rows
 *     [push_hi_begin, m) into push_hi[r] (r = local row; the caller passes
 *     the peer replica's base + this block's first row). NULL push_lo /
 *     push_hi: no store on that side. SPMV_E_ARG when a range leaves
 *     [0, m]; SPMV_E_UNSUPPORTED when the plan is not push-capable.
 *     Ordering is the caller's: a peer's replica may be written only after
 *     the peer's previous SpMV finished reading it and read only after this
 *     launch completed (parallel.iterate: the per-iteration all-gather of the
 *     norm partials orders both). The kernel fences its peer stores at
 *     system scope before it completes. */
#define SPMV_IPC_HANDLE_BYTES 64
int spmv_plan_replicas(spmv_plan p, double** x_a, double** x_b);
int spmv_iter_push_capable(spmv_plan p);
int spmv_ipc_export(spmv_plan p, const double* replica, void* handle);
int spmv_ipc_open(spmv_plan p, const void* handle, double** ptr);
int spmv_iter_step_push(spmv_plan p, const double* x, double* y, double* partials, double* nn, double* push_lo,
                        int64_t push_lo_end, double* push_hi, int64_t push_hi_begin);

/* ---- inspection ---------------------------------------------------------- */

spmv_status spmv_plan_query(spmv_plan p, spmv_plan_info* info);

/* The full Table I feature vector, computed on
 * demand on the device for a single-shard plan (one Theta(N) + Theta(NNZ)
 * pass over rowptr/colind and one Theta(N) pass for the deviations; the
 * feature-guided selection itself only uses the nnz_* subset). Definitions
 * (reading 23): size = 1 iff the CSR + x + y working set fits in L2;
 * density = NNZ / (n_rows * n_cols); bw_i = last - first column + 1; scatter_i
 * = nnz_i / bw_i; clustering_i = ngroups_i / nnz_i (groups of consecutive
 * columns); misses_i = in-row gaps > 16 doubles (128-B line). nnz_* over all
 * rows (as spmv_features); bw_*, scatter_*, clustering_avg over the non-empty
 * rows; misses_avg over all rows; population standard deviations. */
typedef struct spmv_table1 {
  int32_t size_fits_l2, pad_;
  double density;
  double nnz_min, nnz_max, nnz_avg, nnz_sd;
  double bw_min, bw_max, bw_avg, bw_sd;
  double scatter_avg, scatter_sd, clustering_avg, misses_avg;
  int64_t n_nonempty;
} spmv_table1;
spmv_status spmv_plan_table1(spmv_plan p, spmv_table1* out);

/* Plan-resident buffers and stream of shard g (the timed path: no copies
 * when spmv_execute* receives these pointers). A host x given to
 * spmv_execute is copied into the replica only on the column range shard g
 * reads ([col_min, col_max] of its nonzeros: the halo of a banded row block),
 * the rest of the replica is left as it was. */
double* spmv_plan_x_device(spmv_plan p, int g);
double* spmv_plan_y_device(spmv_plan p, int g);
void* spmv_plan_stream(spmv_plan p, int g);  /* a cudaStream_t */

/* Copy a plan structure of shard g to host memory for bit-exact checks.
 * Returns the number of elements (call with dst = NULL to size), or < 0. */
enum {
  SPMV_ARR_TILE_ROWS = 1,    /* int64[n_tiles+1]: R_k = lower_bound(rowptr, k*C) */
  SPMV_ARR_MERGE_ROWS = 2,   /* int64[n_merge_tiles+1]: merge-path split i_k */
  SPMV_ARR_MERGE_NNZ = 3,    /* int64[n_merge_tiles+1]: merge-path split j_k */
  SPMV_ARR_CHUNK_ROW = 4,    /* int64[n_long_chunks] */
  SPMV_ARR_CHUNK_BEGIN = 5,  /* int64[n_long_chunks] */
  SPMV_ARR_CHUNK_END = 6,    /* int64[n_long_chunks] */
  SPMV_ARR_DCOL = 7,         /* uint16[nnz] delta colind */
  SPMV_ARR_HEAD = 8,         /* int32[n_rows] */
  SPMV_ARR_ANCHOR = 9,       /* int32[n_tiles] */
  SPMV_ARR_DECODED = 10,     /* int32[nnz] colind re-decoded on the device from dcol/head (D16), codes/rlen/dict (D8)
                                or the row patterns (D8 row-pattern mode) */
  SPMV_ARR_SHARD_BOUNDS = 11, /* int64[ngpus+1] */
  SPMV_ARR_NZ_ROWMAP = 12,    /* int64[mc+1]: nnz_split non-empty rows (y row ids), rowmap[mc] = n_rows */
  SPMV_ARR_NZ_RPC = 13,       /* int64[mc+1]: their rowptr (rpc[q] = rowptr[rowmap[q]], rpc[mc] = nnz) */
  SPMV_ARR_NZ_TILE_Q = 14,    /* int64[n_nz_tiles+1]: tile_q[k] = last q with rpc[q] <= 256k; tile_q[T] = mc */
  SPMV_ARR_NZ_HOT_COLS = 15,  /* int64[n_hot]: hot columns in column order (reading 20) */
  SPMV_ARR_D8_CODES = 16,     /* uint8[nnz]: D8 codes (index of each row-relative delta in the dictionary) */
  SPMV_ARR_D8_RLEN = 17,      /* uint8[n_rows]: D8 row lengths */
  SPMV_ARR_D8_DICT = 18,      /* int64[d8_n_dict]: D8 dictionary (ascending distinct deltas) */
  SPMV_ARR_PAT_IDS = 19,      /* uint8[n_rows]: row-pattern mode, each row's pattern (reading 31) */
  SPMV_ARR_PAT_LEN = 20,      /* int64[d8_patterns]: the patterns' lengths, numbered by first row */
  SPMV_ARR_PAT_OFS = 21       /* int64[sum of lengths]: their column offsets from the row id, pattern by pattern */
};
int64_t spmv_plan_export(spmv_plan p, int g, int which, void* dst);

/* nnz-balanced contiguous row partition:
 * b_0 = 0, b_G = n, b_g = min{ r : rowptr[r] >= ceil(g*nnz/G) }. Host
 * arrays. Returns SPMV_OK or SPMV_E_ARG. */
spmv_status spmv_shard_bounds(int64_t n, const void* rowptr, int rowptr_bytes, int G, int64_t* bounds);

/* The feature-guided selection as a pure function (callable without a GPU). */
spmv_status spmv_select(const spmv_features* f, const spmv_device_props* d, int rowptr_bytes,
                        const spmv_options* opt, spmv_selection* out);

/* Properties of device `dev` used by the selection (needs a GPU). */
spmv_status spmv_device_query(int dev, spmv_device_props* out);

/* ---- errors --------------------------------------------------------------- */
spmv_status spmv_last_status(void);
const char* spmv_last_error(void);

/* Kernels launched by this library since load (all shards, all calls). */
int64_t spmv_kernel_launches(void);

/* ABI self-description (no GPU needed): out[0..5] = sizeof spmv_options, spmv_features,
 * spmv_device_props, spmv_selection, spmv_plan_info, spmv_table1; returns the count written
 * (min(n, 6)). Bindings compare their struct layouts against it. */
int spmv_abi_sizes(int64_t* out, int n);

#ifdef __cplusplus
}
#endif
#endif /* SPMV_H_ */
