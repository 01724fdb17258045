/* oracle.c -- plain, slow, obviously-correct CPU oracle for the SpMV hot path.
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * The CUDA product path (paper_1711_05487_b200/) never includes, links or
 * calls anything here, and this file includes nothing from it.
 *
 * Build: gcc -O2 -ffp-contract=off -fno-fast-math -fopenmp (no FMA, IEEE fp64).
 *
 * Citations: P:n = /root/reference/PAPER.md line n, S:n = SPEC.md line n,
 * SURVEY 8(c) = /root/repo/SURVEY.md section 8(c) (the readings this build
 * takes where the paper is silent; repeated in DESIGN.md "Readings").
 *
 * rowptr is always int64 here (the Python wrapper widens int32 rowptr);
 * colind int32; values, x, y fp64. Parity status of every function is in
 * oracle/__init__.py and DESIGN.md (all are pinned; none "parity unpinned").
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

/* ---------------------------------------------------------------------------
 * SpMV, Fig. 2 (Sec. II) read as accumulation (SURVEY 8(c3) #1,
 * SPEC S:190-198): for each row i, acc = +0.0; for j in increasing
 * order acc = acc + val[j]*x[colind[j]] (separately rounded, no FMA);
 * y[i] = acc. y is overwritten; an empty row gives exactly 0.0.
 * ------------------------------------------------------------------------- */
static double row_dot(const int64_t* rowptr, const int32_t* colind, const double* val,
                      const double* x, int64_t i) {
  double acc = 0.0;
  for (int64_t j = rowptr[i]; j < rowptr[i + 1]; ++j) {
    double p = val[j] * x[colind[j]];
    acc = acc + p;
  }
  return acc;
}

void oracle_spmv(int64_t n, const int64_t* rowptr, const int32_t* colind, const double* val,
                 const double* x, double* y) {
  for (int64_t i = 0; i < n; ++i) y[i] = row_dot(rowptr, colind, val, x, i);
}

/* Sampled rows: out[q] = y[rows[q]] computed one by one with the same loop. */
void oracle_spmv_rows(const int64_t* rowptr, const int32_t* colind, const double* val,
                      const double* x, const int64_t* rows, int64_t m, double* out) {
  for (int64_t q = 0; q < m; ++q) out[q] = row_dot(rowptr, colind, val, x, rows[q]);
}

/* Per-row bound denominator of BJ.north_star: s_i = sum_j |a_ij * x_j|. */
void oracle_absrow_rows(const int64_t* rowptr, const int32_t* colind, const double* val,
                        const double* x, const int64_t* rows, int64_t m, double* out) {
  for (int64_t q = 0; q < m; ++q) {
    int64_t i = rows ? rows[q] : q;
    double acc = 0.0;
    for (int64_t j = rowptr[i]; j < rowptr[i + 1]; ++j) acc = acc + fabs(val[j] * x[colind[j]]);
    out[q] = acc;
  }
}

/* Neumaier-compensated row sums: the oracle self-check of SURVEY 8(c3) #3. */
void oracle_spmv_neumaier(int64_t n, const int64_t* rowptr, const int32_t* colind,
                          const double* val, const double* x, double* y) {
  for (int64_t i = 0; i < n; ++i) {
    double s = 0.0, c = 0.0;
    for (int64_t j = rowptr[i]; j < rowptr[i + 1]; ++j) {
      double p = val[j] * x[colind[j]];
      double t = s + p;
      if (fabs(s) >= fabs(p)) c = c + ((s - t) + p); else c = c + ((p - t) + s);
      s = t;
    }
    y[i] = s + c;
  }
}

/* ---------------------------------------------------------------------------
 * nnz-balanced contiguous row partition, Sec. IV-A "each partition
 * has approximately equal number of nonzero elements"; reading SURVEY 8(c2):
 * b_0 = 0, b_G = n, b_g = min{ r in [0,n] : rowptr[r] >= ceil(g*nnz/G) }.
 * Reproduces SPEC's examples S:254-255.
 * ------------------------------------------------------------------------- */
static int64_t lower_bound_rp(const int64_t* rowptr, int64_t lo, int64_t hi, int64_t key) {
  /* smallest r in [lo,hi] with rowptr[r] >= key, or hi+1 if none */
  int64_t a = lo, b = hi + 1;
  while (a < b) {
    int64_t mid = a + (b - a) / 2;
    if (rowptr[mid] < key) a = mid + 1; else b = mid;
  }
  return a;
}

void oracle_shard_bounds(int64_t n, const int64_t* rowptr, int64_t nnz, int64_t G, int64_t* b) {
  b[0] = 0;
  for (int64_t g = 1; g < G; ++g) {
    int64_t key = (g * nnz + G - 1) / G; /* ceil(g*nnz/G) */
    int64_t r = lower_bound_rp(rowptr, 0, n, key);
    b[g] = r > n ? n : r;
  }
  b[G] = n;
}

/* Row-parallel OpenMP form of oracle_spmv for the CPU baseline timing: the
 * paper's baseline (static 1-D nnz-balanced row partition). Each
 * row is still summed sequentially by one thread, so y is bitwise identical
 * to oracle_spmv. Returns the thread count used. */
#include <omp.h>
int oracle_spmv_omp(int64_t n, const int64_t* rowptr, const int32_t* colind, const double* val,
                    const double* x, double* y, int nthreads) {
  if (nthreads <= 0) nthreads = omp_get_max_threads();
  int64_t* b = (int64_t*)malloc(sizeof(int64_t) * (nthreads + 1));
  oracle_shard_bounds(n, rowptr, rowptr[n], nthreads, b);
#pragma omp parallel num_threads(nthreads)
  {
    int t = omp_get_thread_num();
    for (int64_t i = b[t]; i < b[t + 1]; ++i) y[i] = row_dot(rowptr, colind, val, x, i);
  }
  free(b);
  return nthreads;
}

/* ---------------------------------------------------------------------------
 * Iterated mode (BJ.configs[5]): x_0 given; for k = 0..K-1:
 * y = A x_k; nu_k = sqrt(sum_{i ascending} y_i^2); x_{k+1} = y / nu_k.
 * Output x_K and nu_0..nu_{K-1}. Returns 0, or -7 (zero norm) at the failing k.
 * nthreads > 1 only parallelises the row loop (bitwise identical).
 * ------------------------------------------------------------------------- */
int oracle_power_iter(int64_t n, const int64_t* rowptr, const int32_t* colind, const double* val,
                      const double* x0, int K, double* x_out, double* nu_out, int nthreads) {
  double* xa = (double*)malloc(sizeof(double) * (size_t)n);
  double* ya = (double*)malloc(sizeof(double) * (size_t)n);
  memcpy(xa, x0, sizeof(double) * (size_t)n);
  int rc = 0;
  for (int k = 0; k < K; ++k) {
    if (nthreads > 1) oracle_spmv_omp(n, rowptr, colind, val, xa, ya, nthreads);
    else oracle_spmv(n, rowptr, colind, val, xa, ya);
    double ss = 0.0;
    for (int64_t i = 0; i < n; ++i) ss = ss + ya[i] * ya[i];
    double nu = sqrt(ss);
    nu_out[k] = nu;
    if (nu == 0.0) { rc = -7; break; }
    for (int64_t i = 0; i < n; ++i) xa[i] = ya[i] / nu;
  }
  memcpy(x_out, xa, sizeof(double) * (size_t)n);
  free(xa); free(ya);
  return rc;
}

/* ---------------------------------------------------------------------------
 * CSR validation (S:32-35 invariants, "first violated invariant and
 * its location"). Order of checks: rowptr[0]==0 (code 1, at 0); rowptr[n]==nnz
 * (code 2, at n); nondecreasing (code 3, smallest i with rowptr[i+1]<rowptr[i]);
 * then over nonzeros j ascending: 0 <= colind[j] < n (code 4) else, if j is
 * not a row head, colind[j] > colind[j-1] (code 5). Returns code, *where.
 * ------------------------------------------------------------------------- */
int oracle_validate(int64_t n, int64_t nnz, const int64_t* rowptr, const int32_t* colind,
                    int64_t* where) {
  *where = -1;
  if (rowptr[0] != 0) { *where = 0; return 1; }
  if (rowptr[n] != nnz) { *where = n; return 2; }
  for (int64_t i = 0; i < n; ++i)
    if (rowptr[i + 1] < rowptr[i]) { *where = i; return 3; }
  for (int64_t i = 0; i < n; ++i) {
    for (int64_t j = rowptr[i]; j < rowptr[i + 1]; ++j) {
      if (colind[j] < 0 || (int64_t)colind[j] >= n) { *where = j; return 4; }
      if (j > rowptr[i] && colind[j] <= colind[j - 1]) { *where = j; return 5; }
    }
  }
  return 0;
}

/* ---------------------------------------------------------------------------
 * Theta(N) features of Table I plus the counts the selection needs
 * (SURVEY 8(a) a2, 8(c2)). Integers exact; nnz_sd = sqrt((double)(N*S2-S1^2))/N
 * with the difference formed exactly in 128-bit (population sd, Table I).
 * "short" rows are those with len <= L_split (empty rows included).
 * maxgap = max over non-head j of colind[j]-colind[j-1] (0 if none);
 * misses = #non-head j with gap > line_elems (Table I misses_i, P:533-537,
 * reading SURVEY 8(c3) #15: 128-B line = 16 doubles).
 * ------------------------------------------------------------------------- */
typedef struct {
  int64_t n, nnz, nnz_min, nnz_max, n_empty, n_long, nnz_long, n_short, max_short;
  uint64_t s1, s2, s1_short, s2_short;
  int64_t maxgap, misses;
  double nnz_avg, nnz_sd, avg_short, sd_short;
} oracle_features_t;

static double pop_sd(uint64_t cnt, uint64_t s1, uint64_t s2) {
  if (cnt == 0) return 0.0;
  unsigned __int128 a = (unsigned __int128)cnt * s2, b = (unsigned __int128)s1 * s1;
  return sqrt((double)(a - b)) / (double)cnt;
}

void oracle_features(int64_t n, const int64_t* rowptr, const int32_t* colind, int64_t L_split,
                     int64_t line_elems, oracle_features_t* f) {
  memset(f, 0, sizeof(*f));
  f->n = n; f->nnz = rowptr[n];
  f->nnz_min = n > 0 ? INT64_MAX : 0;
  for (int64_t i = 0; i < n; ++i) {
    int64_t len = rowptr[i + 1] - rowptr[i];
    if (len < f->nnz_min) f->nnz_min = len;
    if (len > f->nnz_max) f->nnz_max = len;
    f->s1 += (uint64_t)len; f->s2 += (uint64_t)len * (uint64_t)len;
    if (len == 0) f->n_empty++;
    if (len > L_split) { f->n_long++; f->nnz_long += len; }
    else {
      f->n_short++; f->s1_short += (uint64_t)len; f->s2_short += (uint64_t)len * (uint64_t)len;
      if (len > f->max_short) f->max_short = len;
    }
    for (int64_t j = rowptr[i] + 1; j < rowptr[i + 1]; ++j) {
      int64_t g = (int64_t)colind[j] - (int64_t)colind[j - 1];
      if (g > f->maxgap) f->maxgap = g;
      if (g > line_elems) f->misses++;
    }
  }
  f->nnz_avg = n ? (double)f->s1 / (double)n : 0.0;
  f->nnz_sd = pop_sd((uint64_t)n, f->s1, f->s2);
  f->avg_short = f->n_short ? (double)f->s1_short / (double)f->n_short : 0.0;
  f->sd_short = pop_sd((uint64_t)f->n_short, f->s1_short, f->s2_short);
}

/* ---------------------------------------------------------------------------
 * Per-CTA nnz tiles: tile k covers nonzeros
 * [k*C, min((k+1)*C, nnz)); T = max(1, ceil(nnz/C)). It OWNS rows
 * [R_k, R_{k+1}) with R_k = min{ r in [0,n] : rowptr[r] >= k*C } for
 * 0 < k < T, R_0 = 0, R_T = n (the lower_bound rule of the partition above,
 * applied at stride C instead of nnz/G).
 * ------------------------------------------------------------------------- */
void oracle_tile_rows(int64_t n, const int64_t* rowptr, int64_t C, int64_t T, int64_t* R) {
  R[0] = 0;
  for (int64_t k = 1; k < T; ++k) {
    int64_t r = lower_bound_rp(rowptr, 0, n, k * C);
    R[k] = r > n ? n : r;
  }
  R[T] = n;
}

/* ---------------------------------------------------------------------------
 * nnz_split structures (reading 19; the nnz-balanced partition of
 * P:708-711 cut at warp granularity, long rows shared by consecutive pieces
 * as in the decomposition P:608-621). Written as plain sequential scans.
 *   rows with rowptr[i+1] > rowptr[i], in increasing i: rowmap[q] = i,
 *   rpc[q] = rowptr[i]; rowmap[mc] = n, rpc[mc] = nnz. Returns mc.
 *   tile_q[k] = the largest q with rpc[q] <= k*W (k < T), tile_q[T] = mc.
 * ------------------------------------------------------------------------- */
int64_t oracle_nonempty_rows(int64_t n, const int64_t* rowptr, int64_t* rowmap, int64_t* rpc) {
  int64_t q = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (rowptr[i + 1] > rowptr[i]) {
      if (rowmap) rowmap[q] = i;
      if (rpc) rpc[q] = rowptr[i];
      ++q;
    }
  }
  if (rowmap) rowmap[q] = n;
  if (rpc) rpc[q] = rowptr[n];
  return q;
}

void oracle_nz_tiles(int64_t mc, const int64_t* rpc, int64_t W, int64_t T, int64_t* tile_q) {
  int64_t q = 0;
  for (int64_t k = 0; k < T; ++k) {
    while (q + 1 <= mc && rpc[q + 1] <= k * W) ++q;
    tile_q[k] = q;
  }
  tile_q[T] = mc;
}

/* ---------------------------------------------------------------------------
 * Merge-path split (the GPU analogue of the IMB "auto" schedule,
 * P:621-627): merge list A[i] = rowptr[i+1] (i < n) with list B[j] = j
 * (j < nnz); ties go to A. split(d) = (i, d-i) with i the number of A items
 * among the first d merged items. Written here as the sequential merge itself
 * (no binary search), so it is checkable by eye.
 * ------------------------------------------------------------------------- */
void oracle_merge_splits(int64_t n, const int64_t* rowptr, int64_t nnz, int64_t items, int64_t T,
                         int64_t* si, int64_t* sj) {
  /* diagonals d_k = min(k*items, n+nnz), k = 0..T */
  int64_t i = 0, j = 0, d = 0;
  for (int64_t k = 0; k <= T; ++k) {
    int64_t target = k * items; if (target > n + nnz) target = n + nnz;
    while (d < target) {
      if (i < n && (j >= nnz || rowptr[i + 1] <= j)) ++i; else ++j;
      ++d;
    }
    si[k] = i; sj[k] = j;
  }
}

/* ---------------------------------------------------------------------------
 * Long-row chunk table (P:608-621 decomposition; reading SURVEY 8(c2)): for
 * each row with len > L_split in increasing row order, chunks
 * [rowptr[i] + c*C, min(rowptr[i] + (c+1)*C, rowptr[i+1])). Returns the chunk
 * count; fills the arrays when non-NULL.
 * ------------------------------------------------------------------------- */
int64_t oracle_long_chunks(int64_t n, const int64_t* rowptr, int64_t L_split, int64_t C,
                           int64_t* crow, int64_t* cbeg, int64_t* cend) {
  int64_t q = 0;
  for (int64_t i = 0; i < n; ++i) {
    int64_t len = rowptr[i + 1] - rowptr[i];
    if (len <= L_split) continue;
    for (int64_t s = rowptr[i]; s < rowptr[i + 1]; s += C) {
      if (crow) {
        crow[q] = i; cbeg[q] = s;
        cend[q] = s + C < rowptr[i + 1] ? s + C : rowptr[i + 1];
      }
      ++q;
    }
  }
  return q;
}

/* ---------------------------------------------------------------------------
 * Delta-indexed colind (MB class; Table II). Reading SURVEY
 * 8(c2)/(c3) #7-8: width matrix-global, 8 iff maxgap <= 255, 16 iff <= 65535,
 * else 0 (not compressible). dcol[j] = colind[j]-colind[j-1] for
 * non-head j, 0 at row heads (index-aligned with values); head[i] =
 * colind[rowptr[i]] or n for an empty row. Per nnz tile of size C
 * (the tiling above), anchor[k] = colind[k*C] gives the absolute column at
 * each tile start. dcol is written as uint16 regardless of width (width 8
 * values fit). Returns the width.
 * ------------------------------------------------------------------------- */
int oracle_d16_encode(int64_t n, const int64_t* rowptr, const int32_t* colind, uint16_t* dcol,
                      int32_t* head, int64_t* maxgap_out) {
  int64_t maxgap = 0;
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = rowptr[i] + 1; j < rowptr[i + 1]; ++j) {
      int64_t g = (int64_t)colind[j] - (int64_t)colind[j - 1];
      if (g > maxgap) maxgap = g;
    }
  *maxgap_out = maxgap;
  int width = maxgap <= 255 ? 8 : (maxgap <= 65535 ? 16 : 0);
  if (width == 0) return 0;
  for (int64_t i = 0; i < n; ++i) {
    head[i] = rowptr[i + 1] > rowptr[i] ? colind[rowptr[i]] : (int32_t)n;
    for (int64_t j = rowptr[i]; j < rowptr[i + 1]; ++j)
      dcol[j] = j == rowptr[i] ? 0 : (uint16_t)(colind[j] - colind[j - 1]);
  }
  return width;
}

/* Escape-coded 16-bit deltas (reading 21): when
 * the largest gap exceeds 65535 but at most 64 DISTINCT gaps are >= 65472,
 * a gap d < 65472 is stored as d and a gap d >= 65472 as 65472 + (index of d
 * in the ascending table esc[] of those distinct gaps). Returns 16 and the
 * table size in *n_esc (esc needs 64 entries), or 0 when not encodable.
 * Plain widths (8 / 16 without escapes) follow oracle_d16_encode. */
int oracle_d16_encode_esc(int64_t n, const int64_t* rowptr, const int32_t* colind, uint16_t* dcol,
                          int32_t* head, int64_t* maxgap_out, int32_t* esc, int* n_esc) {
  int w = oracle_d16_encode(n, rowptr, colind, dcol, head, maxgap_out);
  *n_esc = 0;
  if (w) return w;
  int k = 0;
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = rowptr[i] + 1; j < rowptr[i + 1]; ++j) {
      int64_t g = (int64_t)colind[j] - (int64_t)colind[j - 1];
      if (g < 65472) continue;
      int found = 0;
      for (int t = 0; t < k; ++t) if (esc[t] == g) { found = 1; break; }
      if (found) continue;
      if (k == 64) return 0;
      esc[k++] = (int32_t)g;
    }
  /* ascending (insertion sort, at most 64 entries) */
  for (int a = 1; a < k; ++a)
    for (int b = a; b > 0 && esc[b - 1] > esc[b]; --b) { int32_t t = esc[b]; esc[b] = esc[b - 1]; esc[b - 1] = t; }
  for (int64_t i = 0; i < n; ++i) {
    head[i] = rowptr[i + 1] > rowptr[i] ? colind[rowptr[i]] : (int32_t)n;
    for (int64_t j = rowptr[i]; j < rowptr[i + 1]; ++j) {
      int64_t g = j == rowptr[i] ? 0 : (int64_t)colind[j] - (int64_t)colind[j - 1];
      if (g >= 65472) {
        int t = 0;
        while (esc[t] != g) ++t;
        g = 65472 + t;
      }
      dcol[j] = (uint16_t)g;
    }
  }
  *n_esc = k;
  return 16;
}

/* escape-aware decode: delta = code < 65472 ? code : esc[code - 65472] */
void oracle_d16_decode_esc(int64_t n, const int64_t* rowptr, const uint16_t* dcol, const int32_t* head,
                           const int32_t* esc, int32_t* col_out) {
  for (int64_t i = 0; i < n; ++i) {
    int64_t c = head[i];
    for (int64_t j = rowptr[i]; j < rowptr[i + 1]; ++j) {
      if (j > rowptr[i]) c += dcol[j] < 65472 ? (int64_t)dcol[j] : (int64_t)esc[dcol[j] - 65472];
      col_out[j] = (int32_t)c;
    }
  }
}

/* decode: col[j] = head[i] + sum_{t=rowptr[i]+1}^{j} dcol[t] */
void oracle_d16_decode(int64_t n, const int64_t* rowptr, const uint16_t* dcol, const int32_t* head,
                       int32_t* col_out) {
  for (int64_t i = 0; i < n; ++i) {
    int64_t c = head[i];
    for (int64_t j = rowptr[i]; j < rowptr[i + 1]; ++j) {
      if (j > rowptr[i]) c += dcol[j];
      col_out[j] = (int32_t)c;
    }
  }
}

void oracle_tile_anchor(const int32_t* colind, int64_t nnz, int64_t C, int64_t T, int32_t* anchor) {
  for (int64_t k = 0; k < T; ++k) anchor[k] = k * C < nnz ? colind[k * C] : 0;
}

/* ---------------------------------------------------------------------------
 * Dictionary-coded 8-bit column deltas ("D8"; the MB-class optimisation of
 * Sec. III-E: "8- or 16-bit deltas wherever possible, but never
 * both"; Table II; reading 26).
 * Row-relative deltas of row i (row id i of the matrix) and its nonzeros
 * j = rowptr[i] .. rowptr[i+1]-1:
 *     delta_j = colind[j] - i               (j = rowptr[i], the row head)
 *     delta_j = colind[j] - colind[j-1]     (j > rowptr[i])
 * dict = the distinct deltas in ascending order. The matrix is D8-codable iff
 * |dict| <= 256 (one byte per code) and every row has <= 255 nonzeros (one
 * byte per row length). code_j = the index of delta_j in dict; rlen[i] =
 * rowptr[i+1] - rowptr[i]. Decode: c = i; c += dict[code_j]; colind[j] = c.
 *
 * oracle_d8_dict: fills dict (>= 256 entries) and returns |dict|, or 257 as
 * soon as a 257th distinct delta appears. Kept as a sorted array with plain
 * insertion (at most 257 entries).
 * ------------------------------------------------------------------------- */
static int d8_find(const int64_t* dict, int nd, int64_t v) {
  int lo = 0, hi = nd; /* first index with dict[idx] >= v */
  while (lo < hi) {
    int mid = (lo + hi) / 2;
    if (dict[mid] < v) lo = mid + 1; else hi = mid;
  }
  return lo;
}

int oracle_d8_dict(int64_t n, const int64_t* rowptr, const int32_t* colind, int64_t* dict) {
  int nd = 0;
  for (int64_t i = 0; i < n; ++i) {
    for (int64_t j = rowptr[i]; j < rowptr[i + 1]; ++j) {
      int64_t d = j == rowptr[i] ? (int64_t)colind[j] - i : (int64_t)colind[j] - (int64_t)colind[j - 1];
      int at = d8_find(dict, nd, d);
      if (at < nd && dict[at] == d) continue;
      if (nd == 256) return 257;
      for (int t = nd; t > at; --t) dict[t] = dict[t - 1];
      dict[at] = d;
      ++nd;
    }
  }
  return nd;
}

/* Encode: returns |dict| (codes and rlen written) or 0 when not D8-codable
 * (|dict| > 256 or a row longer than 255). dict: 256 entries. */
int oracle_d8_encode(int64_t n, const int64_t* rowptr, const int32_t* colind, int64_t* dict, uint8_t* codes,
                     uint8_t* rlen) {
  for (int64_t i = 0; i < n; ++i)
    if (rowptr[i + 1] - rowptr[i] > 255) return 0;
  int nd = oracle_d8_dict(n, rowptr, colind, dict);
  if (nd > 256) return 0;
  for (int64_t i = 0; i < n; ++i) {
    rlen[i] = (uint8_t)(rowptr[i + 1] - rowptr[i]);
    for (int64_t j = rowptr[i]; j < rowptr[i + 1]; ++j) {
      int64_t d = j == rowptr[i] ? (int64_t)colind[j] - i : (int64_t)colind[j] - (int64_t)colind[j - 1];
      codes[j] = (uint8_t)d8_find(dict, nd, d);
    }
  }
  return nd;
}

/* Decode (rowptr from the row lengths: rowptr[i+1] = rowptr[i] + rlen[i]). */
void oracle_d8_decode(int64_t n, const uint8_t* rlen, const uint8_t* codes, const int64_t* dict,
                      int32_t* col_out) {
  int64_t j = 0;
  for (int64_t i = 0; i < n; ++i) {
    int64_t c = i;
    for (int t = 0; t < rlen[i]; ++t, ++j) {
      c += dict[codes[j]];
      col_out[j] = (int32_t)c;
    }
  }
}

/* ---------------------------------------------------------------------------
 * Row-pattern codes (reading 31; the MB answer of Sec. III-E,
 * P:589-597, carried to the P_peak limit of P:341-344 -- indexing eliminated
 * down to one byte per row): the pattern of row i is its length and the
 * column offsets colind[j] - i, j in row i, in order. Patterns are numbered
 * in the order of their first row. Returns the number of patterns and writes
 * ids[n] (the row's pattern), lens[np], ofs[sum of lens] (pattern p's offsets
 * at position sum_{q<p} lens[q]); returns -1 when the matrix is not codable:
 * a row longer than 255, more than maxp patterns, or more than maxofs
 * offsets in total. Each row is compared with the previous row's pattern,
 * then with every pattern in id order.
 * ------------------------------------------------------------------------- */
static int pat_eq(const int64_t* lens, const int64_t* start, const int64_t* ofs, int64_t p, int64_t i,
                  const int64_t* rowptr, const int32_t* colind) {
  const int64_t len = rowptr[i + 1] - rowptr[i];
  if (lens[p] != len) return 0;
  for (int64_t t = 0; t < len; ++t)
    if (ofs[start[p] + t] != (int64_t)colind[rowptr[i] + t] - i) return 0;
  return 1;
}

int64_t oracle_pat_encode(int64_t n, const int64_t* rowptr, const int32_t* colind, int64_t maxp, int64_t maxofs,
                          uint8_t* ids, int64_t* lens, int64_t* ofs) {
  int64_t np = 0, nofs = 0, prev = -1;
  int64_t* start = (int64_t*)malloc(sizeof(int64_t) * (size_t)(maxp > 0 ? maxp : 1));
  if (!start) return -1;
  for (int64_t i = 0; i < n; ++i) {
    const int64_t len = rowptr[i + 1] - rowptr[i];
    if (len > 255) { free(start); return -1; }
    int64_t found = -1;
    if (prev >= 0 && pat_eq(lens, start, ofs, prev, i, rowptr, colind)) found = prev;
    for (int64_t p = 0; found < 0 && p < np; ++p)
      if (pat_eq(lens, start, ofs, p, i, rowptr, colind)) found = p;
    if (found < 0) {
      if (np == maxp || nofs + len > maxofs) { free(start); return -1; }
      start[np] = nofs;
      lens[np] = len;
      for (int64_t t = 0; t < len; ++t) ofs[nofs + t] = (int64_t)colind[rowptr[i] + t] - i;
      nofs += len;
      found = np++;
    }
    ids[i] = (uint8_t)found;
    prev = found;
  }
  free(start);
  return np;
}

/* Decode: colind of row i = i + the offsets of pattern ids[i] (rows in order). */
void oracle_pat_decode(int64_t n, const uint8_t* ids, int64_t np, const int64_t* lens, const int64_t* ofs,
                       int32_t* col_out) {
  int64_t j = 0;
  for (int64_t i = 0; i < n; ++i) {
    int64_t st = 0;
    for (int64_t q = 0; q < ids[i] && q < np; ++q) st += lens[q];
    for (int64_t t = 0; t < lens[ids[i]]; ++t) col_out[j++] = (int32_t)(i + ofs[st + t]);
  }
}
