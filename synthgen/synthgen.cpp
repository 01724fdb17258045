// synthgen.cpp -- seeded synthetic CSR inputs for the five BASELINE.json configs.
//
// This module generates INPUTS only. It holds none of the SpMV method's
// arithmetic (no products, sums, partitions, encodings or features), so both
// the oracle (oracle/) and the CUDA product path may consume its output.
//
// RNG: SplitMix64 in counter mode:
//   r(s,k)  = mix(s + (k+1)*0x9E3779B97F4A7C15)
//   U01     = (r >> 11) * 2^-53  in [0,1)
//   uniform integer in [0,m) = floor(r * m / 2^64)   (128-bit multiply-high)
// Random access by counter makes every array independent of thread count.
//
// Value modes (vals / x):
//   0 = constant (stencil diag / off-diagonal)   1 = U[-1,1] = 2*U01-1
//   2 = dyadic k/1024, k uniform in [-1024,1024]  3 = U(0,1] = 1-U01
//
// Stream keys:
//   row-wise column draws : k = (row << 24) | t
//   R-MAT edge e, level l : k = e*32 + l
//   value of nonzero j    : seed = value seed, k = j
//   x_i                   : seed = x seed,     k = i
#include <cstdint>
#include <cstring>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <omp.h>

namespace {

inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
inline uint64_t rng(uint64_t s, uint64_t k) { return mix64(s + (k + 1) * 0x9E3779B97F4A7C15ULL); }
inline double u01(uint64_t s, uint64_t k) { return (double)(rng(s, k) >> 11) * 0x1.0p-53; }
inline uint64_t below(uint64_t s, uint64_t k, uint64_t m) {
  return (uint64_t)(((unsigned __int128)rng(s, k) * m) >> 64);
}

inline double draw_value(int mode, uint64_t seed, uint64_t k, double cst) {
  switch (mode) {
    case 0: return cst;
    case 1: return 2.0 * u01(seed, k) - 1.0;
    case 2: return (double)((int64_t)below(seed, k, 2049) - 1024) / 1024.0;
    case 3: return 1.0 - u01(seed, k);
    default: return 0.0;
  }
}

inline void put_rp(void* rp, int rp_bytes, int64_t i, int64_t v) {
  if (rp_bytes == 8) ((int64_t*)rp)[i] = v; else ((int32_t*)rp)[i] = (int32_t)v;
}

// parallel exclusive prefix of lens[0..m) into rp[0..m] (rp[0] = 0)
void prefix_rowptr(const std::vector<int64_t>& lens, void* rp, int rp_bytes) {
  const int64_t m = (int64_t)lens.size();
  int nt = omp_get_max_threads();
  std::vector<int64_t> part(nt + 1, 0);
#pragma omp parallel num_threads(nt)
  {
    int t = omp_get_thread_num();
    int64_t lo = m * t / nt, hi = m * (t + 1) / nt, s = 0;
    for (int64_t i = lo; i < hi; ++i) s += lens[i];
    part[t + 1] = s;
#pragma omp barrier
#pragma omp single
    for (int q = 0; q < nt; ++q) part[q + 1] += part[q];
    int64_t acc = part[t];
    for (int64_t i = lo; i < hi; ++i) { put_rp(rp, rp_bytes, i, acc); acc += lens[i]; }
    if (t == nt - 1) put_rp(rp, rp_bytes, m, acc);
  }
}

// ---- stencils ---------------------------------------------------------------
// idx = (z*n + y)*n + x, x fastest; Dirichlet: out-of-grid neighbours dropped.
inline int axis_lo(int64_t c) { return c > 0 ? -1 : 0; }
inline int axis_hi(int64_t c, int64_t n) { return c < n - 1 ? 1 : 0; }

inline int64_t stencil_row_len(int64_t i, int64_t n, int pts) {
  int64_t x = i % n, y = (i / n) % n, z = i / (n * n);
  if (pts == 7) {
    return 1 + (x > 0) + (x < n - 1) + (y > 0) + (y < n - 1) + (z > 0) + (z < n - 1);
  }
  int64_t cx = 1 + (x > 0) + (x < n - 1), cy = 1 + (y > 0) + (y < n - 1), cz = 1 + (z > 0) + (z < n - 1);
  return cx * cy * cz;
}

}  // namespace

extern "C" {

uint64_t sg_rng(uint64_t s, uint64_t k) { return rng(s, k); }
double sg_u01(uint64_t s, uint64_t k) { return u01(s, k); }
uint64_t sg_below(uint64_t s, uint64_t k, uint64_t m) { return below(s, k, m); }

int sg_num_threads(void) { return omp_get_max_threads(); }

// Fill a dense vector v[i] = draw(mode, seed, i0 + i), i in [0, m).
void sg_vector(int64_t m, int64_t i0, uint64_t seed, int mode, double cst, double* out) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < m; ++i) out[i] = draw_value(mode, seed, (uint64_t)(i0 + i), cst);
}

int64_t sg_stencil_nnz_range(int64_t n, int pts, int64_t rb, int64_t re) {
  int64_t s = 0;
#pragma omp parallel for reduction(+ : s) schedule(static)
  for (int64_t i = rb; i < re; ++i) s += stencil_row_len(i, n, pts);
  return s;
}

// Rows [rb, re) of the pts-point stencil on an n^3 grid. rowptr has re-rb+1
// entries rebased to 0; colind/vals hold that range's nonzeros (sorted cols).
// val_mode 0 uses (diag, off); other modes draw per nonzero with key = global
// nonzero index (base = global rowptr[rb], supplied by the caller as nz0).
void sg_stencil_fill(int64_t n, int pts, double diag, double off, int val_mode, uint64_t val_seed,
                     int64_t rb, int64_t re, int64_t nz0, void* rowptr, int rp_bytes,
                     int32_t* colind, double* vals) {
  const int64_t m = re - rb;
  std::vector<int64_t> lens(m);
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < m; ++r) lens[r] = stencil_row_len(rb + r, n, pts);
  prefix_rowptr(lens, rowptr, rp_bytes);
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < m; ++r) {
    const int64_t i = rb + r;
    int64_t j = (rp_bytes == 8) ? ((int64_t*)rowptr)[r] : ((int32_t*)rowptr)[r];
    const int64_t x = i % n, y = (i / n) % n, z = i / (n * n);
    for (int dz = -1; dz <= 1; ++dz)
      for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx) {
          if (pts == 7 && (dx != 0) + (dy != 0) + (dz != 0) > 1) continue;
          if (dz < axis_lo(z) || dz > axis_hi(z, n)) continue;
          if (dy < axis_lo(y) || dy > axis_hi(y, n)) continue;
          if (dx < axis_lo(x) || dx > axis_hi(x, n)) continue;
          const int64_t c = ((z + dz) * n + (y + dy)) * n + (x + dx);
          colind[j] = (int32_t)c;
          const bool d = (dx == 0 && dy == 0 && dz == 0);
          vals[j] = val_mode == 0 ? (d ? diag : off) : draw_value(val_mode, val_seed, (uint64_t)(nz0 + j), 0.0);
          ++j;
        }
  }
}

// rowptr only, rows [rb, re), rebased to 0 (cheap: closed-form lengths).
void sg_stencil_rowptr(int64_t n, int pts, int64_t rb, int64_t re, void* rowptr, int rp_bytes) {
  const int64_t m = re - rb;
  std::vector<int64_t> lens(m);
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < m; ++r) lens[r] = stencil_row_len(rb + r, n, pts);
  prefix_rowptr(lens, rowptr, rp_bytes);
}

// Distinct sorted rows: `count` rows of [0,n) by rejection, stream (seed, t).
void sg_pick_rows(int64_t n, int64_t count, uint64_t seed, int64_t* out) {
  std::vector<int64_t> got;
  got.reserve(count);
  std::vector<char> seen(n, 0);
  for (uint64_t t = 0; (int64_t)got.size() < count; ++t) {
    int64_t r = (int64_t)below(seed, t, (uint64_t)n);
    if (!seen[r]) { seen[r] = 1; got.push_back(r); }
  }
  std::sort(got.begin(), got.end());
  std::memcpy(out, got.data(), sizeof(int64_t) * count);
}

// Random-row matrix (C1, C4). Row i has `diag` (0/1) diagonal entry plus
// k_short (or k_long when i is in `long_rows`) distinct uniform columns drawn
// from [0,n) (excluding i when diag=1) by rejection on stream key (i<<24)|t;
// columns sorted. Values per nonzero: draw(val_mode, val_seed, j).
int64_t sg_randrows_nnz(int64_t n, int diag, int64_t k_short, int64_t n_long, int64_t k_long) {
  return n * (k_short + diag) + n_long * (k_long - k_short);
}

void sg_randrows_fill(int64_t n, int diag, int64_t k_short, const int64_t* long_rows, int64_t n_long,
                      int64_t k_long, uint64_t col_seed, int val_mode, uint64_t val_seed,
                      void* rowptr, int rp_bytes, int32_t* colind, double* vals) {
  std::vector<int64_t> lens(n, k_short + diag);
  std::vector<char> is_long(n, 0);
  for (int64_t q = 0; q < n_long; ++q) { lens[long_rows[q]] = k_long + diag; is_long[long_rows[q]] = 1; }
  prefix_rowptr(lens, rowptr, rp_bytes);
#pragma omp parallel
  {
    std::vector<uint64_t> bitmap;  // for long rows
    std::vector<int32_t> cols;
#pragma omp for schedule(dynamic, 256)
    for (int64_t i = 0; i < n; ++i) {
      const int64_t k = is_long[i] ? k_long : k_short;
      int64_t j0 = (rp_bytes == 8) ? ((int64_t*)rowptr)[i] : ((int32_t*)rowptr)[i];
      cols.clear();
      if (diag) cols.push_back((int32_t)i);
      const uint64_t kbase = (uint64_t)i << 24;
      if (k > 64) {
        bitmap.assign((n + 63) / 64, 0);
        if (diag) bitmap[i >> 6] |= 1ULL << (i & 63);
        int64_t have = 0;
        for (uint64_t t = 0; have < k; ++t) {
          int64_t c = (int64_t)below(col_seed, kbase | t, (uint64_t)n);
          uint64_t bit = 1ULL << (c & 63);
          if (bitmap[c >> 6] & bit) continue;
          bitmap[c >> 6] |= bit;
          ++have;
        }
        for (int64_t w = 0; w < (int64_t)bitmap.size(); ++w) {
          uint64_t b = bitmap[w];
          while (b) { int s = __builtin_ctzll(b); cols.push_back((int32_t)(w * 64 + s)); b &= b - 1; }
        }
      } else {
        int64_t have = 0;
        for (uint64_t t = 0; have < k; ++t) {
          int32_t c = (int32_t)below(col_seed, kbase | t, (uint64_t)n);
          if (std::find(cols.begin(), cols.end(), c) != cols.end()) continue;
          cols.push_back(c);
          ++have;
        }
        std::sort(cols.begin(), cols.end());
      }
      for (size_t q = 0; q < cols.size(); ++q) {
        colind[j0 + q] = cols[q];
        vals[j0 + q] = draw_value(val_mode, val_seed, (uint64_t)(j0 + q), 0.0);
      }
    }
  }
}

// ---- R-MAT --------------------------------------------------------------------
struct Rmat { int64_t n; std::vector<int64_t> rp; std::vector<int32_t> col; };

// scale s, ef*2^s edge draws, s levels each, quadrant probabilities (a,b,c,d):
// a=(row bit 0, col bit 0), b=(0,1), c=(1,0), d=(1,1), MSB first. Rows are
// sources. Duplicates merged, self-loops kept, no permutation.
void* sg_rmat_make(int scale, int64_t edge_factor, double a, double b, double c, uint64_t seed) {
  Rmat* R = new Rmat;
  const int64_t n = (int64_t)1 << scale, E = edge_factor * n;
  R->n = n;
  std::vector<uint32_t> src(E), dst(E);
  const double ab = a + b, abc = a + b + c;
#pragma omp parallel for schedule(static)
  for (int64_t e = 0; e < E; ++e) {
    uint32_t r = 0, q = 0;
    for (int l = 0; l < scale; ++l) {
      double u = u01(seed, (uint64_t)e * 32 + l);
      uint32_t rb = 0, cb = 0;
      if (u < a) {} else if (u < ab) { cb = 1; } else if (u < abc) { rb = 1; } else { rb = 1; cb = 1; }
      r |= rb << (scale - 1 - l);
      q |= cb << (scale - 1 - l);
    }
    src[e] = r; dst[e] = q;
  }
  // counting sort by row (order inside a row fixed afterwards by sort+unique)
  std::vector<int64_t> cnt(n + 1, 0);
  for (int64_t e = 0; e < E; ++e) cnt[src[e] + 1]++;
  for (int64_t i = 0; i < n; ++i) cnt[i + 1] += cnt[i];
  std::vector<int32_t> tmp(E);
  {
    std::vector<int64_t> pos(cnt.begin(), cnt.end() - 1);
    for (int64_t e = 0; e < E; ++e) tmp[pos[src[e]]++] = (int32_t)dst[e];
  }
  std::vector<int64_t> lens(n);
#pragma omp parallel for schedule(dynamic, 1024)
  for (int64_t i = 0; i < n; ++i) {
    int32_t* b0 = tmp.data() + cnt[i];
    int32_t* b1 = tmp.data() + cnt[i + 1];
    std::sort(b0, b1);
    lens[i] = std::unique(b0, b1) - b0;
  }
  R->rp.assign(n + 1, 0);
  for (int64_t i = 0; i < n; ++i) R->rp[i + 1] = R->rp[i] + lens[i];
  R->col.resize(R->rp[n]);
#pragma omp parallel for schedule(dynamic, 1024)
  for (int64_t i = 0; i < n; ++i)
    std::memcpy(R->col.data() + R->rp[i], tmp.data() + cnt[i], sizeof(int32_t) * lens[i]);
  return R;
}
int64_t sg_rmat_n(void* h) { return ((Rmat*)h)->n; }
int64_t sg_rmat_nnz(void* h) { return ((Rmat*)h)->rp.back(); }
void sg_rmat_fill(void* h, int val_mode, uint64_t val_seed, void* rowptr, int rp_bytes,
                  int32_t* colind, double* vals) {
  Rmat* R = (Rmat*)h;
  const int64_t n = R->n, nnz = R->rp[n];
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i <= n; ++i) put_rp(rowptr, rp_bytes, i, R->rp[i]);
#pragma omp parallel for schedule(static)
  for (int64_t j = 0; j < nnz; ++j) {
    colind[j] = R->col[j];
    vals[j] = draw_value(val_mode, val_seed, (uint64_t)j, 0.0);
  }
}
void sg_rmat_free(void* h) { delete (Rmat*)h; }

// Chunked FNV-1a64 checksum: FNV-1a over each 1 MiB chunk in parallel, then
// FNV-1a over the sequence of chunk hashes (thread-count independent).
uint64_t sg_checksum(const void* p, int64_t bytes) {
  const uint64_t P = 0x100000001B3ULL, O = 0xCBF29CE484222325ULL;
  const int64_t CH = 1 << 20, nch = (bytes + CH - 1) / CH;
  std::vector<uint64_t> hs(nch);
  const unsigned char* s = (const unsigned char*)p;
#pragma omp parallel for schedule(static)
  for (int64_t q = 0; q < nch; ++q) {
    uint64_t h = O;
    const int64_t lo = q * CH, hi = std::min(bytes, lo + CH);
    for (int64_t t = lo; t < hi; ++t) { h ^= s[t]; h *= P; }
    hs[q] = h;
  }
  uint64_t h = O;
  for (int64_t q = 0; q < nch; ++q)
    for (int bsh = 0; bsh < 64; bsh += 8) { h ^= (hs[q] >> bsh) & 0xFF; h *= P; }
  return h;
}

}  // extern "C"
