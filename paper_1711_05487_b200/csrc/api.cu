// api.cu -- the C ABI of include/spmv.h: plan lifecycle (upload, inspector,
// selection, structure build), execution, iterated mode, inspection.
//
// C++ exceptions are used internally and never cross the ABI: every entry
// point catches and converts to a spmv_status + thread-local message.
#include <algorithm>
#include <functional>
#include <atomic>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "spmv.h"
#include "internal.h"

using namespace spmv;

namespace {

thread_local spmv_status g_status = SPMV_OK;
thread_local std::string g_msg;
std::atomic<int64_t> g_launches{0};
// live plans holding a persisting-L2 carve-out per device (the limit is
// device-wide: reset only when the last such plan goes)
std::mutex g_l2_mu;
constexpr int kIterRegions = 3;  // iterated mode: partials of up to 3 launches per shard (interior + 2 boundary)
constexpr size_t kStaticSmemMargin = 2048;  // static shared memory of the stream / D8 kernels (< 2 KB)
int g_l2_plans[64] = {0};

struct Err : std::runtime_error {
  spmv_status st;
  Err(spmv_status s, const std::string& m) : std::runtime_error(m), st(s) {}
};

[[noreturn]] void fail(spmv_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  throw Err(s, buf);
}

void ck(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return;
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    fail(SPMV_E_NOMEM, "%s: %s", what, cudaGetErrorString(e));
  }
  fail(SPMV_E_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

void count_launches(int n, const char* what) {
  g_launches += n;
  ck(cudaGetLastError(), what);
}

spmv_status set_ok() {
  g_status = SPMV_OK;
  return SPMV_OK;
}
spmv_status set_err(spmv_status s, const std::string& m) {
  g_status = s;
  g_msg = m;
  return s;
}

double now_ms() {
  using namespace std::chrono;
  return duration<double, std::milli>(steady_clock::now().time_since_epoch()).count();
}

bool is_device_ptr(const void* p, int* dev) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  if (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged) {
    if (dev) *dev = a.device;
    return true;
  }
  return false;
}

bool is_pageable_host(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return a.type == cudaMemoryTypeUnregistered;
}

// Host -> device copy of a large pageable array: chunks are copied by host
// threads into two pinned staging buffers and DMA'd from there, the next
// chunk's host copy overlapping the previous chunk's DMA (the driver's own
// pageable path stages single-threaded: C5's 18.7 GB took ~4.2 s). Pinned or
// device sources and small arrays go straight to cudaMemcpyAsync.
void upload(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  constexpr size_t kChunk = 64ull << 20;
  if (bytes < 2 * kChunk || !is_pageable_host(src) || getenv("SPMV_NO_STAGED_UPLOAD")) {
    ck(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, s), "upload");
    return;
  }
  void* buf[2] = {nullptr, nullptr};
  cudaEvent_t ev[2] = {nullptr, nullptr};
  auto cleanup = [&] {
    for (int i = 0; i < 2; ++i) {
      if (ev[i]) cudaEventDestroy(ev[i]);
      if (buf[i]) cudaFreeHost(buf[i]);
    }
  };
  try {
    for (int i = 0; i < 2; ++i) {
      ck(cudaHostAlloc(&buf[i], kChunk, cudaHostAllocDefault), "cudaHostAlloc");
      ck(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming), "cudaEventCreate");
    }
    const unsigned nt = std::max(1u, std::min(8u, std::thread::hardware_concurrency()));
    const char* sp = static_cast<const char*>(src);
    char* dp = static_cast<char*>(dst);
    int i = 0;
    for (size_t off = 0; off < bytes; off += kChunk, i ^= 1) {
      const size_t n = std::min(kChunk, bytes - off);
      ck(cudaEventSynchronize(ev[i]), "staging");  // the DMA that last used buf[i] is done
      std::vector<std::thread> th;
      const size_t per = (n + nt - 1) / nt;
      for (unsigned t = 0; t < nt; ++t) {
        const size_t a = t * per, b = std::min(n, a + per);
        if (a < b) th.emplace_back([=] { memcpy(static_cast<char*>(buf[i]) + a, sp + off + a, b - a); });
      }
      for (auto& t : th) t.join();
      ck(cudaMemcpyAsync(dp + off, buf[i], n, cudaMemcpyHostToDevice, s), "upload");
      ck(cudaEventRecord(ev[i], s), "event");
    }
    ck(cudaStreamSynchronize(s), "upload");
    cleanup();
  } catch (...) {
    cleanup();
    throw;
  }
}

int64_t rp_at(const void* rp, int bytes, int64_t i) {
  return bytes == 8 ? ((const int64_t*)rp)[i] : (int64_t)((const int32_t*)rp)[i];
}

}  // namespace

struct Shard {
  int dev = 0;
  cudaStream_t stream = nullptr;
  int64_t row0 = 0, m = 0, n_cols = 0, nnz0 = 0, nnz = 0;
  int rp_bytes = 4;
  void* rowptr = nullptr;
  int32_t* col = nullptr;
  double* val = nullptr;
  double* x = nullptr;
  double* y = nullptr;
  uint32_t* headbits = nullptr;
  DevStats* stats = nullptr;
  DevStats hs{};
  int sm_count = 0;  // the shard device's multiProcessorCount (set at plan creation)
  // STREAM: sp[0] over the whole shard; SPLIT: sp[0] short bin, sp[1] medium bin
  StreamPlan sp[2];
  int n_sp = 0;
  bool zero_y = false;
  // MERGE
  int64_t items = 0, Tm = 0;
  int32_t* mrow = nullptr;
  int64_t* mnnz = nullptr;
  int32_t* mcarry_row = nullptr;
  double* mcarry_val = nullptr;
  // SPLIT long rows
  int64_t n_long = 0, n_chunks = 0;
  int32_t* long_rows = nullptr;
  int64_t* chunk_start = nullptr;
  int32_t* chunk_row = nullptr;
  double* chunk_val = nullptr;
  bool long_tiled = false;
  int64_t nblk = 0;
  int64_t* long_seg = nullptr;
  uint16_t* long_c16 = nullptr;
  double* long_partial = nullptr;
  int long_grid = 0;
  bool split_fused = true;
  bool long_tma = false;
  int long_rg = 0;
  // values copied into other layouts at plan time (SPLIT bins, packed D8
  // tiles): refreshed from val by spmv_plan_update_values
  std::vector<std::function<void(cudaStream_t)>> val_refresh;
  // NNZSPLIT (whole shard) / SPLIT short+medium rows as one nnz_split bin
  NzPlan nz;
  bool use_nz = false;
  // SPLIT: side stream for the long rows (concurrent with the bins)
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // iterated mode
  double* allpart = nullptr;  // [2 parities][G shards][kIterRegions launches][kNormPartials]
  // interior-first iteration: tiles [kb, ke) read only the
  // shard's own x block, the others wait for the halo copies
  bool ovl_ready = false, ovl = false;
  int64_t kb = 0, ke = 0;
  // halo push (IterOut::push_*): the lower / upper neighbour that reads this
  // block's first rows [0, push_lo_end) / last rows [push_hi_begin, m) (local)
  int push_lo_peer = -1, push_hi_peer = -1;
  int64_t push_lo_end = 0, push_hi_begin = 0;
  cudaStream_t cp = nullptr;     // halo copy stream
  cudaEvent_t ev_cp = nullptr;   // halo copies of the current iteration done
  double* x2 = nullptr;       // second x replica (deferred-normalisation ping-pong)
  std::vector<void*> ipc_open;  // peers' replicas mapped by spmv_ipc_open (closed on release)
  double* cta_part = nullptr; // per-CTA sums of y^2 (fused iteration epilogue, row-aligned STREAM / D8)
  unsigned int* done = nullptr;  // its last-CTA ticket counter
  double* cta2 = nullptr;        // [2][grid] per-CTA sums of the prologue-norm iteration (parity double-buffered)
  double* nn = nullptr;       // running norm + rescale factor (norm.cu)
  double* nu = nullptr;
  int nu_cap = 0;
  cudaEvent_t ev_part = nullptr, ev_x = nullptr;
  // pipelined host execute (STREAM plans, host x and y): tile blocks with the
  // x chunk each needs, the first row each block completes, copy streams
  struct HostPipe {
    bool ready = false, usable = false;
    bool nz = false;             // nnz_split pass (else STREAM)
    std::vector<int64_t> kb;     // block b = tiles [kb[b], kb[b+1])
    std::vector<int64_t> srow;   // block b completes rows [srow[b], srow[b+1])
    std::vector<int64_t> xhi;    // x[xlo, xhi[b]) is needed by blocks <= b
    int64_t xlo = 0;             // first column the shard reads
    cudaStream_t h2d = nullptr, d2h = nullptr;
    // optional second copy stream per direction (experiment, off: consecutive
    // chunks alternating streams starve the other direction)
    cudaStream_t h2d2 = nullptr, d2h2 = nullptr;
    cudaEvent_t ev_e2 = nullptr;
    std::vector<cudaEvent_t> ev_h, ev_c;
  } hp;
  std::vector<void*> allocs;
  int64_t bytes = 0;

  template <typename T>
  T* alloc(size_t count, size_t pad_bytes = 64) {
    void* p = nullptr;
    const size_t b = count * sizeof(T) + pad_bytes;
    ck(cudaSetDevice(dev), "cudaSetDevice");
    ck(cudaMalloc(&p, b), "cudaMalloc");
    allocs.push_back(p);
    bytes += (int64_t)b;
    return static_cast<T*>(p);
  }
  void free_alloc(void* p) {  // one allocation of this shard, returned early
    auto it = std::find(allocs.begin(), allocs.end(), p);
    if (it == allocs.end()) return;
    allocs.erase(it);
    cudaFree(p);
  }
  void release() {
    cudaSetDevice(dev);
    if (stream) cudaStreamSynchronize(stream);
    for (void* p : ipc_open) cudaIpcCloseMemHandle(p);
    ipc_open.clear();
    for (void* p : allocs) cudaFree(p);
    allocs.clear();
    if (ev_part) cudaEventDestroy(ev_part);
    if (ev_x) cudaEventDestroy(ev_x);
    if (ev_cp) cudaEventDestroy(ev_cp);
    if (cp) cudaStreamDestroy(cp);
    ev_cp = nullptr;
    cp = nullptr;
    for (cudaEvent_t e : hp.ev_h) cudaEventDestroy(e);
    for (cudaEvent_t e : hp.ev_c) cudaEventDestroy(e);
    hp.ev_h.clear();
    hp.ev_c.clear();
    if (hp.h2d2) cudaStreamDestroy(hp.h2d2);
    if (hp.d2h2) cudaStreamDestroy(hp.d2h2);
    if (hp.ev_e2) cudaEventDestroy(hp.ev_e2);
    hp.h2d2 = hp.d2h2 = nullptr;
    hp.ev_e2 = nullptr;
    if (hp.h2d) cudaStreamDestroy(hp.h2d);
    if (hp.d2h) cudaStreamDestroy(hp.d2h);
    hp.h2d = hp.d2h = nullptr;
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
    if (side) cudaStreamDestroy(side);
    side = nullptr;
    if (stream) cudaStreamDestroy(stream);
    stream = nullptr;
  }
  MatView view() const { return MatView{rp_bytes, rowptr, col, val, m, n_cols, nnz}; }
};

struct spmv_plan_s {
  int64_t n_rows = 0, n_cols = 0, nnz = 0;
  int rp_bytes = 4;
  spmv_options opt{};
  spmv_selection sel{};
  spmv_features feat{};
  spmv_device_props props{};
  int d16_width = 0;
  std::vector<Shard> shards;
  std::vector<int64_t> bounds;
  double upload_ms = 0, inspect_ms = 0, select_ms = 0, encode_ms = 0;
  int64_t l_split = 4096, k_long = 100, C = 2048, items = 2048, chunk = 8192;
  double hot_cover = 0.0;
  std::vector<int32_t> esc;  // D16 escape table (sorted distinct deltas >= kEsc0)
  std::vector<int32_t> d8dict;  // D8 dictionary (sorted distinct row-relative deltas, <= kD8Max)
  ProfileBounds pb;          // profile-guided mode: measured / analytic bounds
  double profile_ms = 0.0;  // nnz_split hot-x set: fraction of nonzeros in the hot columns

  bool l2_limit_set = false;  // this plan raised the device's persisting-L2 limit (x window)
  bool push_ready = false, push_ok = false;  // multi-shard iteration: halo push (prepare_push)
  ~spmv_plan_s() {
    for (auto& s : shards) s.release();
    if (l2_limit_set) {
      std::lock_guard<std::mutex> lk(g_l2_mu);
      for (auto& s : shards) {
        if (s.dev < 0 || s.dev >= 64 || g_l2_plans[s.dev] <= 0) continue;
        if (--g_l2_plans[s.dev] > 0) continue;
        cudaSetDevice(s.dev);
        cudaCtxResetPersistingL2Cache();  // demote persisting lines, then give the carve-out back
        cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, 0);
        cudaGetLastError();
      }
    }
  }
  ExecArgs args(Shard& s, const double* x, double* y) const {
    ExecArgs a{};
    a.A = s.view();
    a.x = x;
    a.y = y;
    a.vs = sel.vs;
    a.nnz_max = feat.nnz_max;
    a.sm_count = s.sm_count;
    a.sp[0] = s.sp[0];
    a.sp[1] = s.sp[1];
    a.n_sp = s.n_sp;
    a.zero_y = s.zero_y;
    a.items = s.items;
    a.Tm = s.Tm;
    a.mrow = s.mrow;
    a.mnnz = s.mnnz;
    a.mcarry_row = s.mcarry_row;
    a.mcarry_val = s.mcarry_val;
    a.l_split = l_split;
    a.chunk = chunk;
    a.n_long = s.n_long;
    a.n_chunks = s.n_chunks;
    a.long_rows = s.long_rows;
    a.chunk_start = s.chunk_start;
    a.chunk_row = s.chunk_row;
    a.chunk_val = s.chunk_val;
    a.long_tiled = s.long_tiled;
    a.nblk = s.nblk;
    a.long_seg = s.long_seg;
    a.long_c16 = s.long_c16;
    a.long_partial = s.long_partial;
    a.long_grid = s.long_grid;
    a.split_fused = s.split_fused;
    a.long_tma = s.long_tma;
    a.long_rg = s.long_rg;
    a.nz = s.nz;
    a.use_nz = s.use_nz;
    a.side = s.side;
    a.ev_fork = s.ev_fork;
    a.ev_join = s.ev_join;
    return a;
  }
  int launch(Shard& s, const double* x, double* y, int stage = 0) const {
    ExecArgs a = args(s, x, y);
    a.stage = stage;
    switch (sel.variant) {
      case SPMV_VARIANT_VECTOR: return launch_vector(a, false, s.stream);
      case SPMV_VARIANT_STREAM: return launch_stream(a, s.stream);
      case SPMV_VARIANT_MERGE: return launch_merge(a, s.stream);
      case SPMV_VARIANT_NNZSPLIT: return launch_nzsplit(a, s.stream);
      default: return launch_split(a, s.stream);
    }
  }
};

// ----------------------------------------------------------------------------
// selection (pure function, Table II)
// ----------------------------------------------------------------------------
namespace {
int pow2ceil(int64_t v) {
  int p = 1;
  while (p < v) p <<= 1;
  return p;
}

void select_impl(const spmv_features& f, const spmv_device_props& d, int rp_bytes, const spmv_options& o,
                 spmv_selection& s) {
  const int64_t k_long = o.k_long > 0 ? o.k_long : 100;
  const double avg_s = f.avg_short, sd_s = f.sd_short;
  const int64_t n = f.n, nnz = f.nnz;
  const int64_t ws = 12 * nnz + (int64_t)rp_bytes * (n + 1) + 16 * n;
  const bool skew = n > 0 && ((avg_s > 0 && sd_s / avg_s > 1.0) || (double)f.n_empty > 0.25 * (double)n);
  const bool longr = f.n_long > 0 && (double)f.nnz_max > (double)k_long * f.nnz_avg;
  int classes = 0;
  if (skew || longr) classes |= SPMV_CLASS_IMB;
  int vs = avg_s > 0 ? pow2ceil((int64_t)std::ceil(avg_s)) : 2;
  vs = std::min(32, std::max(2, vs));
  // IMB: long rows dense enough for column-tiled x blocks (a (row, 2048-col
  // block) segment averages >= 64 nonzeros) -> long_row_split (long rows
  // tiled, concurrently with one nnz_split bin of the other rows); any other
  // long-row or skewed matrix -> nnz_split (rows cut at warp-tile edges)
  const int64_t nblk = (f.n_cols + 2047) / 2048;
  const bool dense_long = f.n_long > 0 && f.nnz_long >= 64 * f.n_long * nblk;
  // tiny regular matrices (<= 2^20 nonzeros) are launch-bound: the plain
  // csr_vector kernel beats the warp-specialised stream kernel's set-up
  // (C1: 6 vs 10 us on B200, tools/table5.py)
  // scattered columns (misses/nnz > 0.75, the ML access pattern of Table I)
  // -> nnz_split: its 8 independent L1 gathers per lane beat the row-walking
  // stream kernel once the lanes' rows share no x lines (B200, uniform random
  // rows, tools/exp_random.py: 1M x 30/row 162 vs 274 us, 4M x 8/row 185 vs
  // 267 us, the C4 short rows 77 vs 156 us; equal at x >> L2)
  const bool scattered = nnz > 0 && (double)f.misses > 0.75 * (double)nnz;
  int variant = longr ? (dense_long ? SPMV_VARIANT_SPLIT : SPMV_VARIANT_NNZSPLIT)
                : skew ? SPMV_VARIANT_NNZSPLIT
                : nnz <= (1 << 20) ? SPMV_VARIANT_VECTOR
                : scattered ? SPMV_VARIANT_NNZSPLIT
                : avg_s <= 32 ? SPMV_VARIANT_STREAM
                              : SPMV_VARIANT_VECTOR;
  if (o.force_variant > 0) variant = o.force_variant;
  if (variant == SPMV_VARIANT_STREAM) {
    // cta_stream: one lane per row for rows up to 32 nonzeros (lanes walk
    // consecutive rows in step: coalesced x gathers on banded matrices), else
    // VS = pow2ceil(avg_s / 32), clamp 32 (sweep on B200: VS=1 best on C2, C5)
    vs = avg_s > 32 ? std::min(32, pow2ceil((int64_t)std::ceil(avg_s / 32.0))) : 1;
  }
  if (avg_s <= 4) classes |= SPMV_CLASS_CMP;
  if (ws > d.l2_bytes / 2 && !(classes & SPMV_CLASS_IMB)) classes |= SPMV_CLASS_MB;
  // MB -> delta colind: implemented and bit-exact, but on B200 the
  // plain stream kernel is faster on every measured MB matrix (see below;
  // DESIGN.md reading 9), so deltas are used only when forced. Large deltas
  // can be escape-coded when
  // at most kEscMax distinct values exceed kEsc0, but the
  // per-element escape check costs more than it saves (27-pt 260^3: 1.33 ms
  // with vs 1.09 ms without), so escapes are used only when forced (d16=1)
  const bool d16_ok = f.maxgap <= 65535 || f.n_big_gaps <= kEscMax;
  // (16-bit deltas are not auto-selected: with row-count tiles the plain
  // stream kernel wins on every measured MB matrix, 27-pt 180^3 281.6 vs
  // 313.9 us, C2 31.4 vs 35.0 us; the option d16 = 1 forces them)
  // MB -> dictionary-coded 8-bit deltas (D8, reading 26) when the
  // row-relative deltas take at most 256 values and every row fits a byte
  // length, on regular rows (row-count tiles, one lane per row): 1 B of index
  // per nonzero and per row instead of 4 B colind + 4/8 B rowptr
  const bool d8_ok = f.n_deltas <= kD8Max && f.nnz_max <= kD8MaxRow && nnz > 0;
  const bool regular = f.nnz_max > 0 && (double)f.nnz_max <= 1.25 * f.nnz_avg + 1.0;
  int d16 = (variant == SPMV_VARIANT_STREAM && (classes & SPMV_CLASS_MB) && d8_ok && regular && vs == 1) ? 2 : 0;
  const bool ml = nnz > 0 && (double)f.misses > 0.75 * (double)nnz && 8 * n > d.l2_bytes / 16;
  if (ml) classes |= SPMV_CLASS_ML;
  bool xwin = ml && 8 * n <= d.access_window_max;
  // explicit options override the feature-guided choice
  if (o.force_vs > 0) vs = o.force_vs;
  if (o.d16 == 0) d16 = 0;
  if (o.d16 == 1) d16 = d16_ok ? 1 : 0;
  if (o.d16 == 2) d16 = d8_ok ? 2 : 0;
  if (variant != SPMV_VARIANT_STREAM) d16 = 0;
  if (d16 == 2 && o.d16 == 2 && o.force_vs <= 0) vs = 1;  // forced D8: its kernel runs one lane per row
  if (d16 == 2 && vs != 1) d16 = 0;  // D8: one lane per row
  if (o.xwin == 0) xwin = false;
  if (o.xwin == 1) xwin = true;
  // cta_stream consumer mode: segmented (products first, balanced row walk)
  // for random-gather tiles: the long_row_split short part, or a STREAM
  // matrix whose in-row gaps mostly exceed a cache line
  bool seg = variant == SPMV_VARIANT_STREAM && nnz > 0 && (double)f.misses > 0.75 * (double)nnz;
  if (o.seg == 0) seg = false;
  if (o.seg == 1) seg = variant == SPMV_VARIANT_SPLIT || variant == SPMV_VARIANT_STREAM;
  if (d16) seg = false;
  s.variant = variant;
  s.vs = vs;
  s.d16 = d16;
  s.xwin = xwin ? 1 : 0;
  s.classes = classes;
  s.seg = seg ? 1 : 0;
}

// ---- profile-guided mode -------------------------------------
// Fig. 4 on the measured bounds, strict ">", "P_CSR ~ P_MB" read
// as P_CSR >= (1 - tol) P_MB (reading 22). The thresholds
// are the classifier's hyperparameters, tuned per platform by grid search
// (the paper's KNC values T_IMB = 1.24, T_ML = 1.25);
// the defaults are this library's grid search on B200 (reading 29).
constexpr double kTImbB200 = 2.54, kTMlB200 = 1.08, kTolB200 = 0.10;  // profiles/r02_profile_tuning.json
int classify_profile(const ProfileBounds& b, const spmv_options& o) {
  const double t_imb = o.t_imb > 0 ? o.t_imb : kTImbB200;
  const double t_ml = o.t_ml > 0 ? o.t_ml : kTMlB200;
  const double tol = o.approx_tol > 0 ? o.approx_tol : kTolB200;
  int c = 0;
  if (b.p_csr <= 0) return 0;
  if (b.p_imb / b.p_csr > t_imb) c |= SPMV_CLASS_IMB;
  if (b.p_ml / b.p_csr > t_ml) c |= SPMV_CLASS_ML;
  if (b.p_csr >= (1.0 - tol) * b.p_mb && b.p_mb < b.p_cmp && b.p_cmp < b.p_peak) c |= SPMV_CLASS_MB;
  if (b.p_mb > b.p_cmp || b.p_cmp > b.p_peak) c |= SPMV_CLASS_CMP;
  return c;
}

// Table II for the GPU: IMB -> decomposition (dense long rows:
// long_row_split) or nnz_split (the "auto" analogue); ML -> nnz_split (L1 x
// gathers + hot-x table, the prefetch analogue) with the x window; MB ->
// cta_stream + 16-bit deltas when the gaps fit; CMP -> cta_stream (rows sized
// to lanes, the unroll/vectorise analogue); no class -> the CSR baseline
// (csr_vector), "not worth optimising". Precedence IMB > ML > MB/CMP.
void profile_select_impl(const spmv_features& f, const spmv_device_props& d, const spmv_options& o,
                         const ProfileBounds& b, spmv_selection& s) {
  const int classes = o.force_classes >= 0 ? o.force_classes : classify_profile(b, o);
  const int64_t k_long = o.k_long > 0 ? o.k_long : 100;
  const double avg_s = f.avg_short;
  const bool longr = f.n_long > 0 && (double)f.nnz_max > (double)k_long * f.nnz_avg;
  const int64_t nblk = (f.n_cols + 2047) / 2048;
  const bool dense_long = f.n_long > 0 && f.nnz_long >= 64 * f.n_long * nblk;
  int variant;
  if (classes & SPMV_CLASS_IMB) variant = (longr && dense_long) ? SPMV_VARIANT_SPLIT : SPMV_VARIANT_NNZSPLIT;
  else if (classes & SPMV_CLASS_ML) variant = SPMV_VARIANT_NNZSPLIT;
  else if (classes & (SPMV_CLASS_MB | SPMV_CLASS_CMP)) variant = SPMV_VARIANT_STREAM;
  else variant = SPMV_VARIANT_VECTOR;
  int vs = avg_s > 0 ? std::min(32, std::max(2, pow2ceil((int64_t)std::ceil(avg_s)))) : 2;
  if (variant == SPMV_VARIANT_STREAM)
    vs = avg_s > 32 ? std::min(32, pow2ceil((int64_t)std::ceil(avg_s / 32.0))) : 1;
  int d16 = 0;
  if ((classes & SPMV_CLASS_MB) && variant == SPMV_VARIANT_STREAM)
    d16 = (f.n_deltas <= kD8Max && f.nnz_max <= kD8MaxRow && vs == 1) ? 2 : (f.maxgap <= 65535 ? 1 : 0);
  bool xwin = (classes & SPMV_CLASS_ML) && 8 * f.n <= d.access_window_max;
  if (o.force_vs > 0) vs = o.force_vs;
  if (o.d16 == 0) d16 = 0;
  if (d16 == 2 && vs != 1) d16 = 0;
  if (o.xwin == 0) xwin = false;
  if (o.xwin == 1) xwin = true;
  s.variant = variant;
  s.vs = vs;
  s.d16 = d16;
  s.xwin = xwin ? 1 : 0;
  s.classes = classes;
  s.seg = 0;
}

// profile mode, second stage (reading 30): the D8 conditions of the feature
// rules -- at most 256 distinct row-relative deltas, rows <= 255 nonzeros,
// regular rows, one lane per row
bool profile_stage2_ok(const spmv_features& f, const spmv_selection& s) {
  const bool regular = f.nnz_max > 0 && (double)f.nnz_max <= 1.25 * f.nnz_avg + 1.0;
  return f.n_deltas <= kD8Max && f.nnz_max <= kD8MaxRow && f.nnz > 0 && regular && s.vs == 1;
}

void validate_options(const spmv_options& o) {
  if (o.force_variant < 0 || o.force_variant > 5) fail(SPMV_E_ARG, "force_variant %d out of range", o.force_variant);
  if (o.force_vs != 0 && o.force_vs != 1 && o.force_vs != 2 && o.force_vs != 4 && o.force_vs != 8 &&
      o.force_vs != 16 && o.force_vs != 32)
    fail(SPMV_E_ARG, "force_vs %d not in {0,1,2,4,8,16,32}", o.force_vs);
  if (o.tile_nnz != 0 && (o.tile_nnz % 128 || o.tile_nnz < 128 || o.tile_nnz > 16384))
    fail(SPMV_E_ARG, "tile_nnz %lld must be a multiple of 128 in [128, 16384]", (long long)o.tile_nnz);
  if (o.merge_items != 0 && o.merge_items != 2048) fail(SPMV_E_ARG, "merge_items must be 2048");
  if (o.long_chunk != 0 && (o.long_chunk % 256 || o.long_chunk < 256))
    fail(SPMV_E_ARG, "long_chunk must be a positive multiple of 256");
  if (o.l_split < 0 || o.k_long < 0) fail(SPMV_E_ARG, "negative l_split / k_long");
  if (o.long_mode < 0 || o.long_mode > 3) fail(SPMV_E_ARG, "long_mode must be 0, 1, 2 or 3");
  if (o.select_mode < 0 || o.select_mode > 1) fail(SPMV_E_ARG, "select_mode must be 0 (feature) or 1 (profile)");
  if (!(o.t_imb >= 0) || !(o.t_ml >= 0) || !(o.approx_tol >= 0) || o.approx_tol >= 1)
    fail(SPMV_E_ARG, "t_imb / t_ml must be >= 0 (0 = default) and approx_tol in [0, 1)");
  if (o.force_classes < -1 || o.force_classes > 15) fail(SPMV_E_ARG, "force_classes must be -1 or a class set 0..15");
  if (o.hot_x < -1) fail(SPMV_E_ARG, "hot_x must be -1 (auto), 0 (off) or a column count");
  if (o.split_bins < -1 || o.split_bins > 1) fail(SPMV_E_ARG, "split_bins must be -1, 0 or 1");
  if (o.d16 < -1 || o.d16 > 2) fail(SPMV_E_ARG, "d16 must be -1 (auto), 0 (off), 1 (16-bit deltas) or 2 (D8)");
  if (o.stages < 0 || o.stages > 32 || o.stages % kStreamConsumerWarps)
    fail(SPMV_E_ARG, "stages must be 0 (auto) or a multiple of %d up to 32", kStreamConsumerWarps);
}

void features_from_stats(const std::vector<DevStats>& st, const std::vector<int64_t>& m, spmv_features& f) {
  memset(&f, 0, sizeof f);
  f.nnz_min = LLONG_MAX;
  for (size_t g = 0; g < st.size(); ++g) {
    const DevStats& s = st[g];
    f.n += m[g];
    f.s1 += s.s1;
    f.s2 += s.s2;
    f.s1_short += s.s1_short;
    f.s2_short += s.s2_short;
    if (m[g] > 0) f.nnz_min = std::min<int64_t>(f.nnz_min, s.nnz_min);
    f.nnz_max = std::max<int64_t>(f.nnz_max, s.nnz_max);
    f.n_empty += s.n_empty;
    f.n_long += s.n_long;
    f.nnz_long += s.nnz_long;
    f.n_short += s.n_short;
    f.max_short = std::max<int64_t>(f.max_short, s.max_short);
    f.maxgap = std::max<int64_t>(f.maxgap, s.maxgap);
    f.misses += s.misses;
  }
  if (f.n == 0) f.nnz_min = 0;
  f.col_min = LLONG_MAX;
  f.col_max = -1;
  for (const auto& s : st) {
    f.col_min = std::min<int64_t>(f.col_min, s.col_min);
    f.col_max = std::max<int64_t>(f.col_max, s.col_max);
  }
  if (f.col_max < 0) f.col_min = 0;  // no nonzeros: the empty range [0, 0)
  {  // distinct in-row gaps >= kEsc0 over all shards (kBigTab + 1 = more than kBigTab)
    std::vector<int32_t> big;
    bool over = false;
    for (const auto& s : st) {
      over = over || s.big_over;
      for (int i = 0; i < kBigTab; ++i)
        if (s.bigtab[i] > 0) big.push_back(s.bigtab[i]);
    }
    std::sort(big.begin(), big.end());
    big.erase(std::unique(big.begin(), big.end()), big.end());
    f.n_big_gaps = (over || (int64_t)big.size() > kBigTab) ? kBigTab + 1 : (int64_t)big.size();
  }
  {  // distinct row-relative deltas over all shards (kD8Max + 1 = more than kD8Max)
    std::vector<int32_t> d;
    bool over = false;
    for (const auto& s : st) {
      over = over || s.d_over;
      for (int i = 0; i < kDTab; ++i)
        if (s.dtab[i] != INT32_MIN) d.push_back(s.dtab[i]);
    }
    std::sort(d.begin(), d.end());
    d.erase(std::unique(d.begin(), d.end()), d.end());
    f.n_deltas = (over || (int64_t)d.size() > kD8Max) ? kD8Max + 1 : (int64_t)d.size();
  }
  f.nnz = (int64_t)f.s1;
  auto sd = [](uint64_t cnt, uint64_t s1, uint64_t s2) {
    if (cnt == 0) return 0.0;
    unsigned __int128 a = (unsigned __int128)cnt * s2, b = (unsigned __int128)s1 * s1;
    return std::sqrt((double)(a - b)) / (double)cnt;
  };
  f.nnz_avg = f.n ? (double)f.s1 / (double)f.n : 0.0;
  f.nnz_sd = sd((uint64_t)f.n, f.s1, f.s2);
  f.avg_short = f.n_short ? (double)f.s1_short / (double)f.n_short : 0.0;
  f.sd_short = sd((uint64_t)f.n_short, f.s1_short, f.s2_short);
}

void query_props(int dev, spmv_device_props& p) {
  cudaDeviceProp d;
  ck(cudaGetDeviceProperties(&d, dev), "cudaGetDeviceProperties");
  p.sm_count = d.multiProcessorCount;
  p.cc_major = d.major;
  p.cc_minor = d.minor;
  p.pad_ = 0;
  p.l2_bytes = d.l2CacheSize;
  p.persisting_l2_max = d.persistingL2CacheMaxSize;
  p.access_window_max = d.accessPolicyMaxWindowSize;
  p.global_mem_bytes = (int64_t)d.totalGlobalMem;
}

void shard_bounds_host(int64_t n, const void* rp, int bytes, int G, int64_t* b) {
  const int64_t nnz = rp_at(rp, bytes, n);
  b[0] = 0;
  for (int g = 1; g < G; ++g) {
    const int64_t key = (g * nnz + G - 1) / G;
    int64_t lo = 0, hi = n + 1;
    while (lo < hi) {
      const int64_t mid = lo + (hi - lo) / 2;
      if (rp_at(rp, bytes, mid) < key) lo = mid + 1; else hi = mid;
    }
    b[g] = std::min(lo, n);
  }
  b[G] = n;
}

const char* csr_code_name(int code) {
  switch (code) {
    case 1: return "rowptr[0] != 0";
    case 2: return "rowptr[n] != nnz";
    case 3: return "rowptr decreasing";
    case 4: return "colind out of range";
    case 5: return "colind not strictly increasing in row";
    default: return "?";
  }
}

[[noreturn]] void fail_csr(int code, int64_t where) {
  fail(SPMV_E_CSR, "invalid CSR: code %d (%s) at %s %lld", code, csr_code_name(code),
       code <= 3 ? "row" : "nonzero", (long long)where);
}

// ordered-carry arrays: fixup_capacity(T) entries (hierarchical levels) plus
// the zeroed level counter the fix-up's last CTA uses
void alloc_carries(Shard& s, int64_t T, int32_t*& row, double*& val) {
  const int64_t cap = fixup_capacity(T);
  row = s.alloc<int32_t>((size_t)cap + 2);
  val = s.alloc<double>((size_t)cap);
  ck(cudaMemsetAsync(row + cap, 0, 8, s.stream), "memset");
}

// ---------------------------------------------------------------------------
spmv_plan create_impl(int64_t n_rows, int64_t n_cols, int64_t nnz, const void* rowptr, int rp_bytes,
                      const int32_t* colind, const double* values, int ngpus, const spmv_options* optp) {
  if (!rowptr || (nnz > 0 && (!colind || !values))) fail(SPMV_E_ARG, "null array pointer");
  if (n_rows < 0 || n_cols < 0 || nnz < 0) fail(SPMV_E_ARG, "negative size");
  if (rp_bytes != 4 && rp_bytes != 8) fail(SPMV_E_ARG, "rowptr_bytes must be 4 or 8");
  if (n_rows >= INT32_MAX || n_cols > INT32_MAX)
    fail(SPMV_E_UNSUPPORTED, "n >= 2^31 is not supported (int32 colind / row ids)");
  if (rp_bytes == 4 && nnz > INT32_MAX) fail(SPMV_E_UNSUPPORTED, "nnz >= 2^31 needs a 64-bit rowptr");
  spmv_options opt;
  spmv_options_default(&opt);
  if (optp) {
    if (optp->struct_size != (int32_t)sizeof(spmv_options)) fail(SPMV_E_ARG, "spmv_options.struct_size mismatch");
    opt = *optp;
  }
  validate_options(opt);
  int ndev = 0;
  ck(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
  if (ngpus < 1 || ngpus > 8) fail(SPMV_E_ARG, "ngpus %d out of range [1, 8]", ngpus);
  if (ngpus > ndev && !opt.emulate_devices) fail(SPMV_E_ARG, "ngpus %d > %d visible devices", ngpus, ndev);
  int cur = 0;
  ck(cudaGetDevice(&cur), "cudaGetDevice");

  auto P = std::unique_ptr<spmv_plan_s>(new spmv_plan_s());
  P->n_rows = n_rows;
  P->n_cols = n_cols;
  P->nnz = nnz;
  P->rp_bytes = rp_bytes;
  P->opt = opt;
  P->l_split = opt.l_split > 0 ? opt.l_split : 4096;
  P->k_long = opt.k_long > 0 ? opt.k_long : 100;
  P->C = opt.tile_nnz > 0 ? opt.tile_nnz : 512;
  P->items = 2048;
  P->chunk = opt.long_chunk > 0 ? opt.long_chunk : 8192;
  query_props(cur, P->props);

  // ---- a1: host-side rowptr end checks, shard bounds ----------------------------
  double t_a = now_ms();
  int rp_dev = -1;
  const bool rp_on_dev = is_device_ptr(rowptr, &rp_dev);
  std::vector<unsigned char> rp_host;
  const void* rp_h = rowptr;
  if (rp_on_dev && ngpus > 1) {
    rp_host.resize((size_t)(n_rows + 1) * rp_bytes);
    ck(cudaMemcpy(rp_host.data(), rowptr, rp_host.size(), cudaMemcpyDeviceToHost), "copy rowptr");
    rp_h = rp_host.data();
  }
  int64_t rp0, rpn;
  if (rp_on_dev && ngpus == 1) {
    ck(cudaMemcpy(&rp0, rowptr, rp_bytes, cudaMemcpyDeviceToHost), "copy rowptr[0]");
    ck(cudaMemcpy(&rpn, (const char*)rowptr + n_rows * rp_bytes, rp_bytes, cudaMemcpyDeviceToHost), "rowptr[n]");
    if (rp_bytes == 4) { rp0 = (int32_t)rp0; rpn = (int32_t)rpn; }
  } else {
    rp0 = rp_at(rp_h, rp_bytes, 0);
    rpn = rp_at(rp_h, rp_bytes, n_rows);
  }
  // (always checked, even with validate = 0: the shard bounds and every
  // size below are derived from rowptr[0] and rowptr[n])
  if (rp0 != 0) fail_csr(1, 0);
  if (rpn != nnz) fail_csr(2, n_rows);
  P->bounds.assign(ngpus + 1, 0);
  if (ngpus == 1) { P->bounds[1] = n_rows; }
  else shard_bounds_host(n_rows, rp_h, rp_bytes, ngpus, P->bounds.data());

  // ---- a1: upload every shard ---------------------------------------------------
  P->shards.resize(ngpus);
  for (int g = 0; g < ngpus; ++g) {
    Shard& s = P->shards[g];
    s.dev = opt.emulate_devices ? cur : g;
    ck(cudaSetDevice(s.dev), "cudaSetDevice");
    ck(cudaStreamCreateWithFlags(&s.stream, cudaStreamNonBlocking), "cudaStreamCreate");
    ck(cudaEventCreateWithFlags(&s.ev_part, cudaEventDisableTiming), "cudaEventCreate");
    ck(cudaEventCreateWithFlags(&s.ev_x, cudaEventDisableTiming), "cudaEventCreate");
    cudaDeviceProp dp;
    ck(cudaGetDeviceProperties(&dp, s.dev), "cudaGetDeviceProperties");
    s.sm_count = dp.multiProcessorCount;
    s.row0 = P->bounds[g];
    s.m = P->bounds[g + 1] - P->bounds[g];
    s.n_cols = n_cols;
    s.rp_bytes = rp_bytes;
    s.nnz0 = ngpus == 1 ? 0 : rp_at(rp_h, rp_bytes, s.row0);
    s.nnz = ngpus == 1 ? nnz : rp_at(rp_h, rp_bytes, s.row0 + s.m) - s.nnz0;
    if (s.nnz < 0) fail_csr(3, s.row0);
    s.rowptr = s.alloc<char>((size_t)(s.m + 1) * rp_bytes);
    s.col = s.alloc<int32_t>((size_t)s.nnz);
    s.val = s.alloc<double>((size_t)s.nnz);
    upload(s.rowptr, (const char*)rowptr + s.row0 * rp_bytes, (size_t)(s.m + 1) * rp_bytes, s.stream);
    if (s.nnz) {
      upload(s.col, colind + s.nnz0, (size_t)s.nnz * 4, s.stream);
      upload(s.val, values + s.nnz0, (size_t)s.nnz * 8, s.stream);
    }
    launch_rebase(s.rowptr, rp_bytes, s.m + 1, s.nnz0, s.stream);
    count_launches(s.nnz0 ? 1 : 0, "rebase");
  }
  for (auto& s : P->shards) ck(cudaStreamSynchronize(s.stream), "upload sync");
  // in-process shards on distinct devices exchange partials and x halos with
  // peer copies: enable direct peer access (NVLink / NVSwitch) where the
  // pair supports it (otherwise the runtime stages the copies)
  if (ngpus > 1 && !opt.emulate_devices) {
    for (int a = 0; a < ngpus; ++a)
      for (int b = 0; b < ngpus; ++b) {
        if (a == b) continue;
        int can = 0;
        if (cudaDeviceCanAccessPeer(&can, a, b) == cudaSuccess && can) {
          ck(cudaSetDevice(a), "cudaSetDevice");
          const cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
          if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) ck(e, "cudaDeviceEnablePeerAccess");
          cudaGetLastError();
        }
      }
    ck(cudaSetDevice(cur), "cudaSetDevice");
  }
  P->upload_ms = now_ms() - t_a;

  // ---- a2: inspector (features, validation, max gap) ---------------------------------
  double t_b = now_ms();
  for (auto& s : P->shards) {
    ck(cudaSetDevice(s.dev), "cudaSetDevice");
    s.stats = s.alloc<DevStats>(1);
    s.headbits = s.alloc<uint32_t>((size_t)(s.nnz + 31) / 32 + 1);
    DevStats init{};
    init.nnz_min = LLONG_MAX;
    init.rp_err = LLONG_MAX;
    init.col_err = LLONG_MAX;
    init.col_min = LLONG_MAX;
    init.col_max = -1;
    for (int i = 0; i < kDTab; ++i) init.dtab[i] = INT32_MIN;
    ck(cudaMemcpyAsync(s.stats, &init, sizeof init, cudaMemcpyHostToDevice, s.stream), "stats init");
    ck(cudaMemsetAsync(s.headbits, 0, ((size_t)(s.nnz + 31) / 32 + 1) * 4, s.stream), "memset");
    launch_rowstats(s.view(), P->l_split, s.row0, s.headbits, s.stats, s.stream);
    count_launches(s.m ? 1 : 0, "rowstats");
    ck(cudaMemcpyAsync(&s.hs, s.stats, sizeof(DevStats), cudaMemcpyDeviceToHost, s.stream), "stats");
  }
  for (auto& s : P->shards) {
    ck(cudaStreamSynchronize(s.stream), "rowstats");
    if (s.hs.rp_err != LLONG_MAX) fail_csr(3, s.row0 + s.hs.rp_err);
  }
  for (auto& s : P->shards) {
    ck(cudaSetDevice(s.dev), "cudaSetDevice");
    launch_validate_gaps(s.view(), s.headbits, s.stats, s.stream);
    count_launches(s.nnz ? 1 : 0, "validate_gaps");
    launch_x_reuse(s.view(), s.stats, s.stream);
    count_launches(s.m > 1 && s.nnz ? 1 : 0, "x_reuse");
    ck(cudaMemcpyAsync(&s.hs, s.stats, sizeof(DevStats), cudaMemcpyDeviceToHost, s.stream), "stats");
  }
  for (auto& s : P->shards) {
    ck(cudaStreamSynchronize(s.stream), "validate");
    if (opt.validate && s.hs.col_err != LLONG_MAX) {
      const int code = (s.hs.col_err & 1) ? 5 : 4;
      fail_csr(code, s.nnz0 + (s.hs.col_err >> 1));
    }
  }
  P->inspect_ms = now_ms() - t_b;

  // ---- a5: selection -------------------------------------------------------------
  double t_c = now_ms();
  std::vector<DevStats> st;
  std::vector<int64_t> ms;
  for (auto& s : P->shards) { st.push_back(s.hs); ms.push_back(s.m); }
  features_from_stats(st, ms, P->feat);
  P->feat.n_cols = n_cols;
  select_impl(P->feat, P->props, rp_bytes, opt, P->sel);
  if (opt.select_mode == 1 && opt.force_classes >= 0) {
    // profile-guided mapping of a given class set (no probes: tools/tune_profile.py)
    if (opt.force_variant == 0) profile_select_impl(P->feat, P->props, opt, P->pb, P->sel);
  } else if (opt.select_mode == 1) {
    // profile-guided: three timed micro-benchmarks of the CSR baseline on
    // shard 0 (Sec. III-B), then Fig. 4 and the Table II mapping; their time
    // is the classifier's t_pre
    Shard& s0 = P->shards[0];
    ck(cudaSetDevice(s0.dev), "cudaSetDevice");
    const double t_p = now_ms();
    const int vs0 = P->feat.avg_short > 0
                        ? std::min(32, std::max(2, pow2ceil((int64_t)std::ceil(P->feat.avg_short))))
                        : 2;
    double *px = nullptr, *py = nullptr;
    ck(cudaMalloc(&px, (size_t)std::max<int64_t>(s0.n_cols, 1) * 8 + 64), "cudaMalloc");
    if (cudaMalloc(&py, (size_t)std::max<int64_t>(s0.m, 1) * 8 + 64) != cudaSuccess) {
      cudaFree(px);
      ck(cudaErrorMemoryAllocation, "cudaMalloc");
    }
    const int rc = run_profile_probes(s0.view(), vs0, s0.sm_count, P->props.l2_bytes, px, py, P->pb, s0.stream);
    cudaFree(px);
    cudaFree(py);
    if (rc != 0) ck(cudaGetLastError() != cudaSuccess ? cudaGetLastError() : cudaErrorUnknown, "profile probes");
    P->profile_ms = now_ms() - t_p;
    if (opt.force_variant == 0) profile_select_impl(P->feat, P->props, opt, P->pb, P->sel);
  }
  if (P->sel.d16 == 1) P->d16_width = P->feat.maxgap <= 255 ? 8 : 16;
  auto make_d8dict = [&]() {
    // D8 dictionary: the sorted distinct row-relative deltas of all shards
    P->d16_width = 8;
    std::vector<int32_t> d;
    for (auto& sh : P->shards)
      for (int i = 0; i < kDTab; ++i)
        if (sh.hs.dtab[i] != INT32_MIN) d.push_back(sh.hs.dtab[i]);
    std::sort(d.begin(), d.end());
    d.erase(std::unique(d.begin(), d.end()), d.end());
    if ((int)d.size() > kD8Max) fail(SPMV_E_CUDA, "D8 dictionary overflow (%d entries)", (int)d.size());
    P->d8dict = d;
  };
  if (P->sel.d16 == 2) make_d8dict();
  // escape table: the sorted distinct large deltas of all shards
  if (P->sel.d16 == 1 && P->feat.maxgap > 65535) {
    std::vector<int32_t> big;
    for (auto& sh : P->shards)
      for (int i = 0; i < kBigTab; ++i)
        if (sh.hs.bigtab[i] > 0) big.push_back(sh.hs.bigtab[i]);
    std::sort(big.begin(), big.end());
    big.erase(std::unique(big.begin(), big.end()), big.end());
    P->esc.assign(big.begin(), big.end());
  }
  P->select_ms = now_ms() - t_c;

  // ---- a3/a4: structures for the selected variant ---------------------------------
  double t_d = now_ms();
  // Row-pattern mode of D8 (reading 31): when the shard's rows
  // follow <= 256 patterns (length + column offsets from the row id) holding
  // <= kPatMaxOfs offsets, the per-row byte names the row's pattern and no
  // per-nonzero index is stored at all -- the P_peak limit of P:341-344 up
  // to one byte per row. Patterns are numbered by their first row (the
  // oracle's order); every row is verified against its pattern.
  auto build_patterns = [&](Shard& s, StreamPlan& sp, const MatView& V) -> bool {
    if (V.m == 0) return false;
    if (const char* e = getenv("SPMV_D8_PATTERNS"))
      if (atoi(e) == 0) return false;  // experiments / tests: the 8-bit codes
    unsigned long long* gk = s.alloc<unsigned long long>(2 * kPatGlobal);
    int* flag = s.alloc<int>(1);
    std::vector<void*> tmp = {gk, flag};
    auto done = [&](bool ok) {
      for (void* q : tmp) s.free_alloc(q);
      return ok;
    };
    ck(cudaMemsetAsync(gk, 0, kPatGlobal * 8, s.stream), "memset");
    ck(cudaMemsetAsync(gk + kPatGlobal, 0xff, kPatGlobal * 8, s.stream), "memset");
    ck(cudaMemsetAsync(flag, 0, 4, s.stream), "memset");
    launch_pat_collect(V, sp.row0, gk, gk + kPatGlobal, flag, s.stream);
    count_launches(1, "pattern collect");
    std::vector<unsigned long long> hk(2 * kPatGlobal);
    int hf = 0;
    ck(cudaMemcpyAsync(hk.data(), gk, 16 * kPatGlobal, cudaMemcpyDeviceToHost, s.stream), "patterns");
    ck(cudaMemcpyAsync(&hf, flag, 4, cudaMemcpyDeviceToHost, s.stream), "patterns");
    ck(cudaStreamSynchronize(s.stream), "patterns");
    if (hf) return done(false);
    std::vector<std::pair<unsigned long long, unsigned long long>> pat;  // (first row, hash)
    for (int t = 0; t < kPatGlobal; ++t)
      if (hk[(size_t)t]) pat.push_back({hk[(size_t)(kPatGlobal + t)], hk[(size_t)t]});
    if (pat.empty() || pat.size() > 256) return done(false);
    std::sort(pat.begin(), pat.end());
    // each pattern's offsets, read from its first row
    std::vector<int32_t> desc(256, 0), ofs;
    for (size_t q = 0; q < pat.size(); ++q) {
      const int64_t r = (int64_t)pat[q].first;
      int64_t ab[2] = {0, 0};
      if (V.rp_bytes == 8) {
        ck(cudaMemcpy(ab, (const int64_t*)V.rowptr + r, 16, cudaMemcpyDeviceToHost), "pattern row");
      } else {
        int32_t w[2];
        ck(cudaMemcpy(w, (const int32_t*)V.rowptr + r, 8, cudaMemcpyDeviceToHost), "pattern row");
        ab[0] = w[0];
        ab[1] = w[1];
      }
      const int64_t len = ab[1] - ab[0];
      if (len > 255 || (int64_t)ofs.size() + len > kPatMaxOfs) return done(false);
      std::vector<int32_t> c((size_t)len);
      if (len) ck(cudaMemcpy(c.data(), V.col + ab[0], (size_t)len * 4, cudaMemcpyDeviceToHost), "pattern row");
      desc[q] = (int32_t)((len << 16) | (int64_t)ofs.size());
      for (int64_t t = 0; t < len; ++t) ofs.push_back((int32_t)((int64_t)c[(size_t)t] - (sp.row0 + r)));
    }
    const int np = (int)pat.size(), nofs = (int)ofs.size();
    std::vector<std::pair<unsigned long long, int32_t>> byk;
    for (int q = 0; q < np; ++q) byk.push_back({pat[(size_t)q].second, q});
    std::sort(byk.begin(), byk.end());
    std::vector<unsigned long long> skey;
    std::vector<int32_t> sid;
    for (auto& e : byk) {
      skey.push_back(e.first);
      sid.push_back(e.second);
    }
    unsigned long long* skey_d = s.alloc<unsigned long long>(256);
    int32_t* sid_d = s.alloc<int32_t>(256);
    tmp.push_back(skey_d);
    tmp.push_back(sid_d);
    int32_t* desc_d = s.alloc<int32_t>(256);
    int32_t* ofs_d = s.alloc<int32_t>((size_t)nofs + 16);
    uint8_t* ids = s.alloc<uint8_t>((size_t)V.m);
    ck(cudaMemcpyAsync(skey_d, skey.data(), (size_t)np * 8, cudaMemcpyHostToDevice, s.stream), "patterns");
    ck(cudaMemcpyAsync(sid_d, sid.data(), (size_t)np * 4, cudaMemcpyHostToDevice, s.stream), "patterns");
    ck(cudaMemcpyAsync(desc_d, desc.data(), 256 * 4, cudaMemcpyHostToDevice, s.stream), "patterns");
    if (nofs) ck(cudaMemcpyAsync(ofs_d, ofs.data(), (size_t)nofs * 4, cudaMemcpyHostToDevice, s.stream), "patterns");
    launch_pat_assign(V, sp.row0, skey_d, sid_d, np, desc_d, ofs_d, nofs, ids, flag, s.stream);
    count_launches(1, "pattern assign");
    ck(cudaMemcpyAsync(&hf, flag, 4, cudaMemcpyDeviceToHost, s.stream), "patterns");
    ck(cudaStreamSynchronize(s.stream), "patterns");
    if (hf) {
      tmp.push_back(desc_d);
      tmp.push_back(ofs_d);
      tmp.push_back(ids);
      return done(false);
    }
    sp.d8_bits = 0;
    sp.n_dict = np;
    for (int q = 0; q < 256; ++q) sp.dict[q] = desc[(size_t)q];
    sp.d8_dict_dev = desc_d;
    sp.pat_ofs = ofs_d;
    sp.n_pat_ofs = nofs;
    sp.codes = ids;  // (marks the plan as D8; the kernel stages the ids as its per-row byte)
    sp.rlen = ids;
    return done(true);
  };

  // cta_stream structures over the CSR view V (the whole shard, or one
  // compacted length bin of long_row_split mapped back through rowmap)
  auto build_stream = [&](Shard& s, StreamPlan& sp, const MatView& V, const int32_t* rowmap, int dmode, int vs,
                          bool seg, int64_t maxlen) {
    sp.V = V;
    sp.rowmap = rowmap;
    sp.vs = vs;
    sp.seg = seg;
    const bool d16 = dmode == 1;
    const double avg = V.m ? (double)V.nnz / (double)V.m : 0.0;
    if (dmode == 2) {
      // ---- D8 (d8.cu): row-count tiles of Rt rows (multiple of 16: the row
      // lengths are bulk-copied from k*Rt), the fewest giving >= 576 nonzeros
      // on average (as the int32 path), capacity Rt x longest row
      int64_t Rt = 32;
      double min_nz = 576.0;
      if (const char* e = getenv("SPMV_ROW_TILE_MIN_NNZ")) min_nz = atof(e);  // experiments
      while ((double)Rt * avg < min_nz && Rt < 4096) Rt += 32;
      const int64_t ml = std::max<int64_t>(maxlen, 1);
      int cw = 0;
      if (const char* e = getenv("SPMV_D8_CW")) cw = atoi(e);  // experiments: 4, 6 or 8
      sp.d8_un = 8;
      if (const char* e = getenv("SPMV_D8_UN")) sp.d8_un = atoi(e) == 16 ? 16 : 8;  // experiments: 8 or 16
      // shrink the tile until 4 stages fit (long rows of a forced D8 plan)
      while (Rt > 16 && d8_smem_bytes(Rt * ml, Rt, 4, 8) > 227 * 1024 - kStaticSmemMargin) Rt -= 16;
      sp.rows_per_tile = Rt;
      sp.C = ((Rt * ml + 31) / 32) * 32;
      P->C = sp.C;
      sp.aligned = true;
      sp.stride = sp.C;
      sp.T = std::max<int64_t>(1, (V.m + Rt - 1) / Rt);
      sp.rows_cap = (int)Rt;
      sp.tile_row = s.alloc<int32_t>((size_t)sp.T + 1);
      alloc_carries(s, sp.T, sp.carry_row, sp.carry_val);
      launch_tile_rows_count(sp.tile_row, sp.T, Rt, V.m, s.stream);
      sp.tile_nz = s.alloc<int64_t>((size_t)sp.T + 1);
      launch_tile_nz(V, sp.tile_row, sp.T, sp.tile_nz, s.stream);
      count_launches(2, "d8 tiles");
      sp.row0 = s.row0;
      if (build_patterns(s, sp, V)) {
        // row patterns: the batch width whose multiples fit the longest
        // pattern (the interior rows) with the fewest idle slots -- 27-pt:
        // 9 (3 batches, none idle), 7-pt: 7; ties keep 8. B200, C5: 2123 ->
        // 2045 us with 9
        int64_t L = 0;
        for (int q = 0; q < sp.n_dict; ++q) L = std::max<int64_t>(L, (sp.dict[q] >> 16) & 0xff);
        int best_un = 8;
        for (int un : {8, 9, 7})
          if ((L + un - 1) / un * un < (L + best_un - 1) / best_un * best_un) best_un = un;
        sp.d8_un = best_un;
        if (const char* e = getenv("SPMV_D8_UN")) sp.d8_un = atoi(e);  // experiments: 7, 8, 9 or 16
        if (sp.d8_un != 7 && sp.d8_un != 8 && sp.d8_un != 9 && sp.d8_un != 16) sp.d8_un = 8;
      } else {
      sp.n_dict = (int)P->d8dict.size();
      for (int i = 0; i < sp.n_dict; ++i) sp.dict[i] = P->d8dict[(size_t)i];
      int32_t* dict_dev = s.alloc<int32_t>(256);
      ck(cudaMemcpyAsync(dict_dev, sp.dict, sizeof sp.dict, cudaMemcpyHostToDevice, s.stream), "d8 dict");
      uint8_t* codes = s.alloc<uint8_t>((size_t)V.nnz);
      uint8_t* rlen = s.alloc<uint8_t>((size_t)V.m);
      sp.row0 = s.row0;
      launch_d8_encode(V, sp.row0, dict_dev, sp.n_dict, codes, rlen, s.stream);
      count_launches(V.m ? 1 : 0, "d8 encode");
      // 8-bit codes; 4-bit codes (two per byte, <= 16 dictionary entries) are
      // kept as an experiment: measured SLOWER on B200 (C5 2.41 vs 2.23 ms,
      // C2 32.4 vs 28.3 us -- the nibble extraction lengthens the consumer's
      // decode chain, and the kernel is bound by that latency, not by bytes)
      sp.d8_bits = 8;
      if (const char* e = getenv("SPMV_D8_BITS")) sp.d8_bits = (atoi(e) == 4 && sp.n_dict <= 16) ? 4 : 8;  // experiments
      if (sp.d8_bits == 4) {
        uint8_t* packed = s.alloc<uint8_t>((size_t)(V.nnz + 1) / 2);
        launch_d8_pack4(codes, V.nnz, packed, s.stream);
        count_launches(V.nnz ? 1 : 0, "d8 pack4");
        ck(cudaStreamSynchronize(s.stream), "d8 pack4");
        s.free_alloc(codes);
        codes = packed;
      }
      sp.codes = codes;
      sp.rlen = rlen;
      sp.d8_dict_dev = dict_dev;
      ck(cudaStreamSynchronize(s.stream), "d8 encode");
      }
      // packed tiles (one TMA copy per tile: values | codes | row lengths):
      // experiment, C2 27.1 vs 28.1 us but C5 2.36 vs 2.21 ms -> off by default
      bool packed = false;
      if (const char* e = getenv("SPMV_D8_PACKED")) packed = atoi(e) != 0;  // experiments
      if (packed && sp.d8_bits == 8 && V.nnz > 0) {
        std::vector<int64_t> tz((size_t)sp.T + 1), toff((size_t)sp.T + 1);
        ck(cudaMemcpy(tz.data(), sp.tile_nz, (size_t)(sp.T + 1) * 8, cudaMemcpyDeviceToHost), "tile_nz");
        toff[0] = 0;
        for (int64_t k = 0; k < sp.T; ++k) {
          const int64_t cnt = tz[(size_t)k + 1] - tz[(size_t)k];
          const int64_t nr = std::min<int64_t>(Rt, V.m - k * Rt);
          toff[(size_t)k + 1] = toff[(size_t)k] + ((cnt + 1) & ~1ll) * 8 + ((cnt + 15) & ~15ll) + ((nr + 15) & ~15ll);
        }
        int64_t* toff_dev = s.alloc<int64_t>((size_t)sp.T + 1);
        unsigned char* tiles = s.alloc<unsigned char>((size_t)toff[(size_t)sp.T]);
        ck(cudaMemcpyAsync(toff_dev, toff.data(), (size_t)(sp.T + 1) * 8, cudaMemcpyHostToDevice, s.stream), "toff");
        launch_d8_pack_tiles(sp, toff_dev, tiles, s.stream);
        count_launches(1, "d8 pack tiles");
        {
          StreamPlan spc = sp;
          s.val_refresh.push_back([spc, toff_dev, tiles](cudaStream_t st) {
            launch_d8_pack_tiles(spc, toff_dev, tiles, st);
            count_launches(1, "d8 pack tiles");
          });
        }
        ck(cudaStreamSynchronize(s.stream), "d8 pack tiles");
        sp.d8_tiles = tiles;
        sp.d8_toff = toff_dev;
      }
      // consumer warps per CTA (one stage each): the most resident consumer
      // warps per SM (ties: more CTAs), or SPMV_D8_CW
      int best = -1, best_cw = 4;
      for (int c : {4, 6, 8}) {
        if (cw && c != cw) continue;
        if (d8_smem_bytes(sp.C, Rt, c, sp.d8_bits, sp.n_pat_ofs) > 227 * 1024 - kStaticSmemMargin) continue;
        sp.stages = c;
        sp.grid = d8_prepare(sp, s.sm_count);
        if (sp.grid < 0) { cudaGetLastError(); continue; }
        const int per_sm = d8_per_sm(sp);
        if (per_sm * c > best) { best = per_sm * c; best_cw = c; }
      }
      sp.stages = best_cw;
      sp.grid = d8_prepare(sp, s.sm_count);
      if (sp.grid < 0) {
        cudaGetLastError();
        fail(SPMV_E_CUDA, "D8: cannot fit %lld-nonzero tiles in shared memory", (long long)sp.C);
      }
      return;
    }
    // tile size: P whole passes of the consumer warp over its 32/VS rows
    // (row-step mode), the fewest passes giving >= 640 nonzeros -- a tile
    // that ends just short of a pass boundary keeps the lanes busy, and below
    // ~640 nonzeros the per-tile TMA/mbarrier overhead shows (B200 sweeps:
    // 27-nnz rows 768 = 1 pass (896 = 1.04 passes: +21 %); 7-nnz rows 640 =
    // 2.9 passes, 33.1 us vs 36.6 at 512 and 39.3 at 384), clamp [384, 4096];
    // 512 in the segmented mode
    int64_t C = 512;
    if (!seg) {
      const double rows_per_pass = 32.0 / vs;
      C = 0;
      for (int P = 1; P <= 64 && C < 640; ++P) C = (int64_t)(P * rows_per_pass * avg / 128.0) * 128;
      C = std::min<int64_t>(4096, std::max<int64_t>(384, C));
    }
    sp.C = opt.tile_nnz > 0 ? opt.tile_nnz : C;
    P->C = sp.C;
    // row-aligned tiles when the longest row fits twice in a tile: tile k =
    // rows starting in [k*stride, (k+1)*stride), stride = C - maxlen, so no
    // row crosses a tile (no carries, no fix-up kernel)
    // (B200: removes a ~5 us fix-up launch, worth it below ~256M nonzeros;
    // on C5, 1.5G nonzeros, nnz-aligned tiles measured 7% faster)
    sp.aligned = !seg && maxlen >= 0 && 2 * maxlen <= sp.C && V.nnz < ((int64_t)1 << 28) && opt.reserved[0] == 0;
    if (const char* e = getenv("SPMV_ALIGNED"))  // experiments: force row-aligned tiles
      sp.aligned = !seg && maxlen >= 0 && 2 * maxlen <= sp.C && atoi(e) != 0;
    sp.stride = sp.aligned ? sp.C - maxlen : sp.C;
    sp.T = std::max<int64_t>(1, (V.nnz + sp.stride - 1) / sp.stride);
    // row-count tiles for regular short rows (longest <= 1.25 x average + 1):
    // tile k = rows [k*Rt, (k+1)*Rt), Rt = P whole warp passes (the fewest
    // giving >= 576 nonzeros on average), the stage sized for Rt longest rows,
    // so every pass of the consumer warp is full (C2: 96 rows, 3 full passes,
    // vs 91 rows in 2.85 passes with nnz-cut tiles)
    sp.rows_per_tile = 0;
    const bool regular = maxlen > 0 && (double)maxlen <= 1.25 * avg + 1.0;
    // (also above 2^28 nonzeros, unlike the nnz-cut aligned tiles: C5 27-nnz
    // rows, 32-row tiles, no fix-up: 2.890 vs 2.940 ms per step)
    bool rowtiles = !seg && opt.reserved[0] == 0 && regular && opt.tile_nnz <= 0;
    if (const char* e = getenv("SPMV_ROW_TILES")) rowtiles = rowtiles && atoi(e) != 0;  // experiments
    if (rowtiles) {
      const int64_t rpp = 32 / vs;
      int64_t Rt = rpp;
      double min_nz = 576.0;
      if (const char* e = getenv("SPMV_ROW_TILE_MIN_NNZ")) min_nz = atof(e);  // experiments
      while ((double)Rt * avg < min_nz && Rt < 4096) Rt += rpp;
      const int64_t Crt = ((Rt * maxlen + 31) / 32) * 32;  // capacity only (C5: 864 -> 5 CTAs/SM fit)
      if (Crt <= 4096) {
        sp.aligned = true;
        sp.rows_per_tile = Rt;
        sp.C = Crt;
        P->C = sp.C;
        sp.stride = sp.C;
        sp.T = std::max<int64_t>(1, (V.m + Rt - 1) / Rt);
      }
    }
    // staged rowptr entries: 1.5x the expected rows per tile (+32)
    const double rpt = avg > 0 ? (double)sp.C / avg : (double)sp.C;
    sp.rows_cap = (int)std::min<double>((double)sp.C + 32, 1.5 * rpt + 32);
    if (sp.rows_per_tile > 0) sp.rows_cap = (int)sp.rows_per_tile;  // exact
    if (const char* e = getenv("SPMV_ROWS_CAP")) sp.rows_cap = atoi(e);  // tuning knob
    sp.tile_row = s.alloc<int32_t>((size_t)sp.T + 1);
    alloc_carries(s, sp.T, sp.carry_row, sp.carry_val);
    sp.max_run = (std::max<int64_t>(maxlen, P->feat.nnz_max) + sp.stride - 1) / sp.stride + 1;
    DevStats zero{};
    ck(cudaMemcpyAsync(&s.stats->n_incoming, &zero.n_incoming, 8, cudaMemcpyHostToDevice, s.stream), "stats");
    if (sp.rows_per_tile > 0) {
      launch_tile_rows_count(sp.tile_row, sp.T, sp.rows_per_tile, V.m, s.stream);
    } else {
      launch_tile_rows(V, sp.stride, sp.T, sp.tile_row, s.stats, s.stream);
    }
    count_launches(1, "tile_rows");
    if (sp.aligned) {
      sp.tile_nz = s.alloc<int64_t>((size_t)sp.T + 1);
      launch_tile_nz(V, sp.tile_row, sp.T, sp.tile_nz, s.stream);
      count_launches(1, "tile_nz");
    }
    if (d16) {
      uint16_t* dcol = s.alloc<uint16_t>((size_t)V.nnz);
      int32_t* head = s.alloc<int32_t>((size_t)V.m);
      int32_t* anchor = s.alloc<int32_t>((size_t)sp.T);
      int32_t* esc_dev = s.alloc<int32_t>((size_t)kEscMax);
      sp.n_esc = (int)P->esc.size();
      for (int i = 0; i < sp.n_esc; ++i) sp.esc[i] = P->esc[(size_t)i];
      ck(cudaMemcpyAsync(esc_dev, sp.esc, sizeof sp.esc, cudaMemcpyHostToDevice, s.stream), "esc table");
      launch_d16_encode(V, s.headbits, sp.stride, sp.T, dcol, head, anchor, esc_dev, sp.n_esc, s.stream);
      count_launches(3, "d16_encode");
      sp.dcol = dcol;
      sp.head = head;
      sp.anchor = anchor;
    }
    ck(cudaMemcpyAsync(&s.hs, s.stats, sizeof(DevStats), cudaMemcpyDeviceToHost, s.stream), "stats");
    ck(cudaStreamSynchronize(s.stream), "tiles");
    sp.need_fixup = !sp.aligned && s.hs.n_incoming > 0;
    // (the fix-up costs ~81 us per SpMV on C5, its scattered y lines; three
    // in-kernel alternatives were measured slower on B200: a tile-to-tile
    // carry chain that waits (8.0 vs 3.5 ms: a waiting warp holds its stage
    // and the waits line the CTAs up), done-flags with a release fence per
    // tile and opportunistic resolution (6.2 ms: the fence stalls the warp),
    // and keeping the start part out of y (no shorter fix-up))
    // one stage per consumer warp: measured on B200 (tools/sweep.py, C2/C5),
    // more resident warps beat a deeper ring (the x gathers are latency-bound)
    sp.stages = opt.stages > 0 ? opt.stages : kStreamConsumerWarps;
    // 6 consumer warps (one stage each) when 4 such CTAs fit an SM: more
    // bytes in flight for small row-aligned stages (C2: 4 x 6 x 8.8 KB,
    // 31.4 vs 32.5 us; C5's 11.4-KB stages keep 5 CTAs x 4)
    if (opt.stages == 0 && sp.aligned && vs == 1 && !seg && (!d16 || P->esc.empty()) && !getenv("SPMV_NO_CW6")) {
      const size_t sm6 = stream_smem_bytes(sp.C, 6, V.rp_bytes, sp.rows_cap, d16, false);
      if (4 * (sm6 + 1024) <= 228 * 1024) sp.stages = 6;
    }
    if (const char* e = getenv("SPMV_STREAM_L2PF")) sp.l2pf = atoi(e) != 0;
    // shrink the staged-rowptr capacity until the ring fits (sparser tiles
    // then read rowptr from global memory)
    // (227 KB per CTA includes the kernel's static shared memory: ~1 KB)
    while (sp.rows_cap > 64 &&
           stream_smem_bytes(sp.C, sp.stages, V.rp_bytes, sp.rows_cap, d16, seg) > 227 * 1024 - kStaticSmemMargin)
      sp.rows_cap /= 2;
    sp.grid = stream_prepare(sp, s.sm_count);
    if (sp.grid < 0 && sp.stages > kStreamConsumerWarps) {
      cudaGetLastError();
      sp.stages = kStreamConsumerWarps;
      sp.grid = stream_prepare(sp, s.sm_count);
    }
    if (sp.grid < 0) {
      cudaGetLastError();  // (a failed attribute / occupancy query must not poison the next call)
      fail(SPMV_E_CUDA, "cta_stream: cannot fit tile_nnz=%lld in shared memory", (long long)sp.C);
    }
  };
  // nnz_split pass over the view V (colind/values) restricted to the
  // non-empty rows rowmap[0..mc) with rowptr rpc; y rows [0, s.m)
  auto build_nz = [&](Shard& s, NzPlan& z, const MatView& V, const void* rpc, int32_t* rowmap, int64_t mc,
                      int64_t maxlen) {
    z.V = V;
    z.rpc = rpc;
    z.rowmap = rowmap;
    z.mc = mc;
    z.m_out = s.m;
    z.zero_gaps = true;
    z.persistent = P->sel.variant != SPMV_VARIANT_SPLIT;  // SPLIT: shares the SMs with the long-row kernel
    if (const char* e = getenv("SPMV_NZ_PERSIST")) z.persistent = atoi(e) != 0;
    z.T = (V.nnz + kNzTile - 1) / kNzTile;
    z.tile_q = s.alloc<int32_t>((size_t)z.T + 1);
    z.emask = s.alloc<uint32_t>((size_t)std::max<int64_t>(z.T, 1) * 8);
    z.epre = s.alloc<uint64_t>((size_t)std::max<int64_t>(z.T, 1));
    alloc_carries(s, z.T, z.carry_row, z.carry_val);
    z.max_run = maxlen / kNzTile + 2;
    // x gathers through L2 only when sampled neighbouring rows share under
    // half of their x lines and x exceeds 1 MB (B200: C3 283 -> 275 us, C4
    // 126 -> 123 us; stencils as nnz_split lose 3-9 % without L1)
    z.gather_l2 = s.hs.reuse_tot > 0 && 2 * s.hs.reuse_hit < s.hs.reuse_tot && V.n_cols * 8 > (1 << 20);
    if (const char* e = getenv("SPMV_NZ_GATHER_L2")) z.gather_l2 = atoi(e) != 0;
    launch_nz_tiles(z, s.stream);
    count_launches(4, "nz tiles");
    // a very long run of empty rows (> kNzGapMax) would be zeroed by one warp
    // (R-MAT's long rows alone: 2.6 ms instead of ~60 us on B200): clear y
    // before the pass instead and skip the in-kernel gap zeroing
    {
      int32_t* g = s.alloc<int32_t>(1);
      int32_t gmax = 0;
      launch_nz_max_gap(z, g, s.stream);
      count_launches(1, "nz max gap");
      ck(cudaMemcpyAsync(&gmax, g, 4, cudaMemcpyDeviceToHost, s.stream), "max gap");
      ck(cudaStreamSynchronize(s.stream), "max gap");
      z.memset_y = gmax > kNzGapMax;
      if (z.memset_y) z.zero_gaps = false;
    }
    z.grid = nz_prepare(z, s.sm_count);
    if (z.grid < 0) fail(SPMV_E_CUDA, "nnz_split: occupancy query failed");
  };
  // hot-x set of an nnz_split pass over the plan's own colind copy (ML class,
  // P:599-606 re-designed): the most frequent columns (count >= t, first K in
  // column order, K <= kHotMax) are re-encoded as ~slot when they cover >= 20 %
  // of the nonzeros (auto) or when forced (opt.hot_x > 0 = max K)
  auto build_hot = [&](Shard& s, NzPlan& z, const MatView& V, int32_t* col_own) {
    if (opt.hot_x == 0 || V.nnz == 0 || V.n_cols == 0) return;
    int Kmax = opt.hot_x > 0 ? std::min(opt.hot_x, kHotMax) : kHotMax;
    Kmax &= ~1;  // the smem table is bulk-copied in 16-B units
    if (Kmax < 2) return;
    const int64_t nc = V.n_cols, nb = (nc + 1023) / 1024;
    int32_t *cnt = nullptr, *H = nullptr, *bsum = nullptr, *slot = nullptr;
    unsigned long long* cov = nullptr;
    auto cleanup = [&] {
      cudaFree(cnt); cudaFree(H); cudaFree(bsum); cudaFree(slot); cudaFree(cov);
    };
    try {
      ck(cudaMalloc(&cnt, (size_t)nc * 4), "cudaMalloc");
      ck(cudaMalloc(&H, (size_t)kHotBuckets * 4), "cudaMalloc");
      ck(cudaMalloc(&bsum, (size_t)nb * 4 + 4), "cudaMalloc");
      ck(cudaMalloc(&slot, (size_t)nc * 4), "cudaMalloc");
      ck(cudaMalloc(&cov, 8), "cudaMalloc");
      launch_col_counts(V.col, V.nnz, nc, cnt, H, s.stream);
      count_launches(2, "col counts");
      std::vector<int32_t> h(kHotBuckets);
      ck(cudaMemcpyAsync(h.data(), H, (size_t)kHotBuckets * 4, cudaMemcpyDeviceToHost, s.stream), "hist");
      ck(cudaStreamSynchronize(s.stream), "hist");
      // smallest t >= 1 whose columns (count >= t) number <= Kmax; the top
      // bucket (count >= kHotBuckets-1) is taken whole, truncated to Kmax in
      // column order
      int64_t acc = 0;
      int t = kHotBuckets - 1;
      for (int v = kHotBuckets - 1; v >= 1; --v) {
        if (v < kHotBuckets - 1 && acc + h[v] > Kmax) break;
        acc += h[v];
        t = v;
      }
      launch_hot_flags(cnt, nc, t, bsum, s.stream);
      std::vector<int32_t> bs((size_t)nb + 1, 0);
      ck(cudaMemcpyAsync(bs.data(), bsum, (size_t)nb * 4, cudaMemcpyDeviceToHost, s.stream), "hot flags");
      ck(cudaStreamSynchronize(s.stream), "hot flags");
      int64_t tot = 0;
      for (int64_t b = 0; b < nb; ++b) {
        const int32_t c = bs[b];
        bs[b] = (int32_t)std::min<int64_t>(tot, INT32_MAX);
        tot += c;
      }
      const int K = (int)std::min<int64_t>(tot, Kmax) & ~1;
      if (K < 2) { cleanup(); return; }
      ck(cudaMemcpyAsync(bsum, bs.data(), (size_t)nb * 4, cudaMemcpyHostToDevice, s.stream), "hot offsets");
      int32_t* hot_cols = s.alloc<int32_t>((size_t)K);
      launch_hot_write(cnt, nc, t, bsum, K, hot_cols, slot, s.stream);
      count_launches(2, "hot set");
      // coverage = nonzeros in the hot columns
      std::vector<int32_t> hc((size_t)K);
      std::vector<int32_t> cv((size_t)nc);
      ck(cudaMemcpyAsync(hc.data(), hot_cols, (size_t)K * 4, cudaMemcpyDeviceToHost, s.stream), "hot cols");
      ck(cudaMemcpyAsync(cv.data(), cnt, (size_t)nc * 4, cudaMemcpyDeviceToHost, s.stream), "counts");
      ck(cudaStreamSynchronize(s.stream), "hot set");
      int64_t covered = 0;
      for (int k = 0; k < K; ++k) covered += cv[(size_t)hc[k]];
      const bool on = opt.hot_x > 0 || (double)covered >= 0.2 * (double)V.nnz;
      if (on) {
        launch_hot_encode(col_own, V.nnz, slot, s.stream);  // the plan's own colind copy of V
        count_launches(1, "hot encode");
        z.n_hot = K;
        z.hot_cols = hot_cols;
        z.xhot = s.alloc<double>((size_t)K);
        ck(cudaStreamSynchronize(s.stream), "hot encode");
      }
      P->hot_cover = (double)covered / (double)V.nnz;
      cleanup();
    } catch (...) {
      cleanup();
      throw;
    }
  };
  // compacted bin of the rows with lo <= len <= hi (non-empty): cta_stream
  // plan sp, or (nz != null) one nnz_split pass
  auto build_bin = [&](Shard& s, StreamPlan& sp, const MatView& A, int64_t lo, int64_t hi, int vs, bool seg,
                       int64_t* scan, NzPlan* nz = nullptr) -> bool {
    const int64_t nb = scan_blocks(s.m);
    int64_t nrows = 0;
    launch_row_list(A, lo, hi, nullptr, scan, s.stream);  // count
    count_launches(2, "bin count");
    ck(cudaMemcpyAsync(&nrows, scan + nb, 8, cudaMemcpyDeviceToHost, s.stream), "bin count");
    ck(cudaStreamSynchronize(s.stream), "bin count");
    if (nrows == 0) return false;
    int32_t* rows = s.alloc<int32_t>((size_t)nrows + 1);
    launch_row_list(A, lo, hi, rows, scan, s.stream);
    count_launches(3, "bin rows");
    void* frp = s.alloc<char>((size_t)(s.m + 1) * rp_bytes);
    launch_filtered_csr(A, lo, hi, frp, nullptr, nullptr, scan, s.stream);
    count_launches(3, "bin rowptr");
    int64_t bnnz = 0;
    ck(cudaMemcpyAsync(&bnnz, (char*)frp + s.m * rp_bytes, rp_bytes, cudaMemcpyDeviceToHost, s.stream), "bin nnz");
    ck(cudaStreamSynchronize(s.stream), "bin nnz");
    if (rp_bytes == 4) bnnz = (int32_t)bnnz;
    int32_t* bcol = s.alloc<int32_t>((size_t)bnnz);
    double* bval = s.alloc<double>((size_t)bnnz);
    launch_filtered_csr(A, lo, hi, frp, bcol, bval, scan, s.stream);
    count_launches(4, "bin csr");
    s.val_refresh.push_back([A, lo, hi, frp, bval](cudaStream_t st) {
      launch_filtered_vals(A, lo, hi, frp, bval, st);
      count_launches(A.m ? 1 : 0, "bin values");
    });
    void* brp = s.alloc<char>((size_t)(nrows + 1) * rp_bytes);
    launch_gather_rowptr(frp, rp_bytes, rows, nrows, s.m, brp, s.stream);
    count_launches(1, "bin gather");
    if (nz) {
      // (hot-x only when forced: its one 1024-thread CTA per SM leaves no
      // room for the concurrent long-row kernel; measured 554 vs 281 us on C3)
      if (opt.hot_x > 0) build_hot(s, *nz, MatView{rp_bytes, brp, bcol, bval, nrows, s.n_cols, bnnz}, bcol);
      build_nz(s, *nz, MatView{rp_bytes, brp, bcol, bval, nrows, s.n_cols, bnnz}, brp, rows, nrows,
               hi >= P->l_split ? P->feat.max_short : std::min<int64_t>(hi, P->feat.nnz_max));
      nz->skip_rp = A.rowptr;
      return true;
    }
    build_stream(s, sp, MatView{rp_bytes, brp, bcol, bval, nrows, s.n_cols, bnnz}, rows, 0, vs, seg,
                 std::min<int64_t>(hi, P->feat.nnz_max));
    return true;
  };
  for (auto& s : P->shards) {
    ck(cudaSetDevice(s.dev), "cudaSetDevice");
    const MatView A = s.view();
    if (P->sel.variant == SPMV_VARIANT_STREAM) {
      build_stream(s, s.sp[0], A, nullptr, P->sel.d16, P->sel.vs, P->sel.seg != 0, P->feat.nnz_max);
      s.n_sp = 1;
    } else if (P->sel.variant == SPMV_VARIANT_MERGE) {
      s.items = P->items;
      s.Tm = std::max<int64_t>(1, (s.m + s.nnz + s.items - 1) / s.items);
      s.mrow = s.alloc<int32_t>((size_t)s.Tm + 1);
      s.mnnz = s.alloc<int64_t>((size_t)s.Tm + 1);
      alloc_carries(s, s.Tm, s.mcarry_row, s.mcarry_val);
      launch_merge_splits(A, s.items, s.Tm, s.mrow, s.mnnz, s.stream);
      count_launches(1, "merge_splits");
    } else if (P->sel.variant == SPMV_VARIANT_NNZSPLIT) {
      // the non-empty rows of the whole shard (colind / values used in place)
      int64_t* scan = s.alloc<int64_t>((size_t)scan_blocks(s.m) + 2);
      const int64_t nb = scan_blocks(s.m);
      int64_t mc = 0;
      launch_row_list(A, 1, INT64_MAX, nullptr, scan, s.stream);
      count_launches(2, "nz count");
      ck(cudaMemcpyAsync(&mc, scan + nb, 8, cudaMemcpyDeviceToHost, s.stream), "nz count");
      ck(cudaStreamSynchronize(s.stream), "nz count");
      if (s.m == 0) mc = 0;
      int32_t* rows = s.alloc<int32_t>((size_t)mc + 1);
      void* rpc = s.alloc<char>((size_t)(mc + 1) * rp_bytes);
      if (s.m > 0) {
        launch_row_list(A, 1, INT64_MAX, rows, scan, s.stream);
        count_launches(3, "nz rows");
        launch_gather_rowptr(A.rowptr, rp_bytes, rows, mc, s.m, rpc, s.stream);
        count_launches(1, "nz rowptr");
      } else {
        ck(cudaMemsetAsync(rpc, 0, rp_bytes, s.stream), "memset");
      }
      const double th0 = now_ms();
      build_hot(s, s.nz, A, s.col);
      const double th1 = now_ms();
      build_nz(s, s.nz, A, rpc, rows, mc, P->feat.nnz_max);
      if (getenv("SPMV_PLAN_TRACE"))
        fprintf(stderr, "[spmv plan] nz rows %.2f ms, hot set %.2f ms, nz tiles %.2f ms\n", th0 - t_d, th1 - th0,
                now_ms() - th1);
      s.use_nz = true;
    } else if (P->sel.variant == SPMV_VARIANT_SPLIT) {
      // decomposition by row length (Fig. 6 read through S:120-125):
      // short rows (1 <= len <= T_s) and medium rows (T_s < len <= L_split)
      // become compacted CSR bins run by cta_stream (one lane per short row,
      // a 32-lane group per medium row; segmented mode: one bin up to
      // L_split); long rows (len > L_split) become the chunk table; empty rows
      // are covered by clearing y first
      const bool seg = P->sel.seg != 0;
      const int64_t ts = seg ? P->l_split : std::min<int64_t>(kShortRowMax, P->l_split);
      int64_t* scan = s.alloc<int64_t>((size_t)scan_blocks(s.m) + 2);
      s.n_sp = 0;
      if (opt.split_bins != 0) {
        // all rows up to L_split as one nnz_split bin (zeroes empty and long rows;
        // the long-row reduction runs after it)
        s.use_nz = true;
        if (!build_bin(s, s.sp[0], A, 1, P->l_split, 1, false, scan, &s.nz)) {
          s.nz = NzPlan{};
          s.nz.m_out = s.m;
          s.nz.zero_gaps = true;
          s.nz.skip_rp = A.rowptr;  // T == 0: launch_split clears y before the long rows
        }
      } else {
        if (build_bin(s, s.sp[s.n_sp], A, 1, ts, 1, seg, scan)) ++s.n_sp;
        // medium bin lane group: 32, or force_vs when given
        const int mvs = opt.force_vs > 0 ? opt.force_vs : 32;
        if (P->l_split > ts && build_bin(s, s.sp[s.n_sp], A, ts + 1, P->l_split, mvs, false, scan)) ++s.n_sp;
        s.zero_y = true;
      }
      s.n_long = s.hs.n_long;
      if (s.n_long > 0) {
        const int nb = 1024;
        s.long_rows = s.alloc<int32_t>((size_t)s.n_long);
        s.chunk_start = s.alloc<int64_t>((size_t)s.n_long + 1);
        int32_t* scratch = s.alloc<int32_t>((size_t)nb * 4 + 8);
        launch_long_rows(A, P->l_split, P->chunk, s.long_rows, s.n_long, s.chunk_start, scratch, nb, s.stream);
        count_launches(4, "long_rows");
        ck(cudaMemcpyAsync(&s.n_chunks, s.chunk_start + s.n_long, 8, cudaMemcpyDeviceToHost, s.stream), "chunks");
        ck(cudaStreamSynchronize(s.stream), "long_rows");
        alloc_carries(s, s.n_chunks, s.chunk_row, s.chunk_val);
        // column-tiled long rows when a (row, x block) segment averages >= 64
        // nonzeros (dense-ish long rows: x served from smem, not one L2 sector
        // per nonzero); long_mode 1/2 forces chunks / tiled
        const int64_t nblk = (s.n_cols + kLongXB - 1) / kLongXB;
        const bool dense = s.hs.nnz_long >= 64 * s.n_long * nblk;
        s.long_tiled = opt.long_mode >= 2 || (opt.long_mode == 0 && dense);
        if (s.long_tiled) {
          s.nblk = nblk;
          s.long_seg = s.alloc<int64_t>((size_t)s.n_long * (nblk + 1));
          s.long_partial = s.alloc<double>((size_t)s.n_long * nblk);
          launch_long_seg(A, s.long_rows, s.n_long, nblk, s.long_seg, s.stream);
          count_launches(1, "long_seg");
          // the long rows' column indices as 16-bit offsets inside their x
          // block (a segment never leaves its block, so colind mod kLongXB
          // is the whole index): 10 instead of 12 B per long-row nonzero --
          // the paper's MB answer, index compression, on the
          // part it pays for. B200, C4: long rows alone 58.8 -> 53.3 us, C4
          // 111.6 -> 107.1 us. The array spans all nonzeros (indexed like
          // colind; only the long rows' entries are written), so it is built
          // when the long rows hold >= 1/4 of them.
          const char* ec = getenv("SPMV_LONG_C16");
          if (opt.long_mode != 3 && (ec ? atoi(ec) != 0 : 4 * s.hs.nnz_long >= s.nnz)) {
            s.long_c16 = s.alloc<uint16_t>((size_t)std::max<int64_t>(s.nnz, 1));
            launch_long_c16(A, s.long_rows, s.n_long, s.long_c16, s.stream);
            count_launches(1, "long_c16");
          }
          int per_sm = 0;
          if (const char* e = getenv("SPMV_LONG_CTAS")) per_sm = atoi(e);
          s.long_grid = long_tiled_grid(nblk, s.sm_count, per_sm);
          if (const char* e = getenv("SPMV_SPLIT_FUSED")) s.split_fused = atoi(e) != 0;
          // long_mode 3: TMA-staged long rows, one persistent CTA per SM on the
          // side stream next to the short rows' bin (long_tma.cu)
          if (opt.long_mode == 3 && opt.split_bins != 0 &&
              ((uintptr_t)A.col & 15) == 0 && ((uintptr_t)A.val & 15) == 0) {
            if (long_tma_prepare() != 0) ck(cudaGetLastError(), "long_tma smem attribute");
            s.long_tma = true;
            s.long_rg = long_tma_rg(s.n_long, nblk, s.sm_count);
            s.split_fused = false;
          }
        }
        // the long rows run on a side stream, concurrently with the bins
        ck(cudaStreamCreateWithFlags(&s.side, cudaStreamNonBlocking), "cudaStreamCreate");
        ck(cudaEventCreateWithFlags(&s.ev_fork, cudaEventDisableTiming), "cudaEventCreate");
        ck(cudaEventCreateWithFlags(&s.ev_join, cudaEventDisableTiming), "cudaEventCreate");
      }
    }
    s.x = s.alloc<double>((size_t)n_cols);
    s.y = s.alloc<double>((size_t)s.m);
    s.allpart = s.alloc<double>((size_t)2 * kIterRegions * kNormPartials * ngpus);
  }
  // profile-guided mode, second stage (reading 30): when Fig. 4
  // mapped the matrix to the plain cta_stream kernel (CMP: the CSR baseline
  // is latency-bound on a GPU, far from P_MB) and its indices are D8-codable,
  // Fig. 4's MB test is applied to that CMP-optimised kernel: if it reaches
  // (1 - tol) P_MB, the matrix is now bandwidth-bound and Table II's MB
  // optimisation (index compression, D8) is applied jointly
  if (opt.select_mode == 1 && opt.force_classes < 0 && opt.force_variant == 0 && (opt.d16 < 0 || opt.d16 == 2) &&
      P->sel.variant == SPMV_VARIANT_STREAM && P->sel.d16 == 0 && profile_stage2_ok(P->feat, P->sel) &&
      P->pb.p_mb > 0) {
    Shard& s0 = P->shards[0];
    ck(cudaSetDevice(s0.dev), "cudaSetDevice");
    const double t_p = now_ms();
    ck(cudaMemsetAsync(s0.x, 0, (size_t)s0.n_cols * 8, s0.stream), "memset");
    cudaEvent_t e0, e1;
    ck(cudaEventCreate(&e0), "cudaEventCreate");
    ck(cudaEventCreate(&e1), "cudaEventCreate");
    constexpr int kReps = 5;
    for (int r = 0; r < 2; ++r) P->launch(s0, s0.x, s0.y);
    ck(cudaEventRecord(e0, s0.stream), "event");
    for (int r = 0; r < kReps; ++r) P->launch(s0, s0.x, s0.y);
    ck(cudaEventRecord(e1, s0.stream), "event");
    ck(cudaEventSynchronize(e1), "stage-2 probe");
    float ms = 0.f;
    ck(cudaEventElapsedTime(&ms, e0, e1), "event");
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    count_launches(2 + kReps, "stage-2 probe");
    P->pb.p_stream = ms > 0 ? 2.0 * (double)s0.nnz / ((double)ms / kReps * 1e-3) : 0.0;
    const double tol = opt.approx_tol > 0 ? opt.approx_tol : kTolB200;
    if (P->pb.p_stream >= (1.0 - tol) * P->pb.p_mb) {
      P->sel.classes |= SPMV_CLASS_MB;
      P->sel.d16 = 2;
      make_d8dict();
      for (auto& s : P->shards) {  // rebuild the stream structures with D8 codes
        ck(cudaSetDevice(s.dev), "cudaSetDevice");
        ck(cudaStreamSynchronize(s.stream), "stage-2 rebuild");
        s.sp[0] = StreamPlan{};
        build_stream(s, s.sp[0], s.view(), nullptr, 2, 1, false, P->feat.nnz_max);
      }
    }
    P->profile_ms += now_ms() - t_p;
    P->select_ms += now_ms() - t_p;
  }
  for (auto& s : P->shards) {
    ck(cudaStreamSynchronize(s.stream), "structures");
    if (s.headbits) {  // only needed by the inspector
      cudaFree(s.headbits);
      auto it = std::find(s.allocs.begin(), s.allocs.end(), (void*)s.headbits);
      if (it != s.allocs.end()) s.allocs.erase(it);
      s.bytes -= (int64_t)(((size_t)(s.nnz + 31) / 32 + 1) * 4 + 64);
      s.headbits = nullptr;
    }
    // ML analogue: keep x resident in L2 via an access-policy window
    if (P->sel.xwin) {
      ck(cudaSetDevice(s.dev), "cudaSetDevice");
      const size_t xb = (size_t)n_cols * 8;
      const size_t win = std::min<size_t>(xb, (size_t)P->props.access_window_max);
      const size_t persist = std::min<size_t>(win, (size_t)P->props.persisting_l2_max);
      ck(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, persist), "persisting L2 limit");
      {
        std::lock_guard<std::mutex> lk(g_l2_mu);
        if (s.dev >= 0 && s.dev < 64) ++g_l2_plans[s.dev];
        P->l2_limit_set = true;
      }
      cudaStreamAttrValue v;
      memset(&v, 0, sizeof v);
      v.accessPolicyWindow.base_ptr = s.x;
      v.accessPolicyWindow.num_bytes = win;
      v.accessPolicyWindow.hitRatio = win ? std::min(1.0f, (float)persist / (float)win) : 0.f;
      v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
      v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
      ck(cudaStreamSetAttribute(s.stream, cudaStreamAttributeAccessPolicyWindow, &v), "access policy window");
    }
  }
  P->encode_ms = now_ms() - t_d;
  if (getenv("SPMV_PLAN_TRACE"))
    fprintf(stderr, "[spmv plan] x-line reuse %llu / %llu sampled nonzeros, nz gather_l2 %d\n",
            P->shards[0].hs.reuse_hit, P->shards[0].hs.reuse_tot, (int)P->shards[0].nz.gather_l2);
  if (getenv("SPMV_PLAN_TRACE"))
    fprintf(stderr, "[spmv plan] upload %.2f inspect %.2f select %.2f (profile %.2f) encode %.2f ms\n", P->upload_ms,
            P->inspect_ms, P->select_ms, P->profile_ms, P->encode_ms);
  ck(cudaSetDevice(cur), "cudaSetDevice");
  return P.release();
}

template <typename F>
spmv_status guard(F&& f) {
  try {
    f();
    return set_ok();
  } catch (const Err& e) {
    return set_err(e.st, e.what());
  } catch (const std::bad_alloc&) {
    return set_err(SPMV_E_NOMEM, "host allocation failed");
  } catch (const std::exception& e) {
    return set_err(SPMV_E_CUDA, e.what());
  }
}

// ---- pipelined host execute ---------------------------------------------------
// Host x in, host y out through a STREAM plan: the tiles are cut into NB
// blocks; block b's kernel waits only for the x chunk its columns need
// (uploaded in column order on a copy stream), and its finished rows go back
// on a second copy stream while later blocks compute and upload, so the
// PCIe transfers in both directions overlap each other and the SpMV
// (BJ e2e: C5 moves 453 MB each way per step).
int64_t read_rp(const Shard& s, int64_t r) {
  int64_t v = 0;
  if (s.rp_bytes == 8) {
    ck(cudaMemcpy(&v, (const int64_t*)s.rowptr + r, 8, cudaMemcpyDeviceToHost), "rowptr");
  } else {
    int32_t w = 0;
    ck(cudaMemcpy(&w, (const int32_t*)s.rowptr + r, 4, cudaMemcpyDeviceToHost), "rowptr");
    v = w;
  }
  return v;
}

void host_pipe_prepare(spmv_plan p, Shard& s) {
  auto& h = s.hp;
  if (h.ready) return;
  h.ready = true;
  const StreamPlan& sp = s.sp[0];
  const int64_t xbytes = p->n_cols * 8;
  // (segmented-mode tiles assign a row where it ENDS and add the carries after:
  // a later range would overwrite an earlier range's fix-up, so not pipelined)
  int64_t min_bytes = 16ll << 20;
  if (const char* e = getenv("SPMV_HOST_PIPE_MIN_BYTES")) min_bytes = atoll(e);  // tests: pipeline small plans
  if (p->sel.variant == SPMV_VARIANT_NNZSPLIT && s.use_nz && !s.nz.skip_rp && xbytes >= min_bytes && s.m > 0) {
    // nnz_split: the x gather is random, so the whole column range goes up
    // first; the ranges then overlap the download of y. A row is assigned by
    // the tile where it ends and range b's carries are added after range
    // b+1, so a range must be longer than any row (rows span <= 2 ranges).
    const NzPlan& z = s.nz;
    int64_t nbw = std::min<int64_t>(8, std::max<int64_t>(2, (int64_t)s.m * 8 / (4ll << 20)));
    if (const char* e = getenv("SPMV_HOST_PIPE_BLOCKS")) nbw = atoll(e);  // tests
    const int nb = (int)std::max<int64_t>(1, std::min<int64_t>(nbw, z.T / std::max<int64_t>(2 * z.max_run, 8)));
    if (nb < 2) return;
    h.nz = true;
    h.kb.resize(nb + 1);
    h.srow.resize(nb + 1);
    h.xhi.assign(nb, s.hs.col_max + 1);
    h.xlo = std::min<int64_t>(std::max<long long>(0, s.hs.col_min), s.hs.col_max + 1);
    for (int b = 0; b <= nb; ++b) h.kb[b] = z.T * b / nb;
    h.srow[0] = 0;
    h.srow[nb] = s.m;
    for (int b = 1; b < nb; ++b) {  // first row ending in range b: rowmap[tile_q[kb]]
      int32_t q = 0, r = 0;
      ck(cudaMemcpy(&q, z.tile_q + h.kb[b], 4, cudaMemcpyDeviceToHost), "tile_q");
      ck(cudaMemcpy(&r, z.rowmap + q, 4, cudaMemcpyDeviceToHost), "rowmap");
      h.srow[b] = r;
    }
    ck(cudaStreamCreateWithFlags(&h.h2d, cudaStreamNonBlocking), "cudaStreamCreate");
    ck(cudaStreamCreateWithFlags(&h.d2h, cudaStreamNonBlocking), "cudaStreamCreate");
    h.ev_h.resize(nb);
    h.ev_c.resize(nb);
    for (int b = 0; b < nb; ++b) {
      ck(cudaEventCreateWithFlags(&h.ev_h[b], cudaEventDisableTiming), "cudaEventCreate");
      ck(cudaEventCreateWithFlags(&h.ev_c[b], cudaEventDisableTiming), "cudaEventCreate");
    }
    h.usable = true;
    return;
  }
  if (p->sel.variant != SPMV_VARIANT_STREAM || sp.rowmap || sp.seg || sp.T < 8 || xbytes < min_bytes || s.m == 0)
    return;
  // blocks: one per ~4 MB of x, 2..16 (B200 sweeps: C2 16.8 MB -> 4 blocks
  // 0.655 ms vs 0.677 (2) / 0.773 (8); C5 453 MB -> 16 blocks 11.07 ms vs
  // 11.37 (8) / 11.25 (24))
  int64_t nbw = std::min<int64_t>(16, std::max<int64_t>(2, xbytes / (4ll << 20)));
  if (const char* e = getenv("SPMV_HOST_PIPE_BLOCKS")) nbw = atoll(e);  // tests
  int nb = (int)std::max<int64_t>(2, std::min<int64_t>(nbw, sp.T / 4));
  // tapered blocks (experiment, SPMV_HOST_PIPE_TAPER=t): the first t and the
  // last t blocks a quarter of the others -- measured slower on C5 (11.07 vs
  // 10.4-10.5 ms per e2e step), so off by default
  int taper = 0;
  if (const char* e = getenv("SPMV_HOST_PIPE_TAPER")) taper = std::min(atoi(e), nb / 4);  // experiments
  if (taper > 0) nb += 2 * taper;
  h.kb.resize(nb + 1);
  h.srow.resize(nb + 1);
  h.xhi.resize(nb);
  {
    // block weights: 1 in the middle, 1/4 for the `taper` blocks at each end
    std::vector<double> cw((size_t)nb + 1, 0.0);
    for (int b = 0; b < nb; ++b) cw[(size_t)b + 1] = cw[(size_t)b] + ((b < taper || b >= nb - taper) ? 0.25 : 1.0);
    for (int b = 0; b <= nb; ++b) h.kb[b] = b == nb ? sp.T : (int64_t)((double)sp.T * cw[(size_t)b] / cw[(size_t)nb]);
  }
  std::vector<int64_t> t0(nb + 1);
  int32_t* cm = nullptr;
  ck(cudaMalloc(&cm, 4 * (size_t)nb), "cudaMalloc");
  try {
    ck(cudaMemsetAsync(cm, 0xff, 4 * (size_t)nb, s.stream), "memset");
    for (int b = 0; b <= nb; ++b) {
      const int64_t k = h.kb[b];
      if (sp.aligned) {
        ck(cudaMemcpy(&t0[b], sp.tile_nz + k, 8, cudaMemcpyDeviceToHost), "tile_nz");
      } else {
        t0[b] = std::min<int64_t>(k * sp.stride, s.nnz);
      }
      if (b == 0) { h.srow[b] = 0; continue; }
      if (b == nb) { h.srow[b] = s.m; continue; }
      int32_t R = 0;
      ck(cudaMemcpy(&R, sp.tile_row + k, 4, cudaMemcpyDeviceToHost), "tile_row");
      const bool incoming = !sp.aligned && R > 0 && read_rp(s, R) > t0[b];
      h.srow[b] = R - (incoming ? 1 : 0);
    }
    for (int b = 0; b < nb; ++b) launch_range_colmax(s.col, t0[b], t0[b + 1], cm + b, s.stream);
    std::vector<int32_t> mx(nb);
    ck(cudaMemcpyAsync(mx.data(), cm, 4 * (size_t)nb, cudaMemcpyDeviceToHost, s.stream), "colmax");
    ck(cudaStreamSynchronize(s.stream), "colmax");
    // x is uploaded from the shard's first read column (a row block of a
    // banded matrix reads only its halo range: 1/G of x at G shards)
    const int64_t c_lo = std::max<long long>(0, s.hs.col_min), c_hi = s.hs.col_max + 1;
    h.xlo = std::min<int64_t>(c_lo, c_hi);
    int64_t hi = h.xlo;
    for (int b = 0; b < nb; ++b) {
      hi = std::max<int64_t>(hi, (int64_t)mx[b] + 1);
      h.xhi[b] = b == nb - 1 ? c_hi : std::min<int64_t>(hi, c_hi);
    }
    cudaFree(cm);
  } catch (...) {
    cudaFree(cm);
    throw;
  }
  ck(cudaStreamCreateWithFlags(&h.h2d, cudaStreamNonBlocking), "cudaStreamCreate");
  ck(cudaStreamCreateWithFlags(&h.d2h, cudaStreamNonBlocking), "cudaStreamCreate");
  // (experiment, SPMV_HOST_PIPE_TWO_STREAMS=1: measured slower on C5, 12.9 vs
  // 10.4 ms per e2e step -- the two H2D streams starve the D2H direction)
  if (getenv("SPMV_HOST_PIPE_TWO_STREAMS")) {
    ck(cudaStreamCreateWithFlags(&h.h2d2, cudaStreamNonBlocking), "cudaStreamCreate");
    ck(cudaStreamCreateWithFlags(&h.d2h2, cudaStreamNonBlocking), "cudaStreamCreate");
    ck(cudaEventCreateWithFlags(&h.ev_e2, cudaEventDisableTiming), "cudaEventCreate");
  }
  h.ev_h.resize(nb);
  h.ev_c.resize(nb);
  for (int b = 0; b < nb; ++b) {
    ck(cudaEventCreateWithFlags(&h.ev_h[b], cudaEventDisableTiming), "cudaEventCreate");
    ck(cudaEventCreateWithFlags(&h.ev_c[b], cudaEventDisableTiming), "cudaEventCreate");
  }
  h.usable = true;
}

// nnz_split ranges: K(0), then K(b), F(b-1), copy of range b-1's rows, ...
int host_pipe_run_nz(Shard& s, const double* x, double* y) {
  auto& h = s.hp;
  const NzPlan& z = s.nz;
  const int nb = (int)h.xhi.size();
  int n = 0;
  ck(cudaEventRecord(h.ev_c[0], s.stream), "event");
  ck(cudaStreamWaitEvent(h.h2d, h.ev_c[0], 0), "wait");
  ck(cudaStreamWaitEvent(h.d2h, h.ev_c[0], 0), "wait");
  if (h.xhi[0] > h.xlo)
    ck(cudaMemcpyAsync(s.x + h.xlo, x + h.xlo, (size_t)(h.xhi[0] - h.xlo) * 8, cudaMemcpyHostToDevice, h.h2d),
       "copy x");
  ck(cudaEventRecord(h.ev_h[0], h.h2d), "event");
  ck(cudaStreamWaitEvent(s.stream, h.ev_h[0], 0), "wait");
  n += launch_nz_prologue(z, s.x, s.y, s.stream);
  n += launch_nz_range(z, s.x, s.y, h.kb[0], h.kb[1], s.stream);
  for (int b = 0; b < nb; ++b) {
    if (b + 1 < nb) n += launch_nz_range(z, s.x, s.y, h.kb[b + 1], h.kb[b + 2], s.stream);
    n += launch_nz_fixup_range(z, s.y, h.kb[b], h.kb[b + 1], s.stream);
    ck(cudaEventRecord(h.ev_c[b], s.stream), "event");
    ck(cudaStreamWaitEvent(h.d2h, h.ev_c[b], 0), "wait");
    const int64_t r0 = h.srow[b], r1 = h.srow[b + 1];
    if (r1 > r0)
      ck(cudaMemcpyAsync(y + s.row0 + r0, s.y + r0, (size_t)(r1 - r0) * 8, cudaMemcpyDeviceToHost, h.d2h), "copy y");
  }
  ck(cudaEventRecord(h.ev_h[0], h.d2h), "event");
  ck(cudaStreamWaitEvent(s.stream, h.ev_h[0], 0), "wait");
  return n;
}

// enqueue the pipelined SpMV of shard s (x, y host); returns launches
int host_pipe_run(spmv_plan p, Shard& s, const double* x, double* y) {
  auto& h = s.hp;
  if (h.nz) return host_pipe_run_nz(s, x, y);
  const int nb = (int)h.xhi.size();
  int n = 0;
  const bool two = h.h2d2 != nullptr;
  auto up = [&](int b) { return (two && (b & 1)) ? h.h2d2 : h.h2d; };
  auto down = [&](int b) { return (two && (b & 1)) ? h.d2h2 : h.d2h; };
  ck(cudaEventRecord(h.ev_c[0], s.stream), "event");  // copies start after earlier work on the plan stream
  ck(cudaStreamWaitEvent(h.h2d, h.ev_c[0], 0), "wait");
  ck(cudaStreamWaitEvent(h.d2h, h.ev_c[0], 0), "wait");
  if (two) {
    ck(cudaStreamWaitEvent(h.h2d2, h.ev_c[0], 0), "wait");
    ck(cudaStreamWaitEvent(h.d2h2, h.ev_c[0], 0), "wait");
  }
  int64_t lo = h.xlo;
  for (int b = 0; b < nb; ++b) {
    if (h.xhi[b] > lo)
      ck(cudaMemcpyAsync(s.x + lo, x + lo, (size_t)(h.xhi[b] - lo) * 8, cudaMemcpyHostToDevice, up(b)), "copy x");
    lo = std::max(lo, h.xhi[b]);
    ck(cudaEventRecord(h.ev_h[b], up(b)), "event");
  }
  for (int b = 0; b < nb; ++b) {
    // block b needs every x chunk <= b (column order): chunk b-1 may sit on
    // the other copy stream
    ck(cudaStreamWaitEvent(s.stream, h.ev_h[b], 0), "wait");
    if (two && b > 0) ck(cudaStreamWaitEvent(s.stream, h.ev_h[b - 1], 0), "wait");
    n += launch_stream_range(s.sp[0], s.x, s.y, h.kb[b], h.kb[b + 1], s.stream);
    ck(cudaEventRecord(h.ev_c[b], s.stream), "event");
    ck(cudaStreamWaitEvent(down(b), h.ev_c[b], 0), "wait");
    const int64_t r0 = h.srow[b], r1 = h.srow[b + 1];
    if (r1 > r0)
      ck(cudaMemcpyAsync(y + s.row0 + r0, s.y + r0, (size_t)(r1 - r0) * 8, cudaMemcpyDeviceToHost, down(b)),
         "copy y");
  }
  // the plan stream resumes after the last copies
  ck(cudaEventRecord(h.ev_h[0], h.d2h), "event");
  ck(cudaStreamWaitEvent(s.stream, h.ev_h[0], 0), "wait");
  if (two) {
    ck(cudaEventRecord(h.ev_e2, h.d2h2), "event");
    ck(cudaStreamWaitEvent(s.stream, h.ev_e2, 0), "wait");
  }
  (void)p;
  return n;
}

// the async entry points take device pointers of the shard's device only (a
// host pointer would fault inside the kernel instead of returning an error)
void require_dev(const Shard& s, const void* p, const char* what) {
  int dev = -1;
  if (!is_device_ptr(p, &dev) || dev != s.dev)
    fail(SPMV_E_ARG, "%s must be a device pointer of device %d on the asynchronous path", what, s.dev);
}

// run the plan on x (device pointer valid on every shard's device or the
// shards' replicas) into y (per-shard outputs)
void execute_impl(spmv_plan p, const double* x, double* y, bool sync) {
  if (!p || !x || !y) fail(SPMV_E_ARG, "null argument");
  int xdev = -1, ydev = -1;
  const bool xd = is_device_ptr(x, &xdev), yd = is_device_ptr(y, &ydev);
  int cur = 0;
  cudaGetDevice(&cur);
  if (!xd && !yd && !getenv("SPMV_NO_HOST_PIPE")) {
    bool all = true;
    for (auto& s : p->shards) {
      ck(cudaSetDevice(s.dev), "cudaSetDevice");
      host_pipe_prepare(p, s);
      all = all && s.hp.usable;
    }
    if (all) {
      for (auto& s : p->shards) {
        ck(cudaSetDevice(s.dev), "cudaSetDevice");
        count_launches(host_pipe_run(p, s, x, y), "spmv");
      }
      if (sync)
        for (auto& s : p->shards) ck(cudaStreamSynchronize(s.stream), "spmv sync");
      cudaSetDevice(cur);
      return;
    }
  }
  for (auto& s : p->shards) {
    ck(cudaSetDevice(s.dev), "cudaSetDevice");
    const double* xs = x;
    if (!(xd && xdev == s.dev)) {
      // only the column range the shard reads (include/spmv.h, x_device)
      const int64_t lo = std::max<long long>(0, s.hs.col_min), hi = s.hs.col_max + 1;
      if (x != s.x && hi > lo)
        ck(cudaMemcpyAsync(s.x + lo, x + lo, (size_t)(hi - lo) * 8, cudaMemcpyDefault, s.stream), "copy x");
      xs = s.x;
    }
    double* ys = y + s.row0;
    const bool direct = yd && ydev == s.dev;
    if (!direct) ys = s.y;
    count_launches(p->launch(s, xs, ys), "spmv");
    if (!direct) ck(cudaMemcpyAsync(y + s.row0, s.y, (size_t)s.m * 8, cudaMemcpyDefault, s.stream), "copy y");
  }
  if (sync)
    for (auto& s : p->shards) ck(cudaStreamSynchronize(s.stream), "spmv sync");
  cudaSetDevice(cur);
}

}  // namespace

// ============================================================================
// C ABI
// ============================================================================
extern "C" {

void spmv_options_default(spmv_options* o) {
  if (!o) return;
  memset(o, 0, sizeof *o);
  o->struct_size = (int32_t)sizeof(spmv_options);
  o->d16 = -1;
  o->xwin = -1;
  o->seg = -1;
  o->split_bins = -1;
  o->hot_x = -1;
  o->validate = 1;
  o->force_classes = -1;
}

spmv_plan spmv_plan_create(int64_t n, int64_t nnz, const int64_t* rowptr, const int32_t* colind,
                           const double* values, int ngpus) {
  spmv_plan out = nullptr;
  spmv_plan_create_ex(&out, n, n, nnz, rowptr, 8, colind, values, ngpus, nullptr);
  return out;
}

spmv_status spmv_plan_create_ex(spmv_plan* out, int64_t n_rows, int64_t n_cols, int64_t nnz, const void* rowptr,
                                int rowptr_bytes, const int32_t* colind, const double* values, int ngpus,
                                const spmv_options* opt) {
  if (!out) return set_err(SPMV_E_ARG, "out is NULL");
  *out = nullptr;
  return guard([&] { *out = create_impl(n_rows, n_cols, nnz, rowptr, rowptr_bytes, colind, values, ngpus, opt); });
}

void spmv_plan_destroy(spmv_plan p) { delete p; }

int spmv_execute(spmv_plan p, const double* x, double* y) {
  return guard([&] { execute_impl(p, x, y, true); });
}

int spmv_execute_async(spmv_plan p, const double* x, double* y) { return spmv_execute_stage(p, x, y, 0); }

int spmv_execute_stage(spmv_plan p, const double* x, double* y, int stage) {
  return guard([&] {
    if (!p || !x || !y || stage < 0 || stage > 2) fail(SPMV_E_ARG, "bad argument");
    if (p->shards.size() != 1) fail(SPMV_E_ARG, "spmv_execute_async/_stage need a single-shard plan");
    Shard& s = p->shards[0];
    require_dev(s, x, "x");
    require_dev(s, y, "y");
    count_launches(p->launch(s, x, y, stage), "spmv");
  });
}

int32_t spmv_norm_partial_count(void) { return kNormPartials; }

int spmv_norm_partials(spmv_plan p, const double* y, double* partials) {
  return guard([&] {
    if (!p || !y || !partials || p->shards.size() != 1) fail(SPMV_E_ARG, "bad argument");
    Shard& s = p->shards[0];
    count_launches(launch_norm_partials(y, s.m, partials, s.stream), "norm_partials");
  });
}

int spmv_normalize(spmv_plan p, const double* y, const double* partials, int count, double* x_out, double* nu_dev) {
  return guard([&] {
    if (!p || !y || !partials || !x_out || count < 1 || p->shards.size() != 1) fail(SPMV_E_ARG, "bad argument");
    Shard& s = p->shards[0];
    count_launches(launch_normalize(y, s.m, partials, count, x_out, nu_dev, s.stream), "normalize");
  });
}

int spmv_norm_step(spmv_plan p, const double* partials, int count, double* nn, double* nu_k) {
  return guard([&] {
    if (!p || !partials || !nn || !nu_k || count < 1 || p->shards.size() != 1) fail(SPMV_E_ARG, "bad argument");
    Shard& s = p->shards[0];
    count_launches(launch_norm_step(partials, count, nn, nu_k, s.stream), "norm step");
  });
}

int spmv_unit(spmv_plan p, const double* y, int64_t n, const double* nn, double* x_out) {
  return guard([&] {
    if (!p || !y || !nn || !x_out || n < 0 || p->shards.size() != 1) fail(SPMV_E_ARG, "bad argument");
    Shard& s = p->shards[0];
    count_launches(launch_unit(y, n, nn, x_out, s.stream), "unit");
  });
}

namespace {
// One iteration's SpMV on shard s (iterfuse.cuh): y = f * (A x) with f the
// pending exact rescale nn[1] of the previous step (nn null: f = 1), the
// kNormPartials partials of y^2 and, when nu_k is given (single rank: the
// partials are all of them), the norm step. Row-aligned STREAM / D8 plans do
// all of it inside the SpMV kernel (its last CTA folds the partials and runs
// the norm step): one launch per iteration. Other variants: the SpMV, one
// scale + partials pass over y, the norm-step kernel.
int spmv_iter(const spmv_plan_s* P, Shard& s, const double* x, double* y, double* partials, double* nn,
              double* nu_k, const IterOut* push = nullptr) {
  const StreamPlan& sp = s.sp[0];
  if (P->sel.variant == SPMV_VARIANT_STREAM && sp.aligned && !sp.seg && !sp.rowmap && !sp.need_fixup &&
      !getenv("SPMV_NO_FUSED_NORM")) {
    if (!s.cta_part) {
      s.cta_part = s.alloc<double>((size_t)std::max(sp.grid, 1));
      s.done = s.alloc<unsigned int>(1);
      ck(cudaMemsetAsync(s.done, 0, sizeof(unsigned int), s.stream), "memset");
    }
    IterOut it;
    it.scale = nn ? nn + 1 : nullptr;
    it.cta_part = s.cta_part;
    it.done = s.done;
    it.partials = partials;
    it.nn = nu_k ? nn : nullptr;
    it.nu_k = nu_k;
    if (push) {
      it.push_lo = push->push_lo;
      it.push_lo_end = push->push_lo_end;
      it.push_hi = push->push_hi;
      it.push_hi_begin = push->push_hi_begin;
    }
    return launch_stream_iter(sp, x, y, it, s.stream);
  }
  int n = P->launch(s, x, y);
  n += launch_scale_partials(y, s.m, nn, partials, s.stream);
  if (nu_k) n += launch_norm_step(partials, kNormPartials, nn, nu_k, s.stream);
  return n;
}

// tiles [k0, k1) of a fused-capable plan with the iteration epilogue (partials
// of this launch only; the pending rescale nn[1] applied; no norm step)
int spmv_iter_range(const spmv_plan_s* P, Shard& s, const double* x, double* y, double* partials, double* nn,
                    int64_t k0, int64_t k1) {
  if (k1 <= k0) {
    ck(cudaMemsetAsync(partials, 0, kNormPartials * 8, s.stream), "memset");
    return 0;
  }
  (void)P;
  if (!s.cta_part) {
    s.cta_part = s.alloc<double>((size_t)std::max(s.sp[0].grid, 1));
    s.done = s.alloc<unsigned int>(1);
    ck(cudaMemsetAsync(s.done, 0, sizeof(unsigned int), s.stream), "memset");
  }
  IterOut it;
  it.scale = nn + 1;
  it.cta_part = s.cta_part;
  it.done = s.done;
  it.partials = partials;
  return launch_stream_iter_range(s.sp[0], x, y, it, k0, k1, s.stream);
}

// interior tile range of shard s: tiles whose nonzeros read only x[row0,
// row0 + m) (its own block). Banded row blocks: one contiguous range between
// the tiles reading the lower and the upper halo. Used when it is at least a
// quarter of the tiles.
void prepare_overlap(const spmv_plan_s* P, Shard& s) {
  if (s.ovl_ready) return;
  s.ovl_ready = true;
  const StreamPlan& sp = s.sp[0];
  const bool fused = P->sel.variant == SPMV_VARIANT_STREAM && sp.aligned && !sp.seg && !sp.rowmap &&
                     !sp.need_fixup && sp.tile_nz && !getenv("SPMV_NO_FUSED_NORM") && !getenv("SPMV_NO_OVERLAP");
  ck(cudaSetDevice(s.dev), "cudaSetDevice");
  ck(cudaStreamCreateWithFlags(&s.cp, cudaStreamNonBlocking), "cudaStreamCreate");
  ck(cudaEventCreateWithFlags(&s.ev_cp, cudaEventDisableTiming), "cudaEventCreate");
  if (!fused || s.nnz == 0 || sp.T < 8) return;
  unsigned long long* ext = s.alloc<unsigned long long>(2);
  unsigned long long h[2] = {0ull, (unsigned long long)s.nnz};
  ck(cudaMemcpyAsync(ext, h, 16, cudaMemcpyHostToDevice, s.stream), "halo extent");
  launch_halo_extent(s.col, s.nnz, s.row0, s.row0 + s.m, ext, s.stream);
  count_launches(1, "halo extent");
  std::vector<int64_t> tz((size_t)sp.T + 1);
  ck(cudaMemcpyAsync(h, ext, 16, cudaMemcpyDeviceToHost, s.stream), "halo extent");
  ck(cudaMemcpyAsync(tz.data(), sp.tile_nz, (size_t)(sp.T + 1) * 8, cudaMemcpyDeviceToHost, s.stream), "tile_nz");
  ck(cudaStreamSynchronize(s.stream), "halo extent");
  // tile holding nonzero j: the largest k with tz[k] <= j
  auto tile_of = [&](int64_t j) { return (int64_t)(std::upper_bound(tz.begin(), tz.end() - 1, j) - tz.begin()) - 1; };
  const int64_t kb = h[0] == 0 ? 0 : tile_of((int64_t)h[0] - 1) + 1;
  const int64_t ke = h[1] >= (unsigned long long)s.nnz ? sp.T : tile_of((int64_t)h[1]);
  if (ke - kb >= sp.T / 4) {
    s.ovl = true;
    s.kb = kb;
    s.ke = ke;
  }
}

// Halo push (the exchange fused into the SpMV): usable when
// every shard runs the fused-capable kernel and the rows each peer reads from
// a shard form a prefix of its block (one lower neighbour) and/or a suffix
// (one upper neighbour) -- banded row blocks -- and, across devices, the
// writer has peer access to the reader. Then shard g's kernel stores those
// rows of yh_k into the neighbours' next replicas as it writes them and the
// separate halo copies disappear.
bool prepare_push(spmv_plan_s* P) {
  if (P->push_ready) return P->push_ok;
  P->push_ready = true;
  P->push_ok = false;
  const int G = (int)P->shards.size();
  if (G < 2 || getenv("SPMV_NO_PUSH")) return false;
  for (auto& s : P->shards) {
    const StreamPlan& sp = s.sp[0];
    if (!(P->sel.variant == SPMV_VARIANT_STREAM && sp.aligned && !sp.seg && !sp.rowmap && !sp.need_fixup &&
          stream_push_capable(sp)))
      return false;
    s.push_lo_peer = s.push_hi_peer = -1;
  }
  for (int g = 0; g < G; ++g) {
    Shard& s = P->shards[g];
    for (int h = 0; h < G; ++h) {
      if (h == g) continue;
      const Shard& t = P->shards[h];
      if (t.hs.col_min > t.hs.col_max) continue;  // reads nothing
      const int64_t a = std::max<int64_t>(t.hs.col_min, s.row0), b = std::min<int64_t>(t.hs.col_max + 1, s.row0 + s.m);
      if (a >= b) continue;
      if (s.dev != t.dev) {
        int can = 0;
        if (cudaDeviceCanAccessPeer(&can, s.dev, t.dev) != cudaSuccess || !can) return false;
      }
      if (h < g) {
        if (s.push_lo_peer >= 0 || a != s.row0) return false;
        s.push_lo_peer = h;
        s.push_lo_end = b - s.row0;
      } else {
        if (s.push_hi_peer >= 0 || b != s.row0 + s.m) return false;
        s.push_hi_peer = h;
        s.push_hi_begin = a - s.row0;
      }
    }
  }
  cudaGetLastError();
  P->push_ok = true;
  return true;
}

// ML x-window on the replica the next SpMV reads (the iterate ping-pongs)
void set_xwin(const spmv_plan_s* P, Shard& s, const double* base) {
  if (!P->sel.xwin) return;
  const size_t xb = (size_t)s.n_cols * 8;
  const size_t win = std::min<size_t>(xb, (size_t)P->props.access_window_max);
  const size_t persist = std::min<size_t>(win, (size_t)P->props.persisting_l2_max);
  cudaStreamAttrValue v;
  memset(&v, 0, sizeof v);
  v.accessPolicyWindow.base_ptr = const_cast<double*>(base);
  v.accessPolicyWindow.num_bytes = win;
  v.accessPolicyWindow.hitRatio = win ? std::min(1.0f, (float)persist / (float)win) : 0.f;
  v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
  v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
  ck(cudaStreamSetAttribute(s.stream, cudaStreamAttributeAccessPolicyWindow, &v), "access policy window");
}
}  // namespace

int spmv_execute_norm(spmv_plan p, const double* x, double* y, double* partials) {
  return guard([&] {
    if (!p || !x || !y || !partials || p->shards.size() != 1) fail(SPMV_E_ARG, "bad argument");
    Shard& s = p->shards[0];
    require_dev(s, x, "x");
    require_dev(s, y, "y");
    require_dev(s, partials, "partials");
    count_launches(spmv_iter(p, s, x, y, partials, nullptr, nullptr), "spmv + norm partials");
  });
}

int spmv_iter_step(spmv_plan p, const double* x, double* y, double* partials, double* nn, double* nu_k) {
  return guard([&] {
    if (!p || !x || !y || !partials || !nn || p->shards.size() != 1) fail(SPMV_E_ARG, "bad argument");
    Shard& s = p->shards[0];
    require_dev(s, x, "x");
    require_dev(s, y, "y");
    require_dev(s, partials, "partials");
    require_dev(s, nn, "nn");
    if (nu_k) require_dev(s, nu_k, "nu_k");
    count_launches(spmv_iter(p, s, x, y, partials, nn, nu_k), "iteration step");
  });
}

// ---- halo push across processes (one process per GPU; include/spmv.h) ----

int spmv_plan_replicas(spmv_plan p, double** x_a, double** x_b) {
  return guard([&] {
    if (!p || !x_a || !x_b || p->shards.size() != 1) fail(SPMV_E_ARG, "bad argument");
    Shard& s = p->shards[0];
    ck(cudaSetDevice(s.dev), "cudaSetDevice");
    if (!s.x2) s.x2 = s.alloc<double>((size_t)p->n_cols);
    *x_a = s.x;
    *x_b = s.x2;
  });
}

int spmv_iter_push_capable(spmv_plan p) {
  if (!p || p->shards.size() != 1) return 0;
  const StreamPlan& sp = p->shards[0].sp[0];
  return (p->sel.variant == SPMV_VARIANT_STREAM && sp.aligned && !sp.seg && !sp.rowmap && !sp.need_fixup &&
          stream_push_capable(sp) && !getenv("SPMV_NO_FUSED_NORM"))
             ? 1
             : 0;
}

int spmv_ipc_export(spmv_plan p, const double* replica, void* handle) {
  return guard([&] {
    if (!p || !replica || !handle || p->shards.size() != 1) fail(SPMV_E_ARG, "bad argument");
    Shard& s = p->shards[0];
    if (replica != s.x && replica != s.x2) fail(SPMV_E_ARG, "not a replica of this plan (spmv_plan_replicas)");
    ck(cudaSetDevice(s.dev), "cudaSetDevice");
    cudaIpcMemHandle_t h;
    ck(cudaIpcGetMemHandle(&h, const_cast<double*>(replica)), "cudaIpcGetMemHandle");
    static_assert(sizeof(h) == SPMV_IPC_HANDLE_BYTES, "IPC handle size");
    memcpy(handle, &h, sizeof h);
  });
}

int spmv_ipc_open(spmv_plan p, const void* handle, double** ptr) {
  return guard([&] {
    if (!p || !handle || !ptr || p->shards.size() != 1) fail(SPMV_E_ARG, "bad argument");
    Shard& s = p->shards[0];
    ck(cudaSetDevice(s.dev), "cudaSetDevice");
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof h);
    void* d = nullptr;
    ck(cudaIpcOpenMemHandle(&d, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
    s.ipc_open.push_back(d);
    *ptr = static_cast<double*>(d);
  });
}

int spmv_iter_step_push(spmv_plan p, const double* x, double* y, double* partials, double* nn, double* push_lo,
                        int64_t push_lo_end, double* push_hi, int64_t push_hi_begin) {
  return guard([&] {
    if (!p || !x || !y || !partials || !nn || p->shards.size() != 1) fail(SPMV_E_ARG, "bad argument");
    Shard& s = p->shards[0];
    if (push_lo_end < 0 || push_lo_end > s.m || push_hi_begin < 0 || push_hi_begin > s.m ||
        (push_lo && push_lo_end == 0) || (push_hi && push_hi_begin == s.m))
      fail(SPMV_E_ARG, "push row ranges outside the block");
    if (!spmv_iter_push_capable(p)) fail(SPMV_E_UNSUPPORTED, "the plan's kernel has no halo-push instantiation");
    require_dev(s, x, "x");
    require_dev(s, y, "y");
    require_dev(s, partials, "partials");
    require_dev(s, nn, "nn");
    IterOut po;
    po.push_lo = push_lo;
    po.push_lo_end = push_lo ? push_lo_end : 0;
    po.push_hi = push_hi;
    po.push_hi_begin = push_hi ? push_hi_begin : s.m;
    count_launches(spmv_iter(p, s, x, y, partials, nn, nullptr, &po), "iteration step (push)");
  });
}

// Deferred normalisation (norm.cu, reading 25): iteration k runs
// the SpMV on replica `cur` (x_0, then yh_{k-1}) and writes yh_k straight into
// the shard's block of replica `nxt`; the norm partials, the rank-ordered
// norm step (nu_k = ||yh_k|| / ||yh_{k-1}||, exact power-of-two rescale when
// the magnitude drifts) and the halo exchange of `nxt` follow; no x = y/nu
// pass per iteration. x_iters = yh_{iters-1} / ||yh_{iters-1}|| at the end.
spmv_status spmv_iterate(spmv_plan p, const double* x0, double* x_out, int iters, double* last_norm,
                         double* nu_out) {
  return guard([&] {
    if (!p || !x0 || !x_out || iters < 1) fail(SPMV_E_ARG, "bad argument");
    if (p->n_rows != p->n_cols) fail(SPMV_E_ARG, "iterated mode needs a square matrix");
    const int G = (int)p->shards.size();
    int cur_dev = 0;
    cudaGetDevice(&cur_dev);
    std::vector<double*> cur(G), nxt(G);
    for (int g = 0; g < G; ++g) {
      Shard& s = p->shards[g];
      ck(cudaSetDevice(s.dev), "cudaSetDevice");
      if (s.nu_cap < iters) {
        s.nu = s.alloc<double>((size_t)iters);
        s.nu_cap = iters;
      }
      if (!s.x2) s.x2 = s.alloc<double>((size_t)p->n_cols);
      if (!s.nn) s.nn = s.alloc<double>(4);
      ck(cudaMemsetAsync(s.nn, 0, 32, s.stream), "nn");
      ck(cudaMemcpyAsync(s.x, x0, (size_t)p->n_cols * 8, cudaMemcpyDefault, s.stream), "copy x0");
      cur[g] = s.x;
      nxt[g] = s.x2;
    }
    // multi-shard: interior tiles of every shard first (they read only its own
    // x block), the halo copies of the other blocks concurrently on a copy
    // stream, then the boundary tiles
    const bool push = G > 1 && prepare_push(p);
    if (G > 1 && !push)
      for (auto& s : p->shards) prepare_overlap(p, s);
    // single shard, row-aligned STREAM / D8: the prologue-norm iteration
    const StreamPlan& sp1 = p->shards[0].sp[0];
    const bool fused1 = G == 1 && p->sel.variant == SPMV_VARIANT_STREAM && sp1.aligned && !sp1.seg && !sp1.rowmap &&
                        !sp1.need_fixup && !getenv("SPMV_NO_FUSED_NORM") && !getenv("SPMV_NO_LAGGED_NORM");
    const int grid1 = std::max(sp1.grid, 1);
    double* cta2 = nullptr;
    if (fused1) {
      Shard& s = p->shards[0];
      if (!s.cta2) s.cta2 = s.alloc<double>((size_t)2 * grid1);
      cta2 = s.cta2;
    }
    for (int k = 0; k < iters; ++k) {
      // partials of iteration k live in half (k & 1) of every shard's allpart:
      // shard h may run ahead of a peer that has not yet copied h's partials
      // of iteration k (non-neighbour shards never wait on each other's x
      // halo), but not by two iterations -- its norm step k+1 waits for every
      // peer's partials of k+1, which follow that peer's copies of k
      const size_t RP = (size_t)kIterRegions * kNormPartials;
      const size_t half = (size_t)(k & 1) * G * RP;
      if (G == 1) {
        Shard& s = p->shards[0];
        set_xwin(p, s, cur[0]);
        if (fused1) {
          // one launch per iteration, nothing between two SpMVs: launch k
          // stores its per-CTA sums; launch k+1's last CTA folds them into
          // ||yh_k|| and nu_k and decides the factor launch k+2 applies
          // (iterfuse.cuh, lagged mode)
          IterOut it;
          it.cta_part = cta2 + (size_t)(k & 1) * grid1;
          it.cta_only = true;
          it.st = s.nn;  // lagged-mode state (4 doubles, zeroed)
          it.par = k & 1;
          it.rev = (k & 1) && !getenv("SPMV_NO_REVERSE");  // D8: odd launches walk the tiles backwards
          if (k > 0) {
            it.prev_part = cta2 + (size_t)((k - 1) & 1) * grid1;
            it.prev_grid = grid1;
            it.nu_k = s.nu + (k - 1);
          }
          count_launches(launch_stream_iter(s.sp[0], cur[0], nxt[0] + s.row0, it, s.stream), "iteration step");
        } else {
          // one shard: the norm step runs in the SpMV's epilogue (or its own kernel)
          count_launches(spmv_iter(p, s, cur[0], nxt[0] + s.row0, s.allpart + half, s.nn, s.nu + k),
                         "iteration step");
        }
        std::swap(cur, nxt);
        continue;
      }
      if (push) {
        // the SpMV of every shard writes yh_k into its own block of nxt and
        // the rows its neighbours read straight into THEIR nxt replicas; the
        // neighbour reads them at k + 1, after its norm step k waited for
        // this shard's SpMV (step D), and this shard writes into a replica
        // only after every peer's SpMV k - 1 finished reading it (its own
        // step D of k - 1)
        for (int g = 0; g < G; ++g) {
          Shard& s = p->shards[g];
          ck(cudaSetDevice(s.dev), "cudaSetDevice");
          set_xwin(p, s, cur[g]);
          IterOut po;
          if (s.push_lo_peer >= 0) {
            po.push_lo = nxt[s.push_lo_peer] + s.row0;
            po.push_lo_end = s.push_lo_end;
          }
          if (s.push_hi_peer >= 0) {
            po.push_hi = nxt[s.push_hi_peer] + s.row0;
            po.push_hi_begin = s.push_hi_begin;
          }
          double* part = s.allpart + half + (size_t)g * RP;
          count_launches(spmv_iter(p, s, cur[g], nxt[g] + s.row0, part, s.nn, nullptr, &po), "iteration step (push)");
          ck(cudaMemsetAsync(part + kNormPartials, 0, 2 * kNormPartials * 8, s.stream), "memset");
          ck(cudaEventRecord(s.ev_part, s.stream), "event");
        }
      }
      // A. interior tiles (overlap-capable shards)
      for (int g = 0; g < G && !push; ++g) {
        Shard& s = p->shards[g];
        if (!s.ovl || k == 0) continue;
        ck(cudaSetDevice(s.dev), "cudaSetDevice");
        set_xwin(p, s, cur[g]);
        double* part = s.allpart + half + (size_t)g * RP;
        count_launches(spmv_iter_range(p, s, cur[g], nxt[g] + s.row0, part, s.nn, s.kb, s.ke), "interior tiles");
      }
      // B. halo of yh_{k-1}: the part of each other block inside the x range
      // shard g reads, copied into g's replica (not needed at k = 0: every
      // replica holds x_0)
      if (k > 0 && !push)
        for (int g = 0; g < G; ++g) {
          Shard& s = p->shards[g];
          ck(cudaSetDevice(s.dev), "cudaSetDevice");
          const int64_t lo = s.hs.col_min, hi = s.hs.col_max + 1;
          for (int h = 0; h < G; ++h) {
            if (h == g) continue;
            Shard& t = p->shards[h];
            const int64_t a = std::max<int64_t>(lo, t.row0), b = std::min<int64_t>(hi, t.row0 + t.m);
            if (a >= b) continue;
            ck(cudaStreamWaitEvent(s.cp, t.ev_part, 0), "wait");  // h's yh_{k-1} complete
            ck(cudaMemcpyPeerAsync(cur[g] + a, s.dev, cur[h] + a, t.dev, (size_t)(b - a) * 8, s.cp), "x halo");
          }
          ck(cudaEventRecord(s.ev_cp, s.cp), "event");
        }
      // C. boundary tiles (or the whole shard) once the halo is in
      for (int g = 0; g < G && !push; ++g) {
        Shard& s = p->shards[g];
        ck(cudaSetDevice(s.dev), "cudaSetDevice");
        if (k > 0) ck(cudaStreamWaitEvent(s.stream, s.ev_cp, 0), "wait");
        double* part = s.allpart + half + (size_t)g * RP;
        if (s.ovl && k > 0) {
          count_launches(spmv_iter_range(p, s, cur[g], nxt[g] + s.row0, part + kNormPartials, s.nn, 0, s.kb) +
                             spmv_iter_range(p, s, cur[g], nxt[g] + s.row0, part + 2 * kNormPartials, s.nn, s.ke,
                                             s.sp[0].T),
                         "boundary tiles");
        } else {
          set_xwin(p, s, cur[g]);
          count_launches(spmv_iter(p, s, cur[g], nxt[g] + s.row0, part, s.nn, nullptr), "iteration step");
          ck(cudaMemsetAsync(part + kNormPartials, 0, 2 * kNormPartials * 8, s.stream), "memset");
        }
        ck(cudaEventRecord(s.ev_part, s.stream), "event");
      }
      // D. every shard gathers all partials (rank order) and runs the norm step
      for (int g = 0; g < G; ++g) {
        Shard& s = p->shards[g];
        ck(cudaSetDevice(s.dev), "cudaSetDevice");
        for (int h = 0; h < G; ++h) {
          if (h == g) continue;
          Shard& t = p->shards[h];
          ck(cudaStreamWaitEvent(s.stream, t.ev_part, 0), "wait");
          ck(cudaMemcpyPeerAsync(s.allpart + half + (size_t)h * RP, s.dev, t.allpart + half + (size_t)h * RP, t.dev,
                                 RP * 8, s.stream),
             "partials exchange");
        }
        count_launches(launch_norm_step(s.allpart + half, (int)(G * RP), s.nn, s.nu + k, s.stream), "norm step");
      }
      std::swap(cur, nxt);
    }
    // x_iters = yh_{iters-1} / ||yh_{iters-1}|| on each shard's own block
    for (int g = 0; g < G; ++g) {
      Shard& s = p->shards[g];
      ck(cudaSetDevice(s.dev), "cudaSetDevice");
      if (fused1)
        count_launches(launch_unit_fold(cur[g] + s.row0, s.m, cta2 + (size_t)((iters - 1) & 1) * grid1, grid1,
                                        s.nn, s.nu + (iters - 1), nxt[g] + s.row0, s.stream),
                       "unit");
      else
        count_launches(launch_unit(cur[g] + s.row0, s.m, s.nn, nxt[g] + s.row0, s.stream), "unit");
      set_xwin(p, s, s.x);
    }
    Shard& s0 = p->shards[0];
    std::vector<double> nu(iters);
    ck(cudaSetDevice(s0.dev), "cudaSetDevice");
    for (auto& s : p->shards) ck(cudaStreamSynchronize(s.stream), "iterate");
    ck(cudaMemcpy(nu.data(), s0.nu, (size_t)iters * 8, cudaMemcpyDeviceToHost), "nu");
    for (int g = 0; g < G; ++g) {
      Shard& s = p->shards[g];
      if (s.m) ck(cudaMemcpy(x_out + s.row0, nxt[g] + s.row0, (size_t)s.m * 8, cudaMemcpyDefault), "x_out");
    }
    cudaSetDevice(cur_dev);
    if (nu_out) memcpy(nu_out, nu.data(), (size_t)iters * 8);
    if (last_norm) *last_norm = nu[iters - 1];
    for (int k = 0; k < iters; ++k)
      if (nu[k] == 0.0 || !std::isfinite(nu[k]))
        fail(SPMV_E_ZERO_NORM, "iterated mode: ||y|| == 0 (or not finite) at iteration %d", k);
  });
}

spmv_status spmv_plan_query(spmv_plan p, spmv_plan_info* info) {
  return guard([&] {
    if (!p || !info) fail(SPMV_E_ARG, "null argument");
    memset(info, 0, sizeof *info);
    info->n_rows = p->n_rows;
    info->n_cols = p->n_cols;
    info->nnz = p->nnz;
    info->rowptr_bytes = p->rp_bytes;
    info->ngpus = (int32_t)p->shards.size();
    info->sel = p->sel;
    info->feat = p->feat;
    info->d16_width = p->d16_width;
    info->d16_n_esc = (int32_t)p->esc.size();
    info->p_csr = p->pb.p_csr;
    info->p_mb = p->pb.p_mb;
    info->p_ml = p->pb.p_ml;
    info->p_imb = p->pb.p_imb;
    info->p_cmp = p->pb.p_cmp;
    info->p_peak = p->pb.p_peak;
    info->p_stream = p->pb.p_stream;
    info->bmax = p->pb.bmax;
    info->profile_vs = p->pb.vs;
    info->profile_ctas = p->pb.ctas;
    info->profile_ms = p->profile_ms;
    const Shard& s0 = p->shards[0];
    unsigned long long rh = 0, rt = 0;
    for (const Shard& s : p->shards) { rh += s.hs.reuse_hit; rt += s.hs.reuse_tot; }
    info->x_reuse = rt ? (double)rh / (double)rt : 0.0;
    info->nz_gather_l2 = s0.nz.gather_l2 ? 1 : 0;
    info->stream_stages = s0.sp[0].stages;
    info->stream_grid = s0.sp[0].grid;
    info->d8_n_dict = s0.sp[0].codes && s0.sp[0].d8_bits ? s0.sp[0].n_dict : 0;
    info->d8_patterns = s0.sp[0].codes && !s0.sp[0].d8_bits ? s0.sp[0].n_dict : 0;
    if (s0.sp[0].codes) info->d16_width = s0.sp[0].d8_bits ? s0.sp[0].d8_bits : 8;
    {  // compulsory bytes of one SpMV in the plan's own format
      int64_t kb = 8 * p->n_cols + 8 * p->n_rows + 8 * p->nnz;
      for (const Shard& s : p->shards) {
        const StreamPlan& sp = s.sp[0];
        if (p->sel.variant == SPMV_VARIANT_STREAM && sp.codes)
          kb += (sp.d8_bits == 0 ? 0 : sp.d8_bits == 4 ? (s.nnz + 1) / 2 : s.nnz) + s.m + 8 * (sp.T + 1);  // codes,
                                                                   // row lengths (or pattern ids), tile starts
        else if (p->sel.variant == SPMV_VARIANT_STREAM && sp.dcol)
          kb += 2 * s.nnz + (int64_t)p->rp_bytes * (s.m + 1) + 4 * s.m;  // deltas, rowptr, heads
        else if (s.long_c16)
          kb += 4 * s.nnz - 2 * (int64_t)s.hs.nnz_long + (int64_t)p->rp_bytes * (s.m + 1);  // 16-bit long-row columns
        else
          kb += 4 * s.nnz + (int64_t)p->rp_bytes * (s.m + 1);
      }
      info->kernel_bytes = kb;
    }
    info->iter_push = p->push_ready && p->push_ok ? 1 : 0;
    info->long_c16 = s0.long_c16 ? 1 : 0;
    if (s0.n_long > 0) {
      info->long_mode = s0.long_tma ? 3 : s0.long_tiled ? 2 : 1;
      info->long_rg = s0.long_tma ? s0.long_rg : s0.long_tiled ? 2 : 0;
    }
    info->tile_nnz = s0.sp[0].C;
    info->n_tiles = s0.sp[0].T;
    info->tile_stride = s0.sp[0].stride;
    info->tiles_row_aligned = s0.sp[0].aligned ? 1 : 0;
    info->rows_per_tile = (int32_t)s0.sp[0].rows_per_tile;
    info->merge_items = s0.items;
    info->n_merge_tiles = s0.Tm;
    info->n_nz_rows = s0.nz.mc;
    info->n_nz_tiles = s0.nz.T;
    info->n_hot = s0.nz.n_hot;
    info->hot_cover = p->hot_cover;
    info->l_split = p->l_split;
    info->long_chunk = p->chunk;
    int64_t nc = 0, bytes = 0;
    for (auto& s : p->shards) { nc += s.n_chunks; bytes += s.bytes; }
    info->n_long_chunks = nc;
    info->upload_ms = p->upload_ms;
    info->inspect_ms = p->inspect_ms;
    info->select_ms = p->select_ms;
    info->encode_ms = p->encode_ms;
    info->device_bytes = bytes;
    for (size_t g = 0; g < p->bounds.size() && g < 9; ++g) info->shard_bounds[g] = p->bounds[g];
  });
}

spmv_status spmv_plan_table1(spmv_plan p, spmv_table1* out) {
  return guard([&] {
    if (!p || !out) fail(SPMV_E_ARG, "null argument");
    if (p->shards.size() != 1) fail(SPMV_E_ARG, "spmv_plan_table1 needs a single-shard plan");
    Shard& s = p->shards[0];
    ck(cudaSetDevice(s.dev), "cudaSetDevice");
    Table1 t;
    const int32_t* hot = (s.use_nz && s.nz.n_hot > 0 && s.nz.V.col == s.col) ? s.nz.hot_cols : nullptr;
    if (compute_table1(s.view(), hot, s.sm_count, t, s.stream) != 0) ck(cudaGetLastError(), "table1");
    g_launches += s.m ? 2 : 0;
    memset(out, 0, sizeof *out);
    const double ws = 12.0 * (double)p->nnz + (double)p->rp_bytes * (double)(p->n_rows + 1) + 8.0 * (double)p->n_cols +
                      8.0 * (double)p->n_rows;
    out->size_fits_l2 = ws <= (double)p->props.l2_bytes ? 1 : 0;
    out->density = (p->n_rows && p->n_cols) ? (double)p->nnz / ((double)p->n_rows * (double)p->n_cols) : 0.0;
    out->nnz_min = (double)p->feat.nnz_min;
    out->nnz_max = (double)p->feat.nnz_max;
    out->nnz_avg = p->feat.nnz_avg;
    out->nnz_sd = p->feat.nnz_sd;
    out->bw_min = t.bw_min;
    out->bw_max = t.bw_max;
    out->bw_avg = t.bw_avg;
    out->bw_sd = t.bw_sd;
    out->scatter_avg = t.scatter_avg;
    out->scatter_sd = t.scatter_sd;
    out->clustering_avg = t.clustering_avg;
    out->misses_avg = p->n_rows ? (double)t.misses_total / (double)p->n_rows : 0.0;
    out->n_nonempty = t.n_nonempty;
  });
}

double* spmv_plan_x_device(spmv_plan p, int g) {
  return (p && g >= 0 && g < (int)p->shards.size()) ? p->shards[g].x : nullptr;
}
double* spmv_plan_y_device(spmv_plan p, int g) {
  return (p && g >= 0 && g < (int)p->shards.size()) ? p->shards[g].y : nullptr;
}
void* spmv_plan_stream(spmv_plan p, int g) {
  return (p && g >= 0 && g < (int)p->shards.size()) ? (void*)p->shards[g].stream : nullptr;
}

int64_t spmv_plan_export(spmv_plan p, int g, int which, void* dst) {
  int64_t count = -1;
  spmv_status st = guard([&] {
    if (!p || g < 0 || g >= (int)p->shards.size()) fail(SPMV_E_ARG, "bad plan / shard");
    Shard& s = p->shards[g];
    ck(cudaSetDevice(s.dev), "cudaSetDevice");
    auto widen32 = [&](const int32_t* src, int64_t n) {
      count = n;
      if (!dst || n == 0) return;
      if (!src) fail(SPMV_E_ARG, "structure not built for the selected variant");
      std::vector<int32_t> h((size_t)n);
      ck(cudaMemcpy(h.data(), src, (size_t)n * 4, cudaMemcpyDeviceToHost), "export");
      for (int64_t i = 0; i < n; ++i) ((int64_t*)dst)[i] = h[i];
    };
    auto raw = [&](const void* src, int64_t n, size_t es) {
      count = n;
      if (!dst || n == 0) return;
      if (!src) fail(SPMV_E_ARG, "structure not built for the selected variant");
      ck(cudaMemcpy(dst, src, (size_t)n * es, cudaMemcpyDeviceToHost), "export");
    };
    switch (which) {
      case SPMV_ARR_TILE_ROWS: widen32(s.sp[0].tile_row, s.sp[0].tile_row ? s.sp[0].T + 1 : 0); break;
      case SPMV_ARR_MERGE_ROWS: widen32(s.mrow, s.mrow ? s.Tm + 1 : 0); break;
      case SPMV_ARR_MERGE_NNZ: raw(s.mnnz, s.mnnz ? s.Tm + 1 : 0, 8); break;
      case SPMV_ARR_CHUNK_ROW:
      case SPMV_ARR_CHUNK_BEGIN:
      case SPMV_ARR_CHUNK_END: {
        count = s.n_chunks;
        if (!dst || s.n_chunks == 0) break;
        int64_t* tmp = nullptr;
        ck(cudaMalloc(&tmp, (size_t)s.n_chunks * 24), "cudaMalloc");
        ExecArgs a = p->args(s, nullptr, nullptr);
        launch_chunk_export(a, tmp, s.stream);
        g_launches += 1;
        cudaError_t e = cudaStreamSynchronize(s.stream);
        if (e == cudaSuccess) {
          const int part = which - SPMV_ARR_CHUNK_ROW;
          e = cudaMemcpy(dst, tmp + (size_t)part * s.n_chunks, (size_t)s.n_chunks * 8, cudaMemcpyDeviceToHost);
        }
        cudaFree(tmp);
        ck(e, "chunk export");
        break;
      }
      case SPMV_ARR_DCOL: raw(s.sp[0].dcol, s.sp[0].dcol ? s.nnz : 0, 2); break;
      case SPMV_ARR_HEAD: raw(s.sp[0].head, s.sp[0].head ? s.m : 0, 4); break;
      case SPMV_ARR_ANCHOR: raw(s.sp[0].anchor, s.sp[0].anchor ? s.sp[0].T : 0, 4); break;
      case SPMV_ARR_D8_CODES: {  // one code per nonzero (4-bit codes unpacked, low nibble first)
        const StreamPlan& sp = s.sp[0];
        count = sp.codes && sp.d8_bits ? s.nnz : 0;
        if (!dst || count == 0) break;
        if (sp.d8_bits == 8) {
          ck(cudaMemcpy(dst, sp.codes, (size_t)count, cudaMemcpyDeviceToHost), "export");
        } else {
          std::vector<uint8_t> h((size_t)(count + 1) / 2);
          ck(cudaMemcpy(h.data(), sp.codes, h.size(), cudaMemcpyDeviceToHost), "export");
          for (int64_t j = 0; j < count; ++j) ((uint8_t*)dst)[j] = (uint8_t)((h[(size_t)(j >> 1)] >> ((j & 1) * 4)) & 15);
        }
        break;
      }
      case SPMV_ARR_D8_RLEN: raw(s.sp[0].rlen, s.sp[0].rlen && s.sp[0].d8_bits ? s.m : 0, 1); break;
      case SPMV_ARR_PAT_IDS: raw(s.sp[0].rlen, s.sp[0].rlen && !s.sp[0].d8_bits ? s.m : 0, 1); break;
      case SPMV_ARR_PAT_LEN:
      case SPMV_ARR_PAT_OFS: {
        const StreamPlan& sp = s.sp[0];
        const bool on = sp.codes && !sp.d8_bits;
        count = !on ? 0 : which == SPMV_ARR_PAT_LEN ? sp.n_dict : sp.n_pat_ofs;
        if (!dst || count == 0) break;
        if (which == SPMV_ARR_PAT_LEN) {
          for (int64_t q = 0; q < count; ++q) ((int64_t*)dst)[q] = (sp.dict[q] >> 16) & 0xff;
        } else {
          std::vector<int32_t> h((size_t)count);
          ck(cudaMemcpy(h.data(), sp.pat_ofs, (size_t)count * 4, cudaMemcpyDeviceToHost), "export");
          for (int64_t q = 0; q < count; ++q) ((int64_t*)dst)[q] = h[(size_t)q];
        }
        break;
      }
      case SPMV_ARR_D8_DICT: {
        count = s.sp[0].codes && s.sp[0].d8_bits ? s.sp[0].n_dict : 0;
        if (dst)
          for (int64_t i = 0; i < count; ++i) ((int64_t*)dst)[i] = s.sp[0].dict[i];
        break;
      }
      case SPMV_ARR_DECODED: {
        count = (s.sp[0].dcol || s.sp[0].codes) ? s.nnz : 0;
        if (!dst || count == 0) break;
        int32_t* tmp = nullptr;
        ck(cudaMalloc(&tmp, (size_t)s.nnz * 4 + 64), "cudaMalloc");
        if (s.sp[0].codes && !s.sp[0].d8_bits) launch_pat_decode_export(s.sp[0], tmp, s.stream);
        else if (s.sp[0].codes) launch_d8_decode_export(s.sp[0], s.sp[0].d8_dict_dev, tmp, s.stream);
        else launch_d16_decode_export(s.sp[0], tmp, s.stream);
        g_launches += 1;
        cudaError_t e = cudaStreamSynchronize(s.stream);
        if (e == cudaSuccess) e = cudaMemcpy(dst, tmp, (size_t)s.nnz * 4, cudaMemcpyDeviceToHost);
        cudaFree(tmp);
        ck(e, "decode export");
        break;
      }
      case SPMV_ARR_NZ_ROWMAP: widen32(s.nz.rowmap, s.nz.rowmap ? s.nz.mc + 1 : 0); break;
      case SPMV_ARR_NZ_TILE_Q: widen32(s.nz.tile_q, s.nz.tile_q ? s.nz.T + 1 : 0); break;
      case SPMV_ARR_NZ_HOT_COLS: widen32(s.nz.hot_cols, s.nz.n_hot); break;
      case SPMV_ARR_NZ_RPC: {
        count = s.nz.rpc ? s.nz.mc + 1 : 0;
        if (!dst || count == 0) break;
        if (s.rp_bytes == 8) {
          ck(cudaMemcpy(dst, s.nz.rpc, (size_t)count * 8, cudaMemcpyDeviceToHost), "export");
        } else {
          std::vector<int32_t> h((size_t)count);
          ck(cudaMemcpy(h.data(), s.nz.rpc, (size_t)count * 4, cudaMemcpyDeviceToHost), "export");
          for (int64_t i = 0; i < count; ++i) ((int64_t*)dst)[i] = h[i];
        }
        break;
      }
      case SPMV_ARR_SHARD_BOUNDS:
        count = (int64_t)p->bounds.size();
        if (dst) memcpy(dst, p->bounds.data(), p->bounds.size() * 8);
        break;
      default: fail(SPMV_E_ARG, "unknown array id %d", which);
    }
  });
  return st == SPMV_OK ? count : (int64_t)st;
}

spmv_status spmv_shard_bounds(int64_t n, const void* rowptr, int rowptr_bytes, int G, int64_t* bounds) {
  return guard([&] {
    if (!rowptr || !bounds || n < 0 || G < 1 || (rowptr_bytes != 4 && rowptr_bytes != 8))
      fail(SPMV_E_ARG, "bad argument");
    shard_bounds_host(n, rowptr, rowptr_bytes, G, bounds);
  });
}

spmv_status spmv_select(const spmv_features* f, const spmv_device_props* d, int rowptr_bytes, const spmv_options* opt,
                        spmv_selection* out) {
  return guard([&] {
    if (!f || !d || !out) fail(SPMV_E_ARG, "null argument");
    spmv_options o;
    spmv_options_default(&o);
    if (opt) o = *opt;
    validate_options(o);
    select_impl(*f, *d, rowptr_bytes, o, *out);
  });
}

spmv_status spmv_device_query(int dev, spmv_device_props* out) {
  return guard([&] {
    if (!out) fail(SPMV_E_ARG, "null argument");
    query_props(dev, *out);
  });
}

spmv_status spmv_last_status(void) { return g_status; }
const char* spmv_last_error(void) { return g_msg.c_str(); }
spmv_status spmv_plan_update_values(spmv_plan p, const double* values) {
  return guard([&] {
    if (!p || (!values && p->nnz > 0)) fail(SPMV_E_ARG, "null argument");
    int cur = 0;
    cudaGetDevice(&cur);
    for (auto& s : p->shards) {
      ck(cudaSetDevice(s.dev), "cudaSetDevice");
      ck(cudaStreamSynchronize(s.stream), "update values");  // no SpMV of the plan still reads them
      if (s.nnz) upload(s.val, values + s.nnz0, (size_t)s.nnz * 8, s.stream);
      for (auto& f : s.val_refresh) f(s.stream);
    }
    for (auto& s : p->shards) {
      ck(cudaSetDevice(s.dev), "cudaSetDevice");
      ck(cudaStreamSynchronize(s.stream), "update values");
    }
    cudaSetDevice(cur);
  });
}

int64_t spmv_kernel_launches(void) { return g_launches.load(); }

int spmv_abi_sizes(int64_t* out, int n) {
  const int64_t v[6] = {(int64_t)sizeof(spmv_options), (int64_t)sizeof(spmv_features),
                        (int64_t)sizeof(spmv_device_props), (int64_t)sizeof(spmv_selection),
                        (int64_t)sizeof(spmv_plan_info), (int64_t)sizeof(spmv_table1)};
  if (!out || n <= 0) return 0;
  const int m = n < 6 ? n : 6;
  for (int i = 0; i < m; ++i) out[i] = v[i];
  return m;
}

}  // extern "C"
