// common.cuh -- device helpers shared by the product kernels (sm_100a only).
// Nothing here is shared with oracle/ (the oracle is independent C code).
#pragma once
#include <cstdint>
#include <cstdlib>
#include <utility>
#include <cuda_runtime.h>

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "libspmv targets sm_100a only"
#endif

// Checked build (tools/build_variant.sh checks -DSPMV_CHECKS): device-side
// bounds asserts in the hot kernels (compute-sanitizer is not available on
// the GPU pool); compiled out of the product build
#ifdef SPMV_CHECKS
#include <cassert>
#define SPMV_CHECK(c) assert(c)
#else
#define SPMV_CHECK(c) ((void)0)
#endif

namespace spmv {


// ---- streaming loads: read-only, do not allocate in L1 (values / colind are
// touched exactly once; only the x gather should live in L1/L2) ------------
__device__ __forceinline__ double ld_stream(const double* p) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ int ld_stream(const int* p) {
  int v;
  asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ int ld_stream_u16(const uint16_t* p) {
  unsigned short v;
  asm volatile("ld.global.nc.L1::no_allocate.u16 %0, [%1];" : "=h"(v) : "l"(p));
  return (int)v;
}
__device__ __forceinline__ double2 ld_stream2(const double* p) {
  double2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}
// x gather: read-only path, cached in L1 (neighbouring rows share x entries)
__device__ __forceinline__ double ld_x(const double* p) { return __ldg(p); }
// x gather of the nnz tiles: L1-cached, or L2 only (L2G: rows without x-line
// reuse; B200 measures the same ~270 G gathers/s either way for random
// columns, and .cg leaves L1 to the streams and the in-flight misses)
template <bool L2G>
__device__ __forceinline__ double ld_xg(const double* p) {
  if constexpr (L2G) return __ldcg(p);
  else return __ldg(p);
}

template <typename T>
__device__ __forceinline__ T ld_ro(const T* p) { return __ldg(p); }

// ---- TMA bulk copies (cp.async.bulk, non-tensor) + mbarrier -----------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
// The suspend-time hint lets the waiting warp sleep in hardware until the
// phase completes (or ~the hint elapses) instead of spinning: measured on
// the STREAM kernel, spin loops (SYNCS.TRYWAIT + YIELD + BRA) were ~30 % of
// all issued instructions and competed with the working warps for issue.
#ifndef SPMV_MBAR_HINT
#define SPMV_MBAR_HINT 1
#endif
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
#if !SPMV_MBAR_HINT
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
  return;
#endif
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(1000000u)
      : "memory");
}
// global -> shared bulk copy; bytes % 16 == 0, both addresses 16-B aligned.
// L2 evict_first: the matrix streams are read once per SpMV.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
// bulk prefetch of [src, src + bytes) into L2 (no smem, no completion)
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// ---- programmatic dependent launch (PDL) -------------------------------------
// The hot-path kernels are launched with programmatic stream serialization: a
// kernel's CTAs may be scheduled while its predecessor in the stream drains
// (each CTA triggers its dependents at entry), and every such kernel calls
// pdl_wait() before its first access to data a previous kernel may write
// (x, y, carries); only plan-constant matrix streams may be read before it.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("SPMV_PDL");
    return e ? atoi(e) != 0 : true;
  }();
  return on;
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// SM count of the current device (grid sizing of the helper kernels; the
// persistent hot-path kernels take it from the plan's device properties)
inline int dev_sm_count() {
  static int cache[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  if (!cache[dev]) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
    cache[dev] = v;
  }
  return cache[dev];
}

// ---- warp / subwarp reductions (fixed butterfly order => deterministic) ----
template <int VS>
__device__ __forceinline__ double group_sum(double v) {
#pragma unroll
  for (int o = VS / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o, VS);
  return v;
}

template <typename T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    T w = __shfl_xor_sync(0xffffffffu, v, o);
    v = v > w ? v : w;
  }
  return v;
}
template <typename T>
__device__ __forceinline__ T warp_min(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    T w = __shfl_xor_sync(0xffffffffu, v, o);
    v = v < w ? v : w;
  }
  return v;
}
template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ int64_t lower_bound_dev(const int32_t* rp, int64_t lo, int64_t hi, int64_t key) {
  int64_t a = lo, b = hi + 1;
  while (a < b) {
    int64_t mid = a + ((b - a) >> 1);
    if ((int64_t)rp[mid] < key) a = mid + 1; else b = mid;
  }
  return a;
}
__device__ __forceinline__ int64_t lower_bound_dev(const int64_t* rp, int64_t lo, int64_t hi, int64_t key) {
  int64_t a = lo, b = hi + 1;
  while (a < b) {
    int64_t mid = a + ((b - a) >> 1);
    if (rp[mid] < key) a = mid + 1; else b = mid;
  }
  return a;
}

}  // namespace spmv
