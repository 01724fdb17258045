// iterfuse.cuh -- the iterated mode's per-iteration epilogue fused into the
// persistent SpMV kernels (row-aligned cta_stream and D8): BJ.configs[5]
// "x <- y/||y||" with deferred normalisation (reading 25).
//
//  * pending rescale: y = s * (A x) with s = *scale (the exact power of two the
//    previous norm step asked for; 0 or null = 1), so no separate pass over
//    the block ever rescales it
//  * squares: each consumer warp sums y_r^2 over the rows it writes (its tiles
//    in launch order), the CTA combines its warps in warp order into
//    cta_part[blockIdx.x]; the LAST CTA to finish (ticket counter) folds the
//    CTA partials into the kNormPartials rank partials (slot q = sum over CTAs
//    b = q (mod kNormPartials), b ascending) and, for a single rank, runs the
//    norm step itself (nu_k, nn) -- one launch per iteration, deterministic
//    for a fixed grid
#pragma once
#include "common.cuh"
#include "internal.h"

namespace spmv {

// Values another kernel of the stream wrote (nn, partials, y) are read with
// L2-coherent loads (__ldcg): with programmatic dependent launch the kernels
// overlap, and an L1 line cached by a co-resident CTA of the previous kernel
// (e.g. nn read at its start) can be stale after griddepcontrol.wait --
// measured: the final unit read a pre-epilogue nn[1] through L1.
__device__ __forceinline__ double iter_scale(const IterOut& it) {
  if (!it.scale) return 1.0;
  const double f = __ldcg(it.scale);
  return f != 0.0 ? f : 1.0;
}

// the norm step (norm.cu norm_step_kernel, same arithmetic): ss = sum of
// squares of yh_k; nu_k = ||yh_k|| / nn[0] (||yh_k|| at k = 0), nn[0] =
// ||yh_k|| brought into [2^-256, 2^256] by an exact power of two, nn[1] =
// that factor (applied to the block by the next SpMV / the final unit)
__device__ __forceinline__ void norm_step_scalar(double ss, double* nn, double* nu_k) {
  const double n = sqrt(ss), prev = __ldcg(nn);
  *nu_k = prev > 0.0 ? n / prev : n;
  const int e = (n > 0.0 && isfinite(n)) ? ilogb(n) : 0;
  const bool rs = e > 256 || e < -256;  // squares stay far from overflow (2^1024)
  nn[0] = rs ? scalbn(n, -e) : n;
  nn[1] = rs ? scalbn(1.0, -e) : 1.0;
}

// Called by every consumer thread right after pdl_wait: the exact factor this
// launch applies to its output -- lagged mode: st[2], decided by the previous
// launch's last CTA; else the pending factor of a norm step that already ran
// The exact factor this launch applies to its output: lagged mode st[2 +
// par] (decided by the previous launch's producer lanes), else the pending
// factor *scale of a norm step that already ran, else 1. Read by ONE thread
// per CTA (every consumer thread reading the same word queued ~3.5K requests
// on one L2 slice at each launch start).
__device__ __forceinline__ double iter_factor(const IterOut& it) {
  double f = 1.0;
  if (it.st) f = __ldcg(it.st + 2 + it.par);
  else if (it.scale) f = __ldcg(it.scale);
  return f != 0.0 ? f : 1.0;
}

// Lagged mode: the fold of the previous launch's per-CTA sums, by lanes 1..31
// of the PRODUCER warp of the last CTA at the start of the launch (lane 0
// issues the TMA copies; the other 31 lanes are otherwise idle), so it sits
// on no critical path -- run by the last CTA's consumers after their tiles it
// cost 5.5 % per iteration on C2. Fixed order: lane l sums b = l - 1, l + 30,
// ... ascending, then lane 1 adds the 31 lane sums in lane order. Then
//   N = ||yh_{k-1}||, nu_{k-1} = N / (F_{k-1} N_{k-2})   (N at the first step)
//   F_{k+1} = 2^-e when e = ilogb(N F_k) leaves [-128, 128], else 1
// (F_k = the factor this launch applies, st[2 + par]; F_{k+1} goes to the
// other parity slot, which no CTA of this launch reads). The rescale is
// decided one step late, so a vector may reach ~2^128 lambda^2 before it
// applies: the 2^-128..2^128 band keeps squares finite for |lambda| up to
// ~2^190 (the in-place scheme allowed 2^256 with no lag).
__device__ __forceinline__ void iter_lag_fold_lanes(const IterOut& it) {
  __shared__ double lsum[32];
  const int lane = threadIdx.x & 31;  // 1..31
  const unsigned mask = 0xfffffffeu;
  pdl_wait();  // the previous launch's sums and state
  double a = 0.0;
  for (int b = lane - 1; b < it.prev_grid; b += 31) a += __ldcg(it.prev_part + b);
  lsum[lane] = a;
  __syncwarp(mask);
  if (lane != 1) return;
  double ss = 0.0;
  for (int l = 1; l < 32; ++l) ss += lsum[l];
  const double N = sqrt(ss), Np = __ldcg(it.st), F1 = __ldcg(it.st + 1), F2 = __ldcg(it.st + 2 + it.par);
  const double fprev = F1 != 0.0 ? F1 : 1.0, fcur = F2 != 0.0 ? F2 : 1.0;
  *it.nu_k = Np > 0.0 ? N / (fprev * Np) : N;
  const double mag = N * fcur;
  const int e = (mag > 0.0 && isfinite(mag)) ? ilogb(mag) : 0;
  it.st[0] = N;
  it.st[1] = fcur;
  it.st[2 + (it.par ^ 1)] = (e > 128 || e < -128) ? scalbn(1.0, -e) : 1.0;
}

// Called by every consumer thread (NC threads, warps 1..NC/32 of the CTA;
// the producer warp has exited) after its last tile, wsq = the warp's sum of
// squares (same value in every lane). Named barrier 1 over the consumers.
template <int NC>
__device__ __forceinline__ void iter_epilogue(const IterOut& it, double wsq) {
  if (!it.cta_part) return;
  __shared__ double ws[NC / 32];
  __shared__ double fin[NC / 32];
  __shared__ int last;
  const int t = threadIdx.x - 32;  // consumer thread index
  const int w = t >> 5, lane = t & 31;
  if (lane == 0) ws[w] = wsq;
  asm volatile("bar.sync 1, %0;" ::"r"(NC) : "memory");
  if (t == 0) {
    double c = 0.0;
    for (int q = 0; q < NC / 32; ++q) c += ws[q];
    it.cta_part[blockIdx.x] = c;
    if (!it.cta_only) {  // (lagged mode: no ticket)
      __threadfence();
      const unsigned tk = atomicAdd(it.done, 1u);
      last = tk == gridDim.x - 1;
    }
  }
  if (it.cta_only) return;  // lagged mode: the fold runs in the next launch's producer warp
  asm volatile("bar.sync 1, %0;" ::"r"(NC) : "memory");
  if (!last) return;
  __threadfence();
  const int G = (int)gridDim.x;
  double mine = 0.0;  // this thread's slots, ascending
  for (int q = t; q < kNormPartials; q += NC) {
    double v = 0.0;
    for (int b = q; b < G; b += kNormPartials) v += __ldcg(it.cta_part + b);
    it.partials[q] = v;
    mine += v;
  }
  if (it.nn) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
    if (lane == 0) fin[w] = mine;
    asm volatile("bar.sync 1, %0;" ::"r"(NC) : "memory");
    if (t == 0) {
      double ss = 0.0;
      for (int q = 0; q < NC / 32; ++q) ss += fin[q];
      norm_step_scalar(ss, it.nn, it.nu_k);
    }
  }
  if (t == 0) *it.done = 0u;  // ready for the next launch (it waits for this grid before its epilogue)
}

}  // namespace spmv
