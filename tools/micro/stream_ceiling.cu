// stream_ceiling.cu -- microbenchmark (tools only, not product): the best
// time a plain streaming kernel needs to read R bytes and write W bytes on
// B200, with L2 flushed between timed launches, at the SpMV workloads' sizes.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o stream_ceiling stream_ceiling.cu
// This is the achievable-bandwidth ceiling a CSR SpMV of the same footprint
// can approach (it reads more streams and gathers x, so it can only be slower).
#include <cstdio>
#include <cstdint>
#include <algorithm>
#include <cuda_runtime.h>

struct __align__(32) V4 { double a, b, c, d; };

__device__ __forceinline__ V4 ld256(const V4* p) {
  V4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.f64 {%0,%1,%2,%3}, [%4];"
               : "=d"(v.a), "=d"(v.b), "=d"(v.c), "=d"(v.d) : "l"(p));
  return v;
}

template <int U>
__global__ void __launch_bounds__(512) rd(const V4* __restrict__ in, int64_t n4, double* __restrict__ out,
                                          int64_t nout) {
  double acc = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < n4; i += U * stride) {
    V4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = ld256(in + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) acc += v[u].a + v[u].b + v[u].c + v[u].d;
  }
  for (; i < n4; i += stride) { V4 v = ld256(in + i); acc += v.a + v.b + v.c + v.d; }
  // write stream: out has nout doubles, written once each
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < nout; j += stride) out[j] = acc;
}


// ---- TMA variant: persistent CTAs, one producer lane streams CH-byte bulk
// copies into an S-stage smem ring, 4 consumer warps sum each stage.
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bar_init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c)); }
__device__ __forceinline__ void bar_expect(uint64_t* b, uint32_t bytes) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory"); }
__device__ __forceinline__ void bar_arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory"); }
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t par) {
  asm volatile("{\n.reg .pred P1;\nW: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W;\n}" ::"r"(su32(b)), "r"(par) : "memory");
}
__device__ __forceinline__ void g2s(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(dst)), "l"(src), "r"(bytes), "r"(su32(b)) : "memory");
}
template <int S, int CH>
__global__ void __launch_bounds__(160) rd_tma(const char* __restrict__ in, int64_t nch, double* __restrict__ out, int64_t nout) {
  extern __shared__ __align__(128) char sm[];
  __shared__ uint64_t full[S], empty[S];
  const int w = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) { for (int i = 0; i < S; ++i) { bar_init(&full[i], 1); bar_init(&empty[i], 4); } asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncthreads();
  double acc = 0.0;
  if (w == 4) {
    if (lane == 0) {
      int it = 0;
      for (int64_t c = blockIdx.x; c < nch; c += gridDim.x, ++it) {
        const int st = it % S;
        if (it >= S) bar_wait(&empty[st], ((it / S) - 1) & 1);
        bar_expect(&full[st], CH);
        g2s(sm + st * CH, in + c * CH, CH, &full[st]);
      }
    }
  } else {
    int it = 0;
    for (int64_t c = blockIdx.x; c < nch; c += gridDim.x, ++it) {
      const int st = it % S;
      bar_wait(&full[st], (it / S) & 1);
      const double* d = (const double*)(sm + st * CH);
      for (int j = threadIdx.x; j < CH / 8; j += 128) acc += d[j];
      __syncwarp();
      if (lane == 0) bar_arrive(&empty[st]);
    }
  }
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < nout; j += stride) out[j] = acc;
}

// generic TMA ring: S stages of CH bytes (runtime), 4 consumer warps + 1 producer
__global__ void __launch_bounds__(160) rd_tma_rt(const char* __restrict__ in, int64_t nch, int S, int CH,
                                                 double* __restrict__ out) {
  extern __shared__ __align__(128) char sm[];
  __shared__ uint64_t full[16], empty[16];
  const int w = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) { for (int i = 0; i < S; ++i) { bar_init(&full[i], 1); bar_init(&empty[i], 4); } asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncthreads();
  double acc = 0.0;
  if (w == 4) {
    if (lane == 0) {
      int it = 0;
      for (int64_t c = blockIdx.x; c < nch; c += gridDim.x, ++it) {
        const int st = it % S;
        if (it >= S) bar_wait(&empty[st], ((it / S) - 1) & 1);
        bar_expect(&full[st], CH);
        g2s(sm + (size_t)st * CH, in + c * CH, CH, &full[st]);
      }
    }
  } else {
    int it = 0;
    for (int64_t c = blockIdx.x; c < nch; c += gridDim.x, ++it) {
      const int st = it % S;
      bar_wait(&full[st], (it / S) & 1);
      const double* d = (const double*)(sm + (size_t)st * CH);
      for (int j = threadIdx.x; j < CH / 8; j += 128) acc += d[j];
      __syncwarp();
      if (lane == 0) bar_arrive(&empty[st]);
    }
  }
  if (acc == 1234.5) out[0] = acc;
}

__global__ void flush(double* f, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    f[i] = f[i] * 0.5 + 1.0;
}

int sweep(double* fl, int64_t fl_n, int sms) {
  const int64_t bytes = 4096ll << 20;
  char* in;
  double* out;
  cudaMalloc(&in, bytes);
  cudaMalloc(&out, 64);
  cudaMemset(in, 0, bytes);
  cudaFuncSetAttribute(rd_tma_rt, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int CH : {3072, 6144, 9216, 12288, 16384, 32768})
    for (int S : {2, 4, 8})
      for (int occ : {1, 2, 4, 6, 8}) {
        if ((size_t)S * CH * occ > 200 * 1024) continue;
        const int64_t nch = bytes / CH;
        float best = 1e30f;
        for (int t = 0; t < 5; ++t) {
          flush<<<sms * 4, 512>>>(fl, fl_n);
          cudaEventRecord(e0);
          rd_tma_rt<<<sms * occ, 160, (size_t)S * CH>>>(in, nch, S, CH, out);
          cudaEventRecord(e1);
          cudaEventSynchronize(e1);
          float ms;
          cudaEventElapsedTime(&ms, e0, e1);
          if (t >= 1) best = std::min(best, ms);
        }
        printf("TMA CH %6d S %d ctas/SM %d  inflight/SM %4d KB  %8.1f us  %6.0f GB/s\n", CH, S, occ,
               S * CH * occ / 1024, best * 1e3, nch * (double)CH / (best * 1e-3) / 1e9);
      }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}

int main(int argc, char** argv) {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int64_t fl_n = 64ll << 20;  // 512 MB flush buffer
  double* fl;
  cudaMalloc(&fl, fl_n * 8);
  cudaMemset(fl, 0, fl_n * 8);
  if (argc > 1) return sweep(fl, fl_n, sms);
  struct Case { const char* name; double rd_mb, wr_mb; };
  const Case cases[] = {{"C2-like 200MB rd + 17MB wr", 200.5, 16.8},
                        {"C4-like 430MB rd + 8MB wr", 430.0, 8.0},
                        {"1GB rd + 0 wr", 1024.0, 0.0},
                        {"4GB rd + 0.45GB wr (C5 shape/4)", 4096.0, 453.0}};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (const Case& c : cases) {
    const int64_t n4 = (int64_t)(c.rd_mb * 1e6) / 32;
    const int64_t nout = (int64_t)(c.wr_mb * 1e6) / 8;
    V4* in;
    double* out;
    cudaMalloc(&in, n4 * 32);
    cudaMalloc(&out, std::max<int64_t>(nout, 1) * 8);
    cudaMemset(in, 0, n4 * 32);
    for (int occ : {2, 4}) {
      for (int U : {2, 4}) {
        const int grid = sms * occ;
        float best = 1e30f, sum = 0.f;
        for (int t = 0; t < 12; ++t) {
          flush<<<sms * 4, 512>>>(fl, fl_n);
          cudaEventRecord(e0);
          if (U == 2) rd<2><<<grid, 512>>>(in, n4, out, nout);
          else rd<4><<<grid, 512>>>(in, n4, out, nout);
          cudaEventRecord(e1);
          cudaEventSynchronize(e1);
          float ms;
          cudaEventElapsedTime(&ms, e0, e1);
          if (t >= 2) { best = std::min(best, ms); sum += ms; }
        }
        const double bytes = n4 * 32.0 + nout * 8.0;
        printf("%-34s grid %4d U%d  best %9.1f us (%6.0f GB/s)  mean %9.1f us (%6.0f GB/s)\n", c.name, grid, U,
               best * 1e3, bytes / (best * 1e-3) / 1e9, sum / 10 * 1e3, bytes / (sum / 10 * 1e-3) / 1e9);
      }
    }
    {
      auto run_tma = [&](auto kern, int S, int CH, int ctas) {
        const int smem = S * CH;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        const int64_t nch = n4 * 32 / CH;
        const int grid = sms * ctas;
        float best = 1e30f, sum = 0.f;
        for (int t = 0; t < 12; ++t) {
          flush<<<sms * 4, 512>>>(fl, fl_n);
          cudaEventRecord(e0);
          kern<<<grid, 160, smem>>>((const char*)in, nch, out, nout);
          cudaEventRecord(e1);
          cudaEventSynchronize(e1);
          float ms;
          cudaEventElapsedTime(&ms, e0, e1);
          if (t >= 2) { best = std::min(best, ms); sum += ms; }
        }
        const double bytes = nch * (double)CH + nout * 8.0;
        printf("%-34s TMA S%d CH%5d x%d  best %9.1f us (%6.0f GB/s)  mean %9.1f us (%6.0f GB/s)\n", c.name, S, CH, ctas,
               best * 1e3, bytes / (best * 1e-3) / 1e9, sum / 10 * 1e3, bytes / (sum / 10 * 1e-3) / 1e9);
      };
      run_tma(rd_tma<8, 16384>, 8, 16384, 1);
      run_tma(rd_tma<12, 16384>, 12, 16384, 1);
      run_tma(rd_tma<6, 16384>, 6, 16384, 2);
      run_tma(rd_tma<4, 8192>, 4, 8192, 4);
      run_tma(rd_tma<4, 4096>, 4, 4096, 8);
    }
    cudaFree(in);
    cudaFree(out);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
