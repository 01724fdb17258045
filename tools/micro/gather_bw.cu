// gather_bw.cu -- microbenchmark (tools only, not product): throughput of
// random 8-B x gathers on B200 for the SpMV x-gather roofline.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o gather_bw gather_bw.cu
// Streams idx (int32) + val (f64) with no-allocate loads and gathers x[idx]
// (L1-cached __ldg or L1-bypassing ld.global.cg) for several x sizes.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ int ld_na(const int* p) { int v; asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(v) : "l"(p)); return v; }
__device__ __forceinline__ double ld_na(const double* p) { double v; asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p)); return v; }
__device__ __forceinline__ double ld_cg(const double* p) { double v; asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v) : "l"(p)); return v; }

template <int MODE>  // 0: L1-cached gather, 1: L2-only gather, 2: no gather (stream only)
__global__ void __launch_bounds__(256) kern(const int* __restrict__ idx, const double* __restrict__ val,
                                            const double* __restrict__ x, int64_t n, double* out) {
  double acc = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 7 * stride < n; i += 8 * stride) {
    int c[8]; double v[8], xv[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) { c[u] = ld_na(idx + i + u * stride); v[u] = ld_na(val + i + u * stride); }
#pragma unroll
    for (int u = 0; u < 8; ++u) xv[u] = MODE == 0 ? __ldg(x + c[u]) : MODE == 1 ? ld_cg(x + c[u]) : (double)c[u];
#pragma unroll
    for (int u = 0; u < 8; ++u) acc = fma(v[u], xv[u], acc);
  }
  for (; i < n; i += stride) acc += ld_na(val + i);
  if (acc == 12345.678) out[0] = acc;
}

static uint64_t sm64(uint64_t z) { z += 0x9E3779B97F4A7C15ull; z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull; z = (z ^ (z >> 27)) * 0x94D049BB133111EBull; return z ^ (z >> 31); }

int main() {
  const int64_t n = 64ll << 20;
  std::vector<int> h(n);
  int *idx; double *val, *x, *out;
  cudaMalloc(&idx, n * 4); cudaMalloc(&val, n * 8); cudaMalloc(&x, (64ll << 20) * 8); cudaMalloc(&out, 8);
  cudaMemset(val, 0, n * 8); cudaMemset(x, 0, (64ll << 20) * 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int64_t xs[] = {1 << 14, 1 << 17, 1 << 20, 1 << 22, 1 << 24, 1 << 26};
  for (int64_t X : xs) {
    for (int64_t i = 0; i < n; ++i) h[i] = (int)(sm64(i * 7 + X) % (uint64_t)X);
    cudaMemcpy(idx, h.data(), n * 4, cudaMemcpyHostToDevice);
    for (int mode = 0; mode < 3; ++mode) {
      for (int occ : {8, 16}) {
        int grid = sms * occ;
        auto run = [&]() {
          if (mode == 0) kern<0><<<grid, 256>>>(idx, val, x, n, out);
          else if (mode == 1) kern<1><<<grid, 256>>>(idx, val, x, n, out);
          else kern<2><<<grid, 256>>>(idx, val, x, n, out);
        };
        run(); run();
        cudaEventRecord(a);
        for (int r = 0; r < 10; ++r) run();
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b); ms /= 10;
        printf("x=%9lld (%7.1f MB) mode=%s occ=%2d: %8.1f us  %7.1f Ggather/s  stream %6.0f GB/s\n", (long long)X,
               X * 8 / 1e6, mode == 0 ? "L1 " : mode == 1 ? "L2 " : "none", occ, ms * 1e3, n / (ms * 1e-3) / 1e9,
               n * 12.0 / (ms * 1e-3) / 1e9);
      }
    }
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
