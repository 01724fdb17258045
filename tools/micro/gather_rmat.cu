// gather_rmat.cu -- microbenchmark (tools only): x-gather throughput for
// R-MAT scale-22 column indices (C3's distribution), L1-cached vs L2-only,
// with the L1 carve-out varied, and with columns renumbered by hotness.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <numeric>
#include <cuda_runtime.h>

__device__ __forceinline__ int ld_na(const int* p) { int v; asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(v) : "l"(p)); return v; }
__device__ __forceinline__ double ld_na(const double* p) { double v; asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p)); return v; }
__device__ __forceinline__ double ld_cg(const double* p) { double v; asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v) : "l"(p)); return v; }

__device__ __forceinline__ double ld_nax(const double* p) { double v; asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p)); return v; }
__device__ __forceinline__ double ld_el(const double* p) { double v; asm volatile("ld.global.nc.L1::evict_last.f64 %0, [%1];" : "=d"(v) : "l"(p)); return v; }
__device__ int g_hot;
template <int MODE>
__global__ void __launch_bounds__(256) kern(const int* __restrict__ idx, const double* __restrict__ val,
                                            const double* __restrict__ x, int64_t n, double* out) {
  const int H = g_hot;
  extern __shared__ double dummy[];
  double acc = 0.0;
  // contiguous chunk per warp (like a row-block kernel): warp w owns [w*CH, (w+1)*CH)
  const int64_t nw = (int64_t)gridDim.x * blockDim.x / 32;
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x & 31;
  const int64_t per = (n + nw - 1) / nw;
  const int64_t a = w * per, b = min(n, a + per);
  int64_t i = a + lane;
  for (; i + 7 * 32 < b; i += 8 * 32) {
    int c[8]; double v[8], xv[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) { c[u] = ld_na(idx + i + u * 32); v[u] = ld_na(val + i + u * 32); }
#pragma unroll
    for (int u = 0; u < 8; ++u) xv[u] = MODE == 0 ? __ldg(x + c[u]) : MODE == 1 ? ld_cg(x + c[u]) : MODE == 2 ? (c[u] < H ? __ldg(x + c[u]) : ld_nax(x + c[u])) : (c[u] < H ? ld_el(x + c[u]) : ld_nax(x + c[u]));
#pragma unroll
    for (int u = 0; u < 8; ++u) acc = fma(v[u], xv[u], acc);
  }
  for (; i < b; i += 32) acc += ld_na(val + i);
  if (acc == 12345.678) { out[0] = acc; dummy[0] = acc; }
}

static uint64_t sm64(uint64_t z) { z += 0x9E3779B97F4A7C15ull; z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull; z = (z ^ (z >> 27)) * 0x94D049BB133111EBull; return z ^ (z >> 31); }

int main() {
  const int S = 22;
  const int64_t N = 1ll << S, E = 16ll << S;
  std::vector<int> col(E), row(E);
  for (int64_t e = 0; e < E; ++e) {
    int r = 0, c = 0;
    for (int l = 0; l < S; ++l) {
      double u = (sm64(e * 64 + l) >> 11) * (1.0 / 9007199254740992.0);
      int rb = 0, cb = 0;
      if (u < 0.57) {} else if (u < 0.76) cb = 1; else if (u < 0.95) rb = 1; else { rb = 1; cb = 1; }
      r = (r << 1) | rb; c = (c << 1) | cb;
    }
    row[e] = r; col[e] = c;
  }
  // sort by row (CSR order), keep col order within row
  std::vector<int64_t> ord(E); std::iota(ord.begin(), ord.end(), 0);
  std::stable_sort(ord.begin(), ord.end(), [&](int64_t a, int64_t b) { return row[a] != row[b] ? row[a] < row[b] : col[a] < col[b]; });
  std::vector<int> h(E), hp(E);
  for (int64_t i = 0; i < E; ++i) h[i] = col[ord[i]];
  // hotness renumbering
  std::vector<int64_t> cnt(N, 0); for (int c : h) cnt[c]++;
  std::vector<int> perm(N); std::iota(perm.begin(), perm.end(), 0);
  std::stable_sort(perm.begin(), perm.end(), [&](int a, int b) { return cnt[a] > cnt[b]; });
  std::vector<int> inv(N); for (int i = 0; i < N; ++i) inv[perm[i]] = i;
  for (int64_t i = 0; i < E; ++i) hp[i] = inv[h[i]];
  int *idx; double *val, *x, *out;
  cudaMalloc(&idx, E * 4); cudaMalloc(&val, E * 8); cudaMalloc(&x, N * 8); cudaMalloc(&out, 8);
  cudaMemset(val, 0, E * 8); cudaMemset(x, 0, N * 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaFuncSetAttribute(kern<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(kern<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(kern<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(kern<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int p = 0; p < 2; ++p) {
    cudaMemcpy(idx, p ? hp.data() : h.data(), E * 4, cudaMemcpyHostToDevice);
    for (int mode = 0; mode < 4; ++mode)
      for (int H : {4096, 16384, 65536, 262144}) {
        if (mode < 2 && H != 4096) continue;
        if (mode >= 2 && !p) continue;
        cudaMemcpyToSymbol(g_hot, &H, 4);
        for (int smemkb : {0, 96}) {
          int occ = 8;
          int grid = sms * occ;
          size_t sm = (size_t)smemkb * 1024 / occ;
          int carve = smemkb == 0 ? 0 : (smemkb * 100 + 227) / 228;
          cudaFuncSetAttribute(kern<0>, cudaFuncAttributePreferredSharedMemoryCarveout, carve);
          cudaFuncSetAttribute(kern<1>, cudaFuncAttributePreferredSharedMemoryCarveout, carve);
          cudaFuncSetAttribute(kern<2>, cudaFuncAttributePreferredSharedMemoryCarveout, carve);
          cudaFuncSetAttribute(kern<3>, cudaFuncAttributePreferredSharedMemoryCarveout, carve);
          auto run = [&]() {
            if (mode == 0) kern<0><<<grid, 256, sm>>>(idx, val, x, E, out);
            else if (mode == 1) kern<1><<<grid, 256, sm>>>(idx, val, x, E, out);
            else if (mode == 2) kern<2><<<grid, 256, sm>>>(idx, val, x, E, out);
            else kern<3><<<grid, 256, sm>>>(idx, val, x, E, out);
          };
          run(); run();
          cudaEventRecord(a);
          for (int r = 0; r < 10; ++r) run();
          cudaEventRecord(b); cudaEventSynchronize(b);
          float ms; cudaEventElapsedTime(&ms, a, b); ms /= 10;
          const char* mn[] = {"L1", "L2", "hot-ldg/cold-na", "hot-evl/cold-na"};
          printf("%s mode=%-16s H=%6d smem/SM=%3d KB: %8.1f us  %7.1f Ggather/s\n", p ? "hot-perm" : "natural ",
                 mn[mode], H, smemkb, ms * 1e3, E / (ms * 1e-3) / 1e9);
        }
      }
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
