// pdl_visibility.cu -- microbenchmark (tools only): does griddepcontrol.wait in a
// programmatic-dependent kernel B wait for the COMPLETION of kernel A, or only
// for A's launch_dependents triggers? A triggers at entry, spins, then writes
// a flag; B waits, then reads the flag (plain L1-cacheable load and .cg load).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o pdl_visibility pdl_visibility.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void kA(volatile int* flag, long long spin_ns, int prime) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (prime && __ldca((const int*)flag) == 12345) flag[1] = 0;  // cache the flag line in this SM L1 first
  long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > spin_ns) break;
  }
  if (threadIdx.x == 0 && blockIdx.x == gridDim.x - 1) flag[0] = 1;
}
__global__ void kB(const int* flag, int* out) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0) {
    out[2 * blockIdx.x] = flag[0];
    out[2 * blockIdx.x + 1] = __ldcg(flag);
  }
}
int main() {
  int *flag, *out;
  cudaMalloc(&flag, 4);
  cudaMalloc(&out, 8 * 148 * 4);
  cudaStream_t s;
  cudaStreamCreate(&s);
  for (int prime = 0; prime < 2; ++prime)
    for (int gridA : {1, 148}) {
      int bad_plain = 0, bad_cg = 0, trials = 20;
      for (int t = 0; t < trials; ++t) {
        cudaMemsetAsync(flag, 0, 4, s);
        kA<<<gridA, 32, 0, s>>>(flag, 200000, prime);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(148 * 4);
        cfg.blockDim = dim3(32);
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, kB, (const int*)flag, out);
        int h[8 * 148];
        cudaMemcpyAsync(h, out, sizeof(int) * 2 * 148 * 4, cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        for (int b = 0; b < 148 * 4; ++b) {
          bad_plain += h[2 * b] != 1;
          bad_cg += h[2 * b + 1] != 1;
        }
      }
      printf("A grid %3d prime %d: B CTAs that read flag=0 after griddepcontrol.wait: plain %d, .cg %d (of %d)\n",
             gridA, prime, bad_plain, bad_cg, trials * 148 * 4);
    }
  return 0;
}
