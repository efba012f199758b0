// Launch-overhead microbenchmark: an (almost) empty kernel, normal launch vs
// cudaLaunchCooperativeKernel, same grid, back to back on one stream.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/coop_launch tools/coop_launch.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void tiny(int* p) { if (threadIdx.x == 0 && blockIdx.x == 0 && p[0] == 12345) p[1] = 1; }
__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// grid barrier by arrival counter: fence, arrive, spin (what hm_small.cuh does)
template <int MODE>
__global__ void barrier_kernel(unsigned* c) {
  if (MODE >= 1) __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    atomicAdd(c, 1u);
    if (MODE == 2) { while (ld_acq(c) < gridDim.x) __nanosleep(32); }
    if (MODE == 3) { while (ld_acq(c) < gridDim.x) { } }
    if (MODE == 4) { while (*(volatile unsigned*)c < gridDim.x) { } }
  }
  __syncthreads();
}
int main() {
  int* p; cudaMalloc(&p, 64); cudaMemset(p, 0, 64);
  cudaStream_t s; cudaStreamCreate(&s);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int grid : {16, 64, 148, 256}) {
    void* args[] = {&p};
    for (int coop = 0; coop < 2; ++coop) {
      for (int w = 0; w < 10; ++w) {
        if (coop) cudaLaunchCooperativeKernel((void*)tiny, grid, 256, args, 0, s); else tiny<<<grid, 256, 0, s>>>(p);
      }
      cudaEventRecord(a, s);
      for (int r = 0; r < 1000; ++r) {
        if (coop) cudaLaunchCooperativeKernel((void*)tiny, grid, 256, args, 0, s); else tiny<<<grid, 256, 0, s>>>(p);
      }
      cudaEventRecord(b, s);
      cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      printf("grid %3d %-11s %.2f us/launch\n", grid, coop ? "cooperative" : "normal", ms);
    }
  }
  for (int mode = 0; mode < 5; ++mode) {
    unsigned* c = (unsigned*)p;
    cudaEventRecord(a, s);
    for (int r = 0; r < 200; ++r) {
      cudaMemsetAsync(c, 0, 4, s);
      void* args[] = {&c};
      void* fn = mode == 0 ? (void*)barrier_kernel<0> : mode == 1 ? (void*)barrier_kernel<1> :
                 mode == 2 ? (void*)barrier_kernel<2> : mode == 3 ? (void*)barrier_kernel<3> : (void*)barrier_kernel<4>;
      cudaLaunchCooperativeKernel(fn, 16, 256, args, 0, s);
    }
    cudaEventRecord(b, s); cudaEventSynchronize(b);
    float ms2; cudaEventElapsedTime(&ms2, a, b);
    printf("memset + barrier kernel mode %d (0 none,1 fence,2 spin+nanosleep,3 spin acquire,4 spin volatile): %.2f us\n",
           mode, ms2 * 1000 / 200);
  }
  cudaMemsetAsync(p, 0, 8, s);
  cudaEventRecord(a, s);
  for (int r = 0; r < 1000; ++r) { cudaMemsetAsync(p, 0, 8, s); tiny<<<16, 256, 0, s>>>(p); }
  cudaEventRecord(b, s); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("memset + normal launch: %.2f us\n", ms);
  return 0;
}
