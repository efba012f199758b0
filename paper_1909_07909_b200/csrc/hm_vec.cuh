// hm_vec.cuh — vector kernels of the ||A||_2 estimate: the
// power method on A A^* that hm-toolbox runs before every recompression
// (SPEC S:165-173 estimate_norm2).
//
//   v_0 = x0 / ||x0||;  j = 1..iters:  w = A^T v,  eta = ||w||,  z = A w,  v = z / ||z||
//
// The two products are libhm's own (hodlr/hss_matvec[_t]); these kernels are the
// norms and the scaling. Deterministic: a norm is a fixed grid of fixed-order
// per-block sums (partials), added in block order by one thread of the consumer.
// All HBM-bound streaming passes over n doubles.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace hm {

constexpr int kVecThreads = 256;
constexpr int kVecMaxBlocks = 1024;

// Blocks of the norm pass for a vector of n doubles: a function of n only.
__host__ __device__ inline int vec_blocks(int64_t n) {
  const int64_t b = (n + 4095) / 4096;
  return (int)(b < 1 ? 1 : (b > kVecMaxBlocks ? kVecMaxBlocks : b));
}

// partial[blk] = sum of x[e]^2 over the block's contiguous range, thread t
// taking e = lo + t, lo + t + 256, ... sequentially, then a fixed tree over threads.
__global__ void __launch_bounds__(kVecThreads) vec_sumsq_kernel(const double* __restrict__ x, int64_t n,
                                                                double* __restrict__ partial) {
  __shared__ double red[kVecThreads];
  const int G = gridDim.x;
  const int64_t chunk = (n + G - 1) / G;
  const int64_t lo = (int64_t)blockIdx.x * chunk;
  const int64_t hi = lo + chunk < n ? lo + chunk : n;
  double s = 0.0;
  for (int64_t e = lo + threadIdx.x; e < hi; e += kVecThreads) {
    const double v = x[e];
    s = fma(v, v, s);
  }
  red[threadIdx.x] = s;
  __syncthreads();
#pragma unroll
  for (int w = kVecThreads / 2; w >= 1; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = red[0];
}

__device__ __forceinline__ double vec_norm_from_partials(const double* partial, int G) {
  double s = 0.0;
  for (int i = 0; i < G; ++i) s += partial[i];
  return sqrt(s);
}

// est[0] = sqrt(sum partial) (eta of the current step).
__global__ void vec_norm_write_kernel(const double* __restrict__ partial, int G, double* __restrict__ est) {
  if (threadIdx.x == 0 && blockIdx.x == 0) est[0] = vec_norm_from_partials(partial, G);
}

// out = x / ||x|| (||x|| from the partials of x); the zero vector stays zero,
// so a zero operator leads to eta = 0 (the oracle's early return).
__global__ void __launch_bounds__(kVecThreads) vec_normalize_kernel(const double* __restrict__ x, int64_t n,
                                                                    const double* __restrict__ partial, int G,
                                                                    double* __restrict__ out) {
  __shared__ double nrm;
  if (threadIdx.x == 0) nrm = vec_norm_from_partials(partial, G);
  __syncthreads();
  const double d = nrm;
  for (int64_t e = (int64_t)blockIdx.x * kVecThreads + threadIdx.x; e < n; e += (int64_t)gridDim.x * kVecThreads)
    out[e] = d > 0.0 ? x[e] / d : 0.0;
}

}  // namespace hm
