// Microbenchmarks that fix the roofline denominators MEASURED_PEAKS.json lacks:
//   (1) DFMA-only throughput (fp64 CUDA-core peak),
//   (2) DMMA (mma.sync .f64, SASS DMMA.8x8x4) throughput (fp64 tensor peak),
//   (3) a read-only fp64 stream over a buffer much larger than L2 (achievable read BW),
//   (4) a read+write copy (same definition as MEASURED_PEAKS.json hbm_gbs),
//   (5) DMMA + DFMA side by side, sustained DMMA / read stream, and (6) the ridge.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_peaks tools/fp64_peaks.cu
// Prints one JSON object.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

template <int CH>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double acc[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) acc[c] = threadIdx.x * 1e-9 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += acc[c];
  if (s == 12345.678) out[threadIdx.x] = s;
}

template <int CH>
__global__ void dmma_kernel(double* out, int iters) {
  double d[CH][2];
  double a = 1.0 + threadIdx.x * 1e-12, b = 0.999999;
#pragma unroll
  for (int c = 0; c < CH; ++c) { d[c][0] = c; d[c][1] = -c; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(d[c][0]), "+d"(d[c][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += d[c][0] + d[c][1];
  if (s == 12345.678) out[threadIdx.x] = s;
}

__global__ void read_kernel(const double2* __restrict__ p, size_t n2, double* out) {
  double s0 = 0, s1 = 0;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n2; i += 4 * stride) {
    double2 v0 = __ldg(p + i), v1 = __ldg(p + i + stride), v2 = __ldg(p + i + 2 * stride), v3 = __ldg(p + i + 3 * stride);
    s0 += v0.x + v1.x + v2.x + v3.x;
    s1 += v0.y + v1.y + v2.y + v3.y;
  }
  for (; i < n2; i += stride) { double2 v = __ldg(p + i); s0 += v.x; s1 += v.y; }
  if (s0 + s1 == 12345.678) out[0] = s0;
}

__global__ void copy_kernel(const double2* __restrict__ a, double2* __restrict__ b, size_t n2) {
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += stride) b[i] = a[i];
}

// (5) DMMA and DFMA at once: even warps issue DMMA, odd warps DFMA. If the two
// pipes are independent the combined rate approaches their sum.
template <int CH>
__global__ void mix_kernel(double* out, int iters) {
  const int warp = threadIdx.x >> 5;
  double s = 0;
  if (warp & 1) {
    double acc[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) acc[c] = threadIdx.x * 1e-9 + c;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int c = 0; c < CH; ++c) acc[c] = fma(acc[c], 0.9999999, 1e-7);
    }
#pragma unroll
    for (int c = 0; c < CH; ++c) s += acc[c];
  } else {
    double d[CH][2];
    double a = 1.0 + threadIdx.x * 1e-12, b = 0.999999;
#pragma unroll
    for (int c = 0; c < CH; ++c) { d[c][0] = c; d[c][1] = -c; }
    for (int i = 0; i < iters / 4; ++i) {
#pragma unroll
      for (int c = 0; c < CH; ++c)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(d[c][0]), "+d"(d[c][1]) : "d"(a), "d"(b));
    }
#pragma unroll
    for (int c = 0; c < CH; ++c) s += d[c][0] + d[c][1];
  }
  if (s == 12345.678) out[threadIdx.x] = s;
}

// (6) The ridge: a read stream with KD DMMAs per four 128-bit loads per lane
// (KD / 4 flop per byte), operands taken from the loaded data so neither pipe
// can be skipped. Run back to back (sustained), it shows what the two pipes
// deliver together under the board's power limit.
template <int KD>
__global__ void ridge_kernel(const double2* __restrict__ p, size_t n2, double* out) {
  double d[8][2];
#pragma unroll
  for (int c = 0; c < 8; ++c) d[c][0] = d[c][1] = 0.0;
  const double b = 0.999999;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n2; i += 4 * stride) {
    double2 v[4] = {__ldg(p + i), __ldg(p + i + stride), __ldg(p + i + 2 * stride), __ldg(p + i + 3 * stride)};
#pragma unroll
    for (int c = 0; c < KD; ++c) {
      const double a = (c & 1) ? v[(c >> 1) & 3].y : v[(c >> 1) & 3].x;
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(d[c & 7][0]), "+d"(d[c & 7][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += d[c][0] + d[c][1];
  if (s == 12345.678) out[0] = s;
}

template <typename F>
float time_ms(F f, int reps) {
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  f(); CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    CK(cudaEventRecord(e0));
    f();
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int dev = 0; CK(cudaSetDevice(dev));
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, dev));
  int sms = prop.multiProcessorCount;
  double* out; CK(cudaMalloc(&out, 1 << 20));

  // DFMA: 8 chains per thread, 1024 threads per SM resident x 2
  const int iters = 1 << 14;
  int blocks = sms * 8, threads = 256;
  float ms_dfma = time_ms([&] { dfma_kernel<8><<<blocks, threads>>>(out, iters, 0.9999999, 1e-7); }, 5);
  double dfma_tflops = 2.0 * 8 * iters * (double)blocks * threads / (ms_dfma * 1e-3) / 1e12;

  // DMMA m8n8k4: 2*8*8*4 = 512 flop per warp-instruction
  float ms_dmma = time_ms([&] { dmma_kernel<8><<<blocks, threads>>>(out, iters / 4); }, 5);
  double dmma_tflops = 512.0 * 8 * (iters / 4) * (double)blocks * (threads / 32) / (ms_dmma * 1e-3) / 1e12;

  // DMMA + DFMA warps side by side (half the warps each, same per-warp work as above)
  float ms_mix = time_ms([&] { mix_kernel<8><<<blocks, threads>>>(out, iters); }, 5);
  double mix_flop = 0.5 * (2.0 * 8 * iters * (double)blocks * threads) +
                    0.5 * (512.0 * 8 * (iters / 4) * (double)blocks * (threads / 32));
  double mix_tflops = mix_flop / (ms_mix * 1e-3) / 1e12;

  // Streams over 8 GiB
  size_t bytes = (size_t)8 << 30;
  double2 *a, *b;
  CK(cudaMalloc(&a, bytes));
  CK(cudaMalloc(&b, bytes / 2));
  CK(cudaMemset(a, 0, bytes));
  CK(cudaMemset(b, 0, bytes / 2));
  size_t n2 = bytes / sizeof(double2);
  float ms_read = time_ms([&] { read_kernel<<<sms * 8, 256>>>(a, n2, out); }, 10);
  double read_gbs = bytes / (ms_read * 1e-3) / 1e9;
  size_t c2 = (bytes / 2) / sizeof(double2);
  float ms_copy = time_ms([&] { copy_kernel<<<sms * 8, 256>>>(a, b, c2); }, 10);
  double copy_gbs = 2.0 * (bytes / 2) / (ms_copy * 1e-3) / 1e9;

  // Sustained figures (MEASURED_PEAKS' "sustained" reading: back to back for ~4 s,
  // total work over total time, so a power-capped clock is in the number):
  // DMMA alone, and the read stream alone.
  auto sustained = [&](auto f, double work_per_call) {
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
    f(); CK(cudaDeviceSynchronize());
    int calls = 0;
    float total = 0.f;
    CK(cudaEventRecord(e0));
    while (total < 4000.f) {
      for (int r = 0; r < 20; ++r) f();
      calls += 20;
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      CK(cudaEventElapsedTime(&total, e0, e1));
    }
    return work_per_call * calls / (total * 1e-3);
  };
  double dmma_sus = sustained([&] { dmma_kernel<8><<<blocks, threads>>>(out, iters / 4); },
                              512.0 * 8 * (iters / 4) * (double)blocks * (threads / 32)) / 1e12;
  double read_sus = sustained([&] { read_kernel<<<sms * 8, 256>>>(a, n2, out); }, (double)bytes) / 1e9;

  // the ridge, sustained: read GB/s and DMMA TF/s delivered together
  char ridge_json[1024];
  int rj = 0;
  auto ridge = [&](auto kern, int kd) {
    const double bytes_per = (double)bytes;
    const double dmma_per = (double)(n2 / 4) * kd / 32.0;  // warp-instructions: KD per 4 loads per lane
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
    kern(); CK(cudaDeviceSynchronize());
    int calls = 0;
    float total = 0.f;
    CK(cudaEventRecord(e0));
    while (total < 3000.f) {
      for (int r = 0; r < 10; ++r) kern();
      calls += 10;
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      CK(cudaEventElapsedTime(&total, e0, e1));
    }
    const double sec = total * 1e-3;
    rj += snprintf(ridge_json + rj, sizeof ridge_json - rj, "%s\"kd%d\": {\"flop_per_byte\": %.2f, \"read_gbs\": %.1f, "
                   "\"dmma_tflops\": %.2f}", rj ? ", " : "", kd, kd * 512.0 / 2048.0,
                   bytes_per * calls / sec / 1e9, 512.0 * dmma_per * calls / sec / 1e12);
  };
  ridge([&] { ridge_kernel<16><<<sms * 8, 256>>>(a, n2, out); }, 16);
  ridge([&] { ridge_kernel<24><<<sms * 8, 256>>>(a, n2, out); }, 24);
  ridge([&] { ridge_kernel<32><<<sms * 8, 256>>>(a, n2, out); }, 32);

  printf("{\"gpu\": \"%s\", \"sms\": %d, \"clock_khz\": %d, \"dfma_tflops\": %.3f, \"dmma_m8n8k4_tflops\": %.3f, "
         "\"dmma_plus_dfma_tflops\": %.3f, \"read_stream_gbs\": %.1f, \"copy_rw_gbs\": %.1f, "
         "\"dmma_m8n8k4_tflops_sustained\": %.3f, \"read_stream_gbs_sustained\": %.1f, "
         "\"ridge_sustained\": {%s}}\n",
         prop.name, sms, prop.clockRate, dfma_tflops, dmma_tflops, mix_tflops, read_gbs, copy_gbs, dmma_sus, read_sus,
         ridge_json);
  return 0;
}
