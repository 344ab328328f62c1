// FP32 FMA throughput on one B200: scalar FFMA vs fp32x2 FFMA2 (__ffma2_rn) chains,
// many independent accumulators per thread, full occupancy. Calibrates the router's
// FMA-bound floor (route_units_kernel, C5).
#include <cstdio>
#include <cuda_runtime.h>

template <bool PAIR>
__global__ void fma_kernel(float* out, int iters, float a) {
  constexpr int NA = 16;
  if (PAIR) {
    float2 acc[NA];
    for (int i = 0; i < NA; i++) acc[i] = make_float2(threadIdx.x * 1e-3f + i, i * 0.5f);
    const float2 m = make_float2(a, a), c = make_float2(1e-7f, 2e-7f);
    for (int it = 0; it < iters; it++)
#pragma unroll
      for (int i = 0; i < NA; i++) acc[i] = __ffma2_rn(acc[i], m, c);
    float s = 0;
    for (int i = 0; i < NA; i++) s += acc[i].x + acc[i].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  } else {
    float acc[NA];
    for (int i = 0; i < NA; i++) acc[i] = threadIdx.x * 1e-3f + i;
    for (int it = 0; it < iters; it++)
#pragma unroll
      for (int i = 0; i < NA; i++) acc[i] = fmaf(acc[i], a, 1e-7f);
    float s = 0;
    for (int i = 0; i < NA; i++) s += acc[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 4, threads = 512, iters = 20000;
  float* out;
  cudaMalloc(&out, blocks * threads * sizeof(float));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int pair = 0; pair < 2; pair++) {
    for (int rep = 0; rep < 2; rep++) {
      cudaEventRecord(e0);
      if (pair) fma_kernel<true><<<blocks, threads>>>(out, iters, 0.999f);
      else fma_kernel<false><<<blocks, threads>>>(out, iters, 0.999f);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double fmas = (double)blocks * threads * iters * 16 * (pair ? 2 : 1);
      if (rep) printf("%s: %.1f T FMA/s (%.2f ms)\n", pair ? "FFMA2" : "FFMA ", fmas / ms / 1e9, ms);
    }
  }
  return 0;
}
