// Calibration: row copies (8 KiB rows, gathered source) through the TMA bulk
// path (producer warp -> smem slots -> consumer warp) vs. plain LSU copies.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tma_copy_bench.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c)); }
__device__ __forceinline__ void expect_tx(uint64_t* b, uint32_t x) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(x) : "memory"); }
__device__ __forceinline__ void arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory"); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n\t.reg .pred P1;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W_%=;\n\t}" ::"r"(su32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void bload(uint32_t d, const void* s, uint32_t n, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(d), "l"(s), "r"(n), "r"(su32(b)) : "memory");
}
__device__ __forceinline__ void bstore(void* d, uint32_t s, uint32_t n) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(d), "r"(s), "r"(n) : "memory");
}
template <int N> __device__ __forceinline__ void wread() { asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory"); }

template <int LAG>
__global__ void tma_copy(const char* src, char* dst, const int* perm, int rows_per_cta, int rb, int S) {
  extern __shared__ __align__(128) unsigned char sl[];
  __shared__ uint64_t full[32], empty[32];
  if (threadIdx.x == 0) { for (int s = 0; s < S; s++) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); } asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncthreads();
  const long long r0 = (long long)blockIdx.x * rows_per_cta;
  const uint32_t base = su32(sl);
  if (threadIdx.x == 0) {
    for (int t = 0; t < rows_per_cta; t++) {
      int s = t % S; uint32_t u = t / S;
      if (u > 0) wait(&empty[s], (u - 1) & 1);
      expect_tx(&full[s], rb);
      bload(base + s * rb, src + (long long)perm[r0 + t] * rb, rb, &full[s]);
    }
  } else if (threadIdx.x == 32) {
    int rel = 0;
    for (int t = 0; t < rows_per_cta; t++) {
      int s = t % S; uint32_t u = t / S;
      wait(&full[s], u & 1);
      bstore(dst + (r0 + t) * rb, base + s * rb, rb);
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      wread<LAG>();
      for (; rel < t + 1 - LAG; rel++) arrive(&empty[rel % S]);
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

__global__ void lsu_copy(const char* src, char* dst, const int* perm, int rows_per_cta, int rb) {
  const long long r0 = (long long)blockIdx.x * rows_per_cta;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, W = blockDim.x >> 5;
  for (int t = warp; t < rows_per_cta; t += W) {
    const int4* s = (const int4*)(src + (long long)perm[r0 + t] * rb);
    int4* d = (int4*)(dst + (r0 + t) * rb);
    int4 v[16];
#pragma unroll
    for (int q = 0; q < 16; q++) v[q] = s[q * 32 + lane];
#pragma unroll
    for (int q = 0; q < 16; q++) d[q * 32 + lane] = v[q];
  }
}

int main() {
  const int rb = 8192, rows = 32768;
  char *src, *dst; int* perm;
  cudaMalloc(&src, (size_t)rows * rb); cudaMalloc(&dst, (size_t)rows * rb); cudaMalloc(&perm, rows * 4);
  std::vector<int> h(rows); for (int i = 0; i < rows; i++) h[i] = (int)((i * 7919LL) % rows);
  cudaMemcpy(perm, h.data(), rows * 4, cudaMemcpyHostToDevice);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto report = [&](const char* name, float ms) { printf("%-28s %8.1f us  %7.0f GB/s (r+w)\n", name, ms * 1e3, 2.0 * rows * rb / (ms * 1e-3) / 1e9); };
  // per-CTA rate = (r+w)/2 / grid
  for (int grid : {37, 74, 148, 296, 592}) {
    for (int S : {6, 12, 24}) {
      if ((size_t)S * rb * (grid > 148 ? (grid + 147) / 148 : 1) > 200 * 1024) continue;
      const int rows_used = rows / grid * grid;
      int rpc = rows / grid; size_t sm = (size_t)S * rb;
      auto run = [&](auto kern, const char* tag) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        for (int it = 0; it < 2; it++) kern<<<grid, 64, sm>>>(src, dst, perm, rpc, rb, S);
        cudaEventRecord(a);
        for (int it = 0; it < 5; it++) kern<<<grid, 64, sm>>>(src, dst, perm, rpc, rb, S);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        char nm[64]; snprintf(nm, 64, "tma g=%d S=%d %s", grid, S, tag);
        if (cudaGetLastError() != cudaSuccess) { printf("%s launch error\n", nm); return; }
        report(nm, ms / 5);
      };
      run(tma_copy<1>, "lag1");
      if (S >= 4) run(tma_copy<2>, "lag2");
      if (S >= 8) run(tma_copy<4>, "lag4");
    }
  }
  for (int grid : {148, 296, 592}) {
    int rpc = rows / grid;
    for (int it = 0; it < 2; it++) lsu_copy<<<grid, 256>>>(src, dst, perm, rpc, rb);
    cudaEventRecord(a);
    for (int it = 0; it < 5; it++) lsu_copy<<<grid, 256>>>(src, dst, perm, rpc, rb);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    char nm[64]; snprintf(nm, 64, "lsu g=%d", grid);
    report(nm, ms / 5);
  }
  return 0;
}
