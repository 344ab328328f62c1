// Shared device helpers for the Aurora B200 kernels (sm_100a only).
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include "../../include/aurora_b200.h"

#define AUR_MAXN 32

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ != 1000)
#error "aurora_b200 kernels target sm_100a only"
#endif

__device__ __forceinline__ double warp_min_d(double v) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__device__ __forceinline__ double warp_max_d(double v) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__device__ __forceinline__ int warp_sum_i(int v) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ---- memory-model helpers for cross-CTA / cross-GPU flags ----
__device__ __forceinline__ int ld_acquire_sys(const int* p) {
  int v;
  asm volatile("ld.acquire.sys.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(int* p, int v) {
  asm volatile("st.release.sys.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_release_gpu(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_release_sys_add(int* p, int v) {
  asm volatile("red.release.sys.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_relaxed_sys_add(int* p, int v) {
  asm volatile("red.relaxed.sys.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_relaxed_gpu_add(int* p, int v) {
  asm volatile("red.relaxed.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_release_gpu_add(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// 16-byte global accesses that bypass L1 allocation (streaming copies)
__device__ __forceinline__ int4 ld_nc_v4(const int4* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ void st_na_v4(int4* p, int4 v) {
  asm volatile("st.global.L1::no_allocate.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y),
               "r"(v.z), "r"(v.w)
               : "memory");
}

// internal (gemm.cu -> gemm2sm.cu): the fused combine's destinations, see
// aurora_expert_ffn_combine in include/aurora_b200.h
struct AuroraScatterArgs {
  void* const* ret;
  const int32_t* counts;
  const int32_t* soff;
  const int32_t* roff;
  int32_t* const* ctrs;
  int32_t* ticket;
  int n, rank_base, sys;
  const void* ginfo;  // packed groups: per-row {recv row, weight, single, -} (nullptr: one expert per rank)
  int G;
  void* ybuf;
  long long ycap;
  int to_ret;
};

// Arrival-driven GEMM1 (aurora_expert_ffn_combine with landed): tiles wait for their rows
struct AuroraArrivalArgs {
  int32_t* landed;        // [n_local][n]: rows of block (sender i -> local receiver g) visible
  const int32_t* counts;  // [n][n]
  const int32_t* roff;    // [n][n]
  int n, rank_base, sys;
  int pdl;                // launch as a programmatic dependent of the preceding dispatch
};

#define AUR_CHECK_LAUNCH()                          \
  do {                                              \
    cudaError_t _e = cudaGetLastError();            \
    if (_e != cudaSuccess) return AURORA_ECUDA;     \
  } while (0)
