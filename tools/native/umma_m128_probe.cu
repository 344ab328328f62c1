// Probe: where does tcgen05.mma.cta_group::2 with M = 128 put its accumulator rows?
// One CTA pair, K = 64: CTA r stages A rows [64 r, 64 r + 128) (only the first 64
// feed the M = 128 instruction) and B rows [128 r, +128); the leader issues the
// MMA, both CTAs dump TMEM lanes 0..127 x 256 columns. The host matches every
// (CTA, lane) against the rows of A x B^T.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2410_17043_b200/csrc umma_m128_probe.cu -lcuda
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
#include <cuda_bf16.h>
#include "tc_helpers.cuh"

constexpr int K = 64, NB = 256;

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__global__ void __cluster_dims__(2, 1, 1) probe(const __grid_constant__ CUtensorMap ma,
                                                const __grid_constant__ CUtensorMap mb, float* out, int M) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + 32768);
  uint64_t* done = full + 1;
  uint32_t* tbase = reinterpret_cast<uint32_t*>(done + 1);
  const uint32_t rank = tc::cluster_rank();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    tc::mbar_init(full, 1);
    tc::mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc::smem_u32(tbase)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc::fence_before();
  __syncthreads();
  tc::cluster_sync();
  tc::fence_after();
  const uint32_t tmem = *tbase;
  if (M == 1) {  // each CTA: its own 1-CTA MMA, M = 128 (A rows 0-127), N = 128 (its B half)
    if (threadIdx.x == 0) {
      tc::mbar_expect_tx(full, 32768);
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                   ::"r"(tc::smem_u32(sm)), "l"(reinterpret_cast<uint64_t>(&ma)), "r"(tc::smem_u32(full)), "r"(0), "r"(0) : "memory");
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                   ::"r"(tc::smem_u32(sm + 16384)), "l"(reinterpret_cast<uint64_t>(&mb)), "r"(tc::smem_u32(full)), "r"(0), "r"(128 * (int)rank) : "memory");
    }
    if (threadIdx.x == 32) {
      tc::mbar_wait(full, 0);
      tc::fence_after();
      const uint64_t ad = tc::sw128_desc(sm), bd = tc::sw128_desc(sm + 16384);
      const uint32_t idesc = tc::idesc_bf16(128, 128);
      for (int k = 0; k < K / 16; k++)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                     ::"r"(tmem), "l"(ad + 2 * k), "l"(bd + 2 * k), "r"(idesc), "r"((uint32_t)(k != 0)));
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(tc::smem_u32(done)) : "memory");
    }
    tc::mbar_wait(done, 0);
  } else {
  if (threadIdx.x == 0) {
    const uint32_t f0 = tc::mapa(tc::smem_u32(full), 0);
    if (rank == 0) tc::mbar_expect_tx(full, 2 * 32768);
    tc::tma_load_2d_pair(sm, &ma, f0, 0, (M == 128 ? 64 : 128) * (int)rank);
    tc::tma_load_2d_pair(sm + 16384, &mb, f0, 0, 128 * (int)rank);
  }
  if (rank == 0 && threadIdx.x == 32) {
    tc::mbar_wait(full, 0);
    tc::fence_after();
    const uint64_t ad = tc::sw128_desc(sm), bd = tc::sw128_desc(sm + 16384);
    const uint32_t idesc = tc::idesc_bf16(M, NB);
    for (int k = 0; k < K / 16; k++) tc::umma_bf16_pair(tmem, ad + 2 * k, bd + 2 * k, idesc, k != 0);
    tc::umma_commit_pair(done, 0x3);
  }
  tc::mbar_wait_cluster(done, 0);
  }
  tc::fence_after();
  if (warp < 4) {
    for (int c0 = 0; c0 < NB; c0 += 32) {
      uint32_t r[32];
      TC_TMEM_LD32(tmem + ((uint32_t)(warp * 32) << 16) + c0, r);
      tc::tmem_ld_wait();
      for (int q = 0; q < 32; q++)
        out[((size_t)rank * 128 + warp * 32 + lane) * NB + c0 + q] = __uint_as_float(r[q]);
    }
  }
  tc::fence_before();
  __syncthreads();
  tc::cluster_sync();
  if (warp == 1) {
    tc::fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
  }
}

int main(int argc, char** argv) {
  const int M = argc > 1 ? atoi(argv[1]) : 128;
  const int AR = 256;  // A rows in memory (rows past M are zero)
  const int Mrows = (M == 1) ? 128 : M;
  std::vector<__nv_bfloat16> hA((size_t)AR * K), hB((size_t)NB * K);
  std::vector<float> fA((size_t)AR * K, 0.f), fB((size_t)NB * K);
  srand(1);
  for (int i = 0; i < AR; i++)
    for (int k = 0; k < K; k++) {
      float v = (i < Mrows) ? (float)((rand() % 17) - 8) / 8.0f : 0.f;
      hA[(size_t)i * K + k] = __float2bfloat16(v);
      fA[(size_t)i * K + k] = v;
    }
  for (int i = 0; i < NB; i++)
    for (int k = 0; k < K; k++) {
      float v = (float)((rand() % 17) - 8) / 8.0f;
      hB[(size_t)i * K + k] = __float2bfloat16(v);
      fB[(size_t)i * K + k] = v;
    }
  __nv_bfloat16 *dA, *dB;
  float* dO;
  cudaMalloc(&dA, hA.size() * 2);
  cudaMalloc(&dB, hB.size() * 2);
  cudaMalloc(&dO, 2 * 128 * NB * 4);
  cudaMemcpy(dA, hA.data(), hA.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB.data(), hB.size() * 2, cudaMemcpyHostToDevice);
  cudaMemset(dO, 0, 2 * 128 * NB * 4);
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  EncFn enc = (EncFn)fp;
  CUtensorMap ma, mb;
  cuuint64_t da[2] = {K, (cuuint64_t)AR}, db[2] = {K, NB}, st[1] = {K * 2};
  cuuint32_t box[2] = {64, 128}, es[2] = {1, 1};
  enc(&ma, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dA, da, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  enc(&mb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dB, db, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const int smem = 32768 + 1024 + 64;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe<<<2, 192, smem>>>(ma, mb, dO, M);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
  std::vector<float> hO(2 * 128 * NB);
  cudaMemcpy(hO.data(), dO, hO.size() * 4, cudaMemcpyDeviceToHost);
  // reference C = A x B^T for rows < M
  std::vector<float> C((size_t)Mrows * NB);
  for (int i = 0; i < Mrows; i++)
    for (int j = 0; j < NB; j++) {
      double s = 0;
      for (int k = 0; k < K; k++) s += (double)fA[(size_t)i * K + k] * fB[(size_t)j * K + k];
      C[(size_t)i * NB + j] = (float)s;
    }
  int matched = 0;
  for (int r = 0; r < 2; r++)
    for (int l = 0; l < 128; l++) {
      const float* got = &hO[((size_t)r * 128 + l) * NB];
      bool allzero = true;
      for (int j = 0; j < NB; j++) allzero &= got[j] == 0.f;
      int found = -1, coloff = -1;
      for (int i = 0; i < Mrows && found < 0; i++) {
        for (int off : {0, 128}) {  // full row, or the row's N half starting at column off
          bool ok = true;
          const int w = (off == 0) ? NB : 128;
          for (int j = 0; j < w && ok; j++) ok = std::fabs(got[j] - C[(size_t)i * NB + off + j]) < 1e-3f;
          if (ok) { found = i; coloff = off; break; }
        }
      }
      if (found >= 0) matched++;
      if (l % 16 == 0 || l == 63 || l == 64 || l == 127)
        printf("cta %d lane %3d -> %s row %d (cols from %d)\n", r, l, allzero ? "zero" : (found >= 0 ? "C" : "??"), found, coloff);
    }
  printf("M=%d matched lanes: %d\n", M, matched);
  return 0;
}
