// Probe: 2-D TMA tile::gather4 into a 128B-swizzled shared buffer vs the plain
// tile load of the same rows (box {64 cols, R rows}); prints mismatches.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda.h>
#include <cuda_runtime.h>

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k(const __grid_constant__ CUtensorMap mg, const __grid_constant__ CUtensorMap mt, const int* rows,
                  uint8_t* out_g, uint8_t* out_t) {
  __shared__ __align__(1024) uint8_t bg[128 * 128], bt[128 * 128];
  __shared__ __align__(8) uint64_t bar[2];
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar[0])), "r"(128 * 128) : "memory");
    for (int j = 0; j < 32; j++)
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                   :: "r"(su(bg + j * 512)), "l"(&mg), "r"(0), "r"(rows[4 * j]), "r"(rows[4 * j + 1]), "r"(rows[4 * j + 2]),
                      "r"(rows[4 * j + 3]), "r"(su(&bar[0])) : "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar[1])), "r"(128 * 128) : "memory");
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 :: "r"(su(bt)), "l"(&mt), "r"(0), "r"(0), "r"(su(&bar[1])) : "memory");
    for (int b = 0; b < 2; b++)
      asm volatile("{\n\t.reg .pred P1;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W_%=;\n\t}" ::"r"(su(&bar[b])) : "memory");
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 128 * 128; i += blockDim.x) { out_g[i] = bg[i]; out_t[i] = bt[i]; }
}

int main() {
  const int R = 1024, C = 64;  // bf16 matrix R x C (128 B rows)
  std::vector<uint16_t> h(R * C);
  for (int i = 0; i < R * C; i++) h[i] = (uint16_t)(i * 2654435761u >> 16);
  uint16_t* dx; cudaMalloc(&dx, R * C * 2); cudaMemcpy(dx, h.data(), R * C * 2, cudaMemcpyHostToDevice);
  // gather rows: identity 0..127 so the gathered tile must equal the plain tile
  std::vector<int> rows(128); for (int i = 0; i < 128; i++) rows[i] = i;
  int* dr; cudaMalloc(&dr, 512); cudaMemcpy(dr, rows.data(), 512, cudaMemcpyHostToDevice);
  EncFn enc; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  for (int box_rows_g : {1, 4}) {
    CUtensorMap mg, mt;
    cuuint64_t dims[2] = {(cuuint64_t)C, (cuuint64_t)R}, str[1] = {(cuuint64_t)C * 2};
    cuuint32_t boxg[2] = {64, (cuuint32_t)box_rows_g}, boxt[2] = {64, 128}, es[2] = {1, 1};
    CUresult r1 = enc(&mg, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dx, dims, str, boxg, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    CUresult r2 = enc(&mt, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dx, dims, str, boxt, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    uint8_t *og, *ot; cudaMalloc(&og, 16384); cudaMalloc(&ot, 16384);
    cudaMemset(og, 0, 16384); cudaMemset(ot, 0, 16384);
    k<<<1, 128>>>(mg, mt, dr, og, ot);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<uint8_t> hg(16384), ht(16384);
    cudaMemcpy(hg.data(), og, 16384, cudaMemcpyDeviceToHost); cudaMemcpy(ht.data(), ot, 16384, cudaMemcpyDeviceToHost);
    int bad = 0; for (int i = 0; i < 16384; i++) bad += hg[i] != ht[i];
    printf("gather box rows %d: encode %d/%d, kernel %s, bytes differing from the tile load: %d\n", box_rows_g, (int)r1,
           (int)r2, cudaGetErrorString(e), bad);
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
