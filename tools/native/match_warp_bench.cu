// Cycles per perfect_matching as K2 runs it: one warp, graph rows arriving per
// lane and reduced to warp-uniform words, on the C2 decomposition graphs
// (c2_graphs.txt: P lo/hi, S lo/hi per line). FastMatch8b (fastmatch8b.cuh) vs
// FastMatch8d (fastmatch8d.cuh, the in-layer matcher); results checked equal.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>
#include "../../paper_2410_17043_b200/csrc/fastmatch8b.cuh"
#include "../../paper_2410_17043_b200/csrc/fastmatch8d.cuh"

template <int V>
__global__ void bench(const uint32_t* g, int ng, int reps, uint64_t* out, long long* cyc) {
  const int lane = threadIdx.x;
  uint64_t acc = 0;
  long long t0 = clock64();
  for (int r = 0; r < reps; r++)
    for (int i = 0; i < ng; i++) {
      const uint32_t w = g[4 * i + (lane & 3)];
      const uint32_t p0 = __shfl_sync(0xffffffffu, w, 0), p1 = __shfl_sync(0xffffffffu, w, 1);
      const uint32_t s0 = __shfl_sync(0xffffffffu, w, 2), s1 = __shfl_sync(0xffffffffu, w, 3);
      uint64_t mlb = 0;  // right->left index table (the matching)
      if constexpr (V == 0) {
        FastMatch8b f;
        f.P = ((uint64_t)p1 << 32) | p0;
        f.S = ((uint64_t)s1 << 32) | s0;
        f.run(8);
        mlb = f.MR;
      } else {
        FastMatch8d f;
        f.P = ((uint64_t)p1 << 32) | p0;
        f.S = ((uint64_t)s1 << 32) | s0;
        f.run(8);
        mlb = f.MR;
      }
      acc += mlb;
      if (r == 0 && lane == 0) out[i] = mlb;
    }
  long long t1 = clock64();
  if (lane == 0) { cyc[0] = t1 - t0; cyc[1] = (long long)acc; }
}

int main(int argc, char** argv) {
  FILE* f = fopen(argc > 1 ? argv[1] : "tools/native/c2_graphs.txt", "r");
  std::vector<uint32_t> h;
  uint32_t a, b, c, d;
  while (fscanf(f, "%u %u %u %u", &a, &b, &c, &d) == 4) { h.push_back(a); h.push_back(b); h.push_back(c); h.push_back(d); }
  const int ng = (int)h.size() / 4, reps = 8;
  uint32_t* dg; uint64_t *o0, *o1; long long* cy;
  cudaMalloc(&dg, h.size() * 4); cudaMalloc(&o0, ng * 8); cudaMalloc(&o1, ng * 8); cudaMalloc(&cy, 16);
  cudaMemcpy(dg, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  long long c0[2], c1[2];
  bench<0><<<1, 32>>>(dg, ng, 1, o0, cy);
  bench<0><<<1, 32>>>(dg, ng, reps, o0, cy);
  cudaMemcpy(c0, cy, 16, cudaMemcpyDeviceToHost);
  bench<1><<<1, 32>>>(dg, ng, 1, o1, cy);
  bench<1><<<1, 32>>>(dg, ng, reps, o1, cy);
  cudaMemcpy(c1, cy, 16, cudaMemcpyDeviceToHost);
  std::vector<uint64_t> r0(ng), r1(ng);
  cudaMemcpy(r0.data(), o0, ng * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(r1.data(), o1, ng * 8, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int i = 0; i < ng; i++) bad += r0[i] != r1[i];
  printf("graphs %d  8b %.0f  8d %.0f cyc/match  mismatches %d  err %s\n", ng, (double)c0[0] / (ng * reps),
         (double)c1[0] / (ng * reps), bad, cudaGetErrorString(cudaGetLastError()));
  return bad != 0;
}
