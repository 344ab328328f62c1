// Cycles per perfect_matching section (greedy + tables, bfs, build_vb, HK dfs, Kuhn) of FastMatch8d on the
// C2 decomposition graphs (one warp), and the branch-light DFS variant FastMatch8e (fm8e.cuh, one exit test
// per step, push / pop by selects) for comparison. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
// -std=c++17 -DHAVE_8E -o match_sections match_sections.cu; run: ./match_sections c2_graphs.txt
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>
#include "fm8d_prof.cuh"
#undef AUR_HD
#include "../../paper_2410_17043_b200/csrc/fastmatch8d.cuh"
#ifdef HAVE_8E
#include "fm8e.cuh"
#endif
#include "fm8f.cuh"
template <class M>
__global__ void bench(const uint32_t* g, int ng, int reps, uint64_t* out, long long* cyc) {
  const int lane = threadIdx.x;
  uint64_t acc = 0;
  long long sec[5] = {0, 0, 0, 0, 0};
  long long t0 = clock64();
  for (int r = 0; r < reps; r++)
    for (int i = 0; i < ng; i++) {
      const uint32_t w = g[4 * i + (lane & 3)];
      const uint32_t p0 = __shfl_sync(0xffffffffu, w, 0), p1 = __shfl_sync(0xffffffffu, w, 1);
      const uint32_t s0 = __shfl_sync(0xffffffffu, w, 2), s1 = __shfl_sync(0xffffffffu, w, 3);
      M f;
      f.P = ((uint64_t)p1 << 32) | p0;
      f.S = ((uint64_t)s1 << 32) | s0;
      f.run(8);
      if constexpr (sizeof(M) == sizeof(FastMatch8dP)) for (int k = 0; k < 5; k++) sec[k] += ((FastMatch8dP*)&f)->sec[k];
      acc += f.MR;
      if (r == 0 && lane == 0) out[i] = f.MR;
    }
  long long t1 = clock64();
  if (lane == 0) { cyc[0] = t1 - t0; cyc[1] = (long long)acc; for (int k = 0; k < 5; k++) cyc[2 + k] = sec[k]; }
}
template <class M>
double run(const uint32_t* dg, int ng, uint64_t* o, long long* cy, long long* h) {
  const int reps = 8;
  bench<M><<<1, 32>>>(dg, ng, 1, o, cy);
  bench<M><<<1, 32>>>(dg, ng, reps, o, cy);
  cudaMemcpy(h, cy, 7 * 8, cudaMemcpyDeviceToHost);
  return (double)h[0] / (ng * reps);
}
int main(int argc, char** argv) {
  FILE* f = fopen(argc > 1 ? argv[1] : "tools/native/c2_graphs.txt", "r");
  std::vector<uint32_t> h;
  uint32_t a, b, c, d;
  while (fscanf(f, "%u %u %u %u", &a, &b, &c, &d) == 4) { h.push_back(a); h.push_back(b); h.push_back(c); h.push_back(d); }
  const int ng = (int)h.size() / 4;
  uint32_t* dg; uint64_t *o0, *o1; long long* cy; long long hc[7];
  cudaMalloc(&dg, h.size() * 4); cudaMalloc(&o0, ng * 8); cudaMalloc(&o1, ng * 8); cudaMalloc(&cy, 64);
  cudaMemcpy(dg, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  double c8d = run<FastMatch8d>(dg, ng, o0, cy, hc);
  double cp = run<FastMatch8dP>(dg, ng, o1, cy, hc);
  printf("8d %.0f cyc/match; profiled %.0f: greedy %.0f bfs %.0f vb %.0f dfs %.0f kuhn %.0f\n", c8d, cp,
         hc[2] / (ng * 8.0), hc[3] / (ng * 8.0), hc[4] / (ng * 8.0), hc[5] / (ng * 8.0), hc[6] / (ng * 8.0));
#ifdef HAVE_8E
  double ce = run<FastMatch8e>(dg, ng, o1, cy, hc);
  std::vector<uint64_t> r0(ng), r1(ng);
  cudaMemcpy(r0.data(), o0, ng * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(r1.data(), o1, ng * 8, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int i = 0; i < ng; i++) bad += r0[i] != r1[i];
  printf("8e %.0f cyc/match, mismatches %d\n", ce, bad);
#endif
  {
    double cf = run<FastMatch8f>(dg, ng, o1, cy, hc);
    std::vector<uint64_t> r0(ng), r1(ng);
    cudaMemcpy(r0.data(), o0, ng * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(r1.data(), o1, ng * 8, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int i = 0; i < ng; i++) bad += r0[i] != r1[i];
    printf("8f (lane-parallel bfs) %.0f cyc/match, mismatches %d\n", cf, bad);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
