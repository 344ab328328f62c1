// Cycles per perfect_matching on the C2 decomposition graphs (one thread), for
// the K2 matchers: FastMatch8 (fastmatch.cuh) vs FastMatch8b (fastmatch8b.cuh).
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>
#include "../../paper_2410_17043_b200/csrc/fastmatch.cuh"
#include "../../paper_2410_17043_b200/csrc/fastmatch8b.cuh"
#ifdef PROFILE
#include "/tmp/k2/fm8p.cuh"
#endif

__global__ void bench(const uint32_t* g, int ng, int reps, uint32_t* out_a, uint64_t* out_b, long long* cyc) {
  long long t0 = clock64();
  uint32_t acc = 0;
  for (int r = 0; r < reps; r++)
    for (int i = 0; i < ng; i++) {
      FastMatch8 f;
      f.pref[0] = g[4 * i] ^ (acc & 0);
      f.pref[1] = g[4 * i + 1];
      f.sup[0] = g[4 * i + 2];
      f.sup[1] = g[4 * i + 3];
      f.run(8);
      acc += f.ml;
      if (r == 0) out_a[i] = f.ml;
    }
  long long t1 = clock64();
  for (int r = 0; r < reps; r++)
    for (int i = 0; i < ng; i++) {
      FastMatch8b f;
      f.P = ((uint64_t)g[4 * i + 1] << 32) | (g[4 * i] ^ (acc & 0));
      f.S = ((uint64_t)g[4 * i + 3] << 32) | g[4 * i + 2];
      f.run(8);
      acc += (uint32_t)f.ML;
      if (r == 0) out_b[i] = f.ML;
    }
  long long t2 = clock64();
  long long t3 = clock64();
#ifdef PROFILE
  long long cg = 0, ch = 0, ck = 0;
  for (int i = 0; i < ng; i++) {
    FastMatch8p f;
    f.P = ((uint64_t)g[4 * i + 1] << 32) | g[4 * i];
    f.S = ((uint64_t)g[4 * i + 3] << 32) | g[4 * i + 2];
    f.run(8);
    cg += f.cg; ch += f.ch; ck += f.ck;
  }
  printf("8b sections per match: greedy %lld  hk %lld  kuhn %lld\n", cg / ng, ch / ng, ck / ng);
#endif
  cyc[0] = t1 - t0;
  cyc[1] = t2 - t1;
  cyc[3] = t3 - t2;
  cyc[2] = acc;
}

int main(int argc, char** argv) {
  FILE* f = fopen(argc > 1 ? argv[1] : "tools/native/c2_graphs.txt", "r");
  std::vector<uint32_t> h;
  uint32_t a, b, c, d;
  while (fscanf(f, "%u %u %u %u", &a, &b, &c, &d) == 4) { h.push_back(a); h.push_back(b); h.push_back(c); h.push_back(d); }
  const int ng = (int)h.size() / 4, reps = 4;
  uint32_t *dg, *oa; uint64_t* ob; long long* cy;
  cudaMalloc(&dg, h.size() * 4); cudaMalloc(&oa, ng * 8); cudaMalloc(&ob, ng * 8); cudaMalloc(&cy, 32);
  cudaMemcpy(dg, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  bench<<<1, 1>>>(dg, ng, 1, oa, ob, cy);
  bench<<<1, 1>>>(dg, ng, reps, oa, ob, cy);
  std::vector<uint32_t> ra(2 * ng); std::vector<uint64_t> rb(ng); long long hc[4];
  cudaMemcpy(ra.data(), oa, ng * 8, cudaMemcpyDeviceToHost); cudaMemcpy(rb.data(), ob, ng * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(hc, cy, 32, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int i = 0; i < ng; i++) {
    uint32_t nb = 0;
    for (int u = 0; u < 8; u++) nb |= (uint32_t)((rb[i] >> (8 * u)) & 15) << (4 * u);
    if (nb != ra[i]) bad++;
  }
  printf("graphs %d  FastMatch8 %.0f  FastMatch8b %.0f cyc/match  mismatches %d\n", ng,
         (double)hc[0] / (ng * reps), (double)hc[1] / (ng * reps), bad);
  return bad != 0;
}
