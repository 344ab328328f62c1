// Host check: FastMatch8e (fm8e.cuh) == FastMatch8d on 2M random graphs. g++ -O2 -std=c++17 check8e.cpp
#include <cstdint>
#include <cstdio>
#include <random>
#include "../../paper_2410_17043_b200/csrc/fastmatch8d.cuh"
#include "fm8e.cuh"
int main() {
  std::mt19937 rng(7); int bad = 0, okc = 0;
  for (int it = 0; it < 2000000; it++) {
    const int n = 1 + (int)(rng() % 8);
    uint64_t P = 0, S = 0;
    const double ps = 0.2 + 0.8 * (rng() % 1000) / 1000.0, pp = (rng() % 1000) / 1000.0;
    for (int i = 0; i < n; i++) for (int j = 0; j < n; j++)
      if ((rng() % 1000) / 1000.0 < ps) { S |= 1ull << (8 * i + j); if ((rng() % 1000) / 1000.0 < pp) P |= 1ull << (8 * i + j); }
    if (it % 3 == 0) for (int i = 0; i < n; i++) S |= 1ull << (8 * i + (i + it) % n);
    FastMatch8d a; a.P = P; a.S = S; bool oa = a.run(n);
    FastMatch8e b; b.P = P; b.S = S; bool ob = b.run(n);
    bool same = oa == ob;
    if (same && oa) for (int u = 0; u < n; u++) same &= a.ml(u, n) == b.ml(u, n);
    okc += oa;
    if (!same && bad++ < 5) printf("mismatch n=%d\n", n);
  }
  printf("bad %d (perfect %d)\n", bad, okc);
  return bad != 0;
}
