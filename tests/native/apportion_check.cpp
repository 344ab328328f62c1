// Host run of csrc/apportion.cuh for tests/test_apportion_cpu.py: reads cases
// "n n_local ctot mode combine bw[n] counts[n*n]" from stdin, prints C[n].
#include <cstdint>
#include <cstdio>
#include "../../paper_2410_17043_b200/csrc/apportion.cuh"

int main() {
  int n, nl, ctot, mode, comb;
  while (std::scanf("%d %d %d %d %d", &n, &nl, &ctot, &mode, &comb) == 5) {
    double bw[32];
    int32_t counts[32 * 32];
    for (int i = 0; i < n; i++) std::scanf("%lf", &bw[i]);
    for (int i = 0; i < n * n; i++) std::scanf("%d", &counts[i]);
    int C[32];
    aur_apportion(counts, bw, n, nl, ctot, mode, comb != 0, C);
    for (int i = 0; i < n; i++) std::printf("%d%c", C[i], i + 1 < n ? ' ' : '\n');
  }
  return 0;
}
