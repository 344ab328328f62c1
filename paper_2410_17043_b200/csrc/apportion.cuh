// Copy-CTA apportioning for the dispatch / combine engine. A process drives
// n_local ranks with ctot copy CTAs in total; each group of n_local
// consecutive ranks (one process) splits its CTAs by
//   mode 0: evenly;
//   mode 1: volume -- dispatch: rows a rank sends (row sum of counts, local
//           rows included), combine: rows it returns (column sum). With all
//           ranks on one GPU this gives the hot rank the copy capacity its
//           own GPU would have; with one rank per GPU it is the identity;
//   mode 2: bandwidth -- C4 emulation: a rank's copy rate follows its
//           ClusterSpec bandwidth (core.py:179-181), quantised to 1/1024.
// Every rank gets at least one CTA; the rest is split by the largest-remainder
// rule (ties: lower rank). Host + device, integer arithmetic only, mirrored
// bit-for-bit by paper_2410_17043_b200/apportion.py.
#pragma once
#include <stdint.h>

#if !defined(AUR_HD)
#if defined(__CUDACC__)
#define AUR_HD __host__ __device__ __forceinline__
#else
#define AUR_HD inline
#endif
#endif

// per-rank weight (see above); counts row-major with row stride ld
AUR_HD long long aur_weight(const int32_t* counts, int ld, const double* bw, int n, int i, int mode, bool combine) {
  long long v = 1;
  if (mode == 1) {
    v = 0;
    for (int q = 0; q < n; q++) v += combine ? counts[q * ld + i] : counts[i * ld + q];
  } else if (mode == 2 && bw) {
    v = (long long)(bw[i] * 1024.0 + 0.5);
  }
  return v < 0 ? 0 : v;
}

// C[0..n) from per-rank weights w[0..n)
AUR_HD void aur_apportion_w(const long long* w_all, int n, int n_local, int ctot, int* C) {
  for (int g0 = 0; g0 < n; g0 += n_local) {
    const int m = n_local;
    const long long* w = w_all + g0;
    long long W = 0;
    for (int r = 0; r < m; r++) W += w[r];
    const long long spare = ctot - m;
    if (W == 0 || spare <= 0) {
      for (int r = 0; r < m; r++) C[g0 + r] = ctot / m + (r < ctot % m ? 1 : 0);
      continue;
    }
    long long given = 0, rem[32];
    for (int r = 0; r < m; r++) {
      const long long q = spare * w[r] / W;
      rem[r] = spare * w[r] - q * W;
      C[g0 + r] = 1 + (int)q;
      given += q;
    }
    for (long long left = spare - given; left > 0; left--) {  // largest remainder, lowest rank on ties
      int best = 0;
      for (int r = 1; r < m; r++)
        if (rem[r] > rem[best]) best = r;
      C[g0 + best]++;
      rem[best] = -1;
    }
  }
}

AUR_HD void aur_apportion(const int32_t* counts, const double* bw, int n, int n_local, int ctot, int mode,
                          bool combine, int* C) {
  long long w[32];
  for (int i = 0; i < n; i++) w[i] = aur_weight(counts, n, bw, n, i, mode, combine);
  aur_apportion_w(w, n, n_local, ctot, C);
}
