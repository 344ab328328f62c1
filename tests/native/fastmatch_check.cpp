// Host check of the K2 fast-path matcher (paper_2410_17043_b200/csrc/fastmatch.cuh)
// against the oracle's perfect_matching restatement, on random bitmask graphs.
#include <cstdint>
#include <cstdio>
#include <random>

#include "../../paper_2410_17043_b200/csrc/fastmatch.cuh"
#include "../../paper_2410_17043_b200/csrc/fastmatch8b.cuh"
#include "../../paper_2410_17043_b200/csrc/fastmatch8d.cuh"
#include "../../paper_2410_17043_b200/csrc/fastmatch16.cuh"

extern "C" int oracle_perfect_matching_masks(int n, const uint32_t* sup, const uint32_t* pref, int* perm);

template <int NB>
static int check(std::mt19937& rng, int iters) {
  int bad = 0;
  for (int it = 0; it < iters; it++) {
    const int n = 1 + (int)(rng() % NB);
    uint32_t sup[32], pref[32];
    const double ps = 0.2 + 0.8 * (rng() % 1000) / 1000.0, pp = (rng() % 1000) / 1000.0;
    for (int i = 0; i < n; i++) {
      sup[i] = pref[i] = 0;
      for (int j = 0; j < n; j++) {
        if ((rng() % 1000) / 1000.0 < ps) {
          sup[i] |= 1u << j;
          if ((rng() % 1000) / 1000.0 < pp) pref[i] |= 1u << j;
        }
      }
    }
    if (it % 3 == 0)  // balanced-matrix-like supports always have a perfect matching
      for (int i = 0; i < n; i++) sup[i] |= 1u << ((i + it) % n);
    int ref[32];
    const int ok_ref = oracle_perfect_matching_masks(n, sup, pref, ref);
    FastMatch<NB> fm;
    for (int u = 0; u < NB; u++) {
      fm.pref.set(u, u < n ? pref[u] : 0);
      fm.sup.set(u, u < n ? sup[u] : 0);
    }
    const bool ok = fm.run(n);
    bool same = ok == (bool)ok_ref;
    if (same && ok)
      for (int u = 0; u < n; u++) same &= (int)fm.ml.get(u) == ref[u];
    if (!same && bad++ < 5) {
      std::printf("mismatch NB=%d n=%d ok=%d/%d\n", NB, n, (int)ok, ok_ref);
    }
  }
  return bad;
}

static int check8(std::mt19937& rng, int iters) {
  int bad = 0;
  for (int it = 0; it < iters; it++) {
    const int n = 1 + (int)(rng() % 8);
    uint32_t sup[32], pref[32];
    const double ps = 0.2 + 0.8 * (rng() % 1000) / 1000.0, pp = (rng() % 1000) / 1000.0;
    for (int i = 0; i < n; i++) {
      sup[i] = pref[i] = 0;
      for (int j = 0; j < n; j++)
        if ((rng() % 1000) / 1000.0 < ps) {
          sup[i] |= 1u << j;
          if ((rng() % 1000) / 1000.0 < pp) pref[i] |= 1u << j;
        }
    }
    if (it % 3 == 0)
      for (int i = 0; i < n; i++) sup[i] |= 1u << ((i + it) % n);
    int ref[32];
    const int ok_ref = oracle_perfect_matching_masks(n, sup, pref, ref);
    FastMatch8 fm;
    fm.pref[0] = fm.pref[1] = fm.sup[0] = fm.sup[1] = 0;
    for (int u = 0; u < n; u++) {
      FastMatch8::setb(fm.pref, u, pref[u]);
      FastMatch8::setb(fm.sup, u, sup[u]);
    }
    const bool ok = fm.run(n);
    bool same = ok == (bool)ok_ref;
    if (same && ok)
      for (int u = 0; u < n; u++) same &= (int)FastMatch8::getn(fm.ml, u) == ref[u];
    if (!same && bad++ < 5) std::printf("mismatch FastMatch8 n=%d ok=%d/%d\n", n, (int)ok, ok_ref);
    // the K2 fast path (shift-register stacks, byte tables)
    FastMatch8b fb;
    fb.P = fb.S = 0;
    for (int u = 0; u < n; u++) {
      fb.P |= (uint64_t)pref[u] << (8 * u);
      fb.S |= (uint64_t)sup[u] << (8 * u);
    }
    const bool okb = fb.run(n);
    bool sameb = okb == (bool)ok_ref;
    if (sameb && okb)
      for (int u = 0; u < n; u++) sameb &= (int)((fb.ML >> (8 * u)) & 15) == ref[u];
    if (!sameb && bad++ < 5) std::printf("mismatch FastMatch8b n=%d ok=%d/%d\n", n, (int)okb, ok_ref);
    // the K2 in-layer matcher (no candidate stacks)
    FastMatch8d fd;
    fd.P = fb.P;
    fd.S = 0;
    for (int u = 0; u < n; u++) fd.S |= (uint64_t)sup[u] << (8 * u);
    const bool okd = fd.run(n);
    bool samed = okd == (bool)ok_ref;
    if (samed && okd)
      for (int u = 0; u < n; u++) {
        samed &= (int)fd.ml((uint32_t)u, n) == ref[u];
        if (!fd.kuhned) samed &= (int)((fd.MLB >> (8 * u)) & 0xFF) == (1 << ref[u]);
      }
    if (!samed && bad++ < 5) std::printf("mismatch FastMatch8d n=%d ok=%d/%d\n", n, (int)okd, ok_ref);
  }
  return bad;
}

// the n <= 16 K2 matcher (16-bit lanes, shift-register stacks)
static int check16(std::mt19937& rng, int iters) {
  int bad = 0;
  for (int it = 0; it < iters; it++) {
    const int n = 1 + (int)(rng() % 16);
    uint32_t sup[32], pref[32];
    const double ps = 0.2 + 0.8 * (rng() % 1000) / 1000.0, pp = (rng() % 1000) / 1000.0;
    for (int i = 0; i < n; i++) {
      sup[i] = pref[i] = 0;
      for (int j = 0; j < n; j++)
        if ((rng() % 1000) / 1000.0 < ps) {
          sup[i] |= 1u << j;
          if ((rng() % 1000) / 1000.0 < pp) pref[i] |= 1u << j;
        }
    }
    if (it % 3 == 0)
      for (int i = 0; i < n; i++) sup[i] |= 1u << ((i + it) % n);
    int ref[32];
    const int ok_ref = oracle_perfect_matching_masks(n, sup, pref, ref);
    FastMatch16 f;
    f.P.clear();
    f.S.clear();
    for (int u = 0; u < n; u++) {
      FastMatch16::set_lane(f.P, (uint32_t)u, pref[u]);
      FastMatch16::set_lane(f.S, (uint32_t)u, sup[u]);
    }
    const bool ok = f.run(n);
    bool same = ok == (bool)ok_ref;
    if (same && ok)
      for (int u = 0; u < n; u++) same &= (int)FastMatch16::nib(f.ML, u) == ref[u];
    if (!same && bad++ < 5) std::printf("mismatch FastMatch16 n=%d ok=%d/%d\n", n, (int)ok, ok_ref);
  }
  return bad;
}

int main() {
  std::mt19937 rng(12345);
  int bad = check<8>(rng, 200000) + check<16>(rng, 100000) + check8(rng, 600000) + check16(rng, 300000);
  std::printf("fastmatch mismatches: %d\n", bad);
  return bad != 0;
}
