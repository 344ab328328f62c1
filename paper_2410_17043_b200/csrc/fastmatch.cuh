// Register-resident Hopcroft-Karp + Kuhn perfect matching for n <= 16, the
// exact restatement of moeplan.matching.perfect_matching (matching.py:20-112)
// used by the K2 fast path. Host+device so tests/cpu can check it against the
// oracle without a GPU.
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define AUR_HD __host__ __device__ __forceinline__
#else
#define AUR_HD inline
#endif

AUR_HD int aur_ffs(uint32_t x) {
#if defined(__CUDA_ARCH__)
  return __ffs((int)x);
#else
  return __builtin_ffs((int)x);
#endif
}

// W 32-bit words holding fields of BITS bits (BITS divides 32). 32-bit words
// keep every get/set to a shift, a mask and (W > 1) a short select chain.
template <int BITS, int W>
struct Pk {
  uint32_t w[W];
  static constexpr unsigned PER = 32 / BITS;
  static constexpr uint32_t FM = (BITS == 32) ? ~0u : ((1u << BITS) - 1);
  AUR_HD void fill(uint32_t v) {
#pragma unroll
    for (int k = 0; k < W; k++) w[k] = v;
  }
  AUR_HD uint32_t get(unsigned idx) const {
    const unsigned wi = idx / PER, sh = (idx % PER) * BITS;
    uint32_t r = w[0];
#pragma unroll
    for (unsigned k = 1; k < W; k++)
      if (wi == k) r = w[k];
    return (r >> sh) & FM;
  }
  AUR_HD void set(unsigned idx, uint32_t v) {
    const unsigned wi = idx / PER, sh = (idx % PER) * BITS;
    const uint32_t m = FM << sh, nv = (v & FM) << sh;
#pragma unroll
    for (unsigned k = 0; k < W; k++)
      if (wi == k) w[k] = (w[k] & ~m) | nv;
  }
};

template <int NB>
struct FastMatch {
  static constexpr int MW = NB * NB / 32;        // words of NB-bit masks
  static constexpr int NW = NB * 4 / 32;         // words of nibble arrays
  static constexpr int DB = NB <= 8 ? 4 : 8;     // bits per BFS distance
  static constexpr int DW = NB * DB / 32;
  static constexpr uint32_t DINF = (1u << DB) - 1;  // _INF
  Pk<NB, MW> pref, sup;   // adjacency masks per left vertex
  Pk<4, NW> ml, mr;       // matches (valid where the free bit is clear)
  uint32_t freeL, freeR;
  Pk<DB, DW> dist;        // BFS level, DINF = _INF
  Pk<4, NW> us, vs;       // DFS stack: vertex and chosen right vertex per depth
  Pk<NB, MW> left;        // DFS stack: candidates still to try per depth

  AUR_HD void augment_path(int top, int v) {
    vs.set(top, v);
    for (int l = top; l >= 0; l--) {
      const int uu = (int)us.get(l), vv = (int)vs.get(l);
      ml.set(uu, vv);
      mr.set(vv, uu);
    }
    freeL &= ~(1u << (int)us.get(0));
    freeR &= ~(1u << v);
  }

  // hopcroft_karp dfs(root), matching.py:57-65. A vertex on the stack at depth
  // d has BFS distance d (roots are free, dist 0; children need dist[u] + 1),
  // so dist[u] + 1 == depth + 1.
  AUR_HD bool hk_dfs(int root) {
    int top = 0;
    us.set(0, root);
    left.set(0, pref.get(root));
    while (top >= 0) {
      const uint32_t m = (uint32_t)left.get(top);
      if (m == 0) {
        dist.set(us.get(top), DINF);
        top--;
        continue;
      }
      const int v = aur_ffs(m) - 1;
      left.set(top, m & (m - 1));
      if ((freeR >> v) & 1) {
        augment_path(top, v);
        return true;
      }
      const int w = (int)mr.get(v);
      if ((int)dist.get(w) == top + 1) {
        vs.set(top, v);
        top++;
        us.set(top, w);
        left.set(top, pref.get(w));
      }
    }
    return false;
  }

  // perfect_matching's augment(u, seen), matching.py:96-106
  AUR_HD bool kuhn(int root) {
    uint32_t seen = 0;
    int top = 0;
    us.set(0, root);
    left.set(0, sup.get(root));
    while (top >= 0) {
      const uint32_t m = (uint32_t)left.get(top) & ~seen;
      if (m == 0) {
        top--;
        continue;
      }
      const int v = aur_ffs(m) - 1;
      left.set(top, m & (m - 1));
      seen |= 1u << v;
      if ((freeR >> v) & 1) {
        augment_path(top, v);
        return true;
      }
      vs.set(top, v);
      top++;
      us.set(top, (int)mr.get(v));
      left.set(top, sup.get((int)mr.get(v)));
    }
    return false;
  }

  AUR_HD bool run(int n) {
    const uint32_t all = (1u << n) - 1;
    freeL = all;
    freeR = all;
    ml.fill(0);
    mr.fill(0);
    // First Hopcroft-Karp phase in closed form: every left vertex is free, so
    // bfs() gives all of them dist 0 and finds a free right vertex iff some
    // preferred edge exists; dfs(u) can then only accept a free right vertex
    // (a matched w has dist 0 != dist[u] + 1), i.e. it takes the lowest free
    // preferred v -- a greedy pass in index order. The dist[u] = _INF marks it
    // leaves behind are recomputed by the next bfs().
    uint32_t any_pref = 0;
#pragma unroll
    for (int u = 0; u < NB; u++) any_pref |= pref.get(u);
    if (!any_pref) goto kuhn_phase;
#pragma unroll
    for (int u = 0; u < NB; u++) {
      const uint32_t m = pref.get(u) & freeR;
      if (u < n && m) {
        const int v = aur_ffs(m) - 1;
        ml.set(u, v);
        mr.set(v, u);
        freeL &= ~(1u << u);
        freeR &= ~(1u << v);
      }
    }
    for (;;) {  // hopcroft_karp main loop, matching.py:67-72
      uint32_t frontier = freeL;
#pragma unroll
      for (int u = 0; u < NB; u++)
        if (u < n) dist.set(u, ((freeL >> u) & 1) ? 0 : DINF);
      bool found = false;
      int level = 0;
      while (frontier) {
        uint32_t reach = 0;
        for (uint32_t f = frontier; f; f &= f - 1) reach |= (uint32_t)pref.get(aur_ffs(f) - 1);
        if (reach & freeR) found = true;
        uint32_t next = 0;
        for (uint32_t r = reach & ~freeR; r; r &= r - 1) {
          const int w = (int)mr.get(aur_ffs(r) - 1);
          if (dist.get(w) == DINF) {
            dist.set(w, level + 1);
            next |= 1u << w;
          }
        }
        frontier = next;
        level++;
      }
      if (!found) break;
      for (int u = 0; u < n; u++)
        if ((freeL >> u) & 1) hk_dfs(u);
    }
  kuhn_phase:
    for (int u = 0; u < n; u++)
      if (((freeL >> u) & 1) && !kuhn(u)) return false;
    return true;
  }
};

// n <= 8 specialisation. Adjacency rows, DFS candidate stacks and BFS layers
// are bytes of two 32-bit words, matches nibbles of one word, and a
// byte-per-right-vertex copy of the match (mrb) turns every BFS level into a
// handful of SWAR operations: reach = OR of the frontier's rows, next =
// partners of the matched vertices reached. dist[w] == dist[u] + 1 becomes
// "w is on BFS layer depth+1 and its dfs has not failed" (a vertex on the DFS
// stack at depth d has BFS distance d).
struct FastMatch8 {
  uint32_t pref[2], sup[2];
  uint32_t ml, mr;
  uint32_t mrb[2];
  uint32_t freeL, freeR;
  uint32_t layer[2];
  uint32_t alive;
  uint32_t us, vs;
  uint32_t left[2];

  AUR_HD static uint32_t getb(const uint32_t (&a)[2], int i) {
    return ((i < 4 ? a[0] : a[1]) >> ((i & 3) * 8)) & 0xFFu;
  }
  AUR_HD static void setb(uint32_t (&a)[2], int i, uint32_t v) {
    const int sh = (i & 3) * 8;
    const uint32_t m = 0xFFu << sh;
    if (i < 4) a[0] = (a[0] & ~m) | (v << sh);
    else a[1] = (a[1] & ~m) | (v << sh);
  }
  AUR_HD static uint32_t getn(uint32_t w, int i) { return (w >> (4 * i)) & 15u; }
  AUR_HD static void setn(uint32_t& w, int i, uint32_t v) {
    w = (w & ~(15u << (4 * i))) | (v << (4 * i));
  }
  // bit b of a 4-bit value -> 0xFF in byte b
  AUR_HD static uint32_t spread4(uint32_t b) { return ((b * 0x00204081u) & 0x01010101u) * 0xFFu; }
  // OR of the bytes of a[] whose index is set in mask
  AUR_HD static uint32_t gather_or(const uint32_t (&a)[2], uint32_t mask) {
    uint32_t r = (a[0] & spread4(mask & 15u)) | (a[1] & spread4((mask >> 4) & 15u));
    r |= r >> 16;
    r |= r >> 8;
    return r & 0xFFu;
  }
  AUR_HD void match(int u, int v) {
    setn(ml, u, v);
    setn(mr, v, u);
    setb(mrb, v, 1u << u);
  }
  AUR_HD void augment_path(int top, int v) {
    setn(vs, top, v);
    for (int l = top; l >= 0; l--) match((int)getn(us, l), (int)getn(vs, l));
    freeL &= ~(1u << getn(us, 0));
    freeR &= ~(1u << v);
  }
  AUR_HD bool hk_dfs(int root) {  // matching.py:57-65
    int top = 0;
    setn(us, 0, root);
    setb(left, 0, getb(pref, root));
    while (top >= 0) {
      const uint32_t m = getb(left, top);
      if (!m) {
        alive &= ~(1u << getn(us, top));  // dist[u] = _INF
        top--;
        continue;
      }
      const int v = aur_ffs(m) - 1;
      setb(left, top, m & (m - 1));
      if ((freeR >> v) & 1u) {
        augment_path(top, v);
        return true;
      }
      const int w = (int)getn(mr, v);
      if (top + 1 < 8 && (((getb(layer, top + 1) & alive) >> w) & 1u)) {
        setn(vs, top, v);
        top++;
        setn(us, top, w);
        setb(left, top, getb(pref, w));
      }
    }
    return false;
  }
  AUR_HD bool kuhn(int root) {  // matching.py:96-106
    uint32_t seen = 0;
    int top = 0;
    setn(us, 0, root);
    setb(left, 0, getb(sup, root));
    while (top >= 0) {
      const uint32_t m = getb(left, top) & ~seen;
      if (!m) {
        top--;
        continue;
      }
      const int v = aur_ffs(m) - 1;
      setb(left, top, m & (m - 1));
      seen |= 1u << v;
      if ((freeR >> v) & 1u) {
        augment_path(top, v);
        return true;
      }
      const int w = (int)getn(mr, v);
      setn(vs, top, v);
      top++;
      setn(us, top, w);
      setb(left, top, getb(sup, w));
    }
    return false;
  }
  // pref / sup rows must be zero beyond n
  AUR_HD bool run(int n) {
    const uint32_t all = (1u << n) - 1;
    freeL = freeR = all;
    ml = mr = 0;
    mrb[0] = mrb[1] = 0;
    if (pref[0] | pref[1]) {
      // first Hopcroft-Karp phase: all left free -> greedy lowest free preferred vertex
      for (int u = 0; u < n; u++) {
        const uint32_t m = getb(pref, u) & freeR;
        if (m) {
          const int v = aur_ffs(m) - 1;
          match(u, v);
          freeL &= ~(1u << u);
          freeR &= ~(1u << v);
        }
      }
      for (;;) {
        layer[0] = layer[1] = 0;
        uint32_t frontier = freeL, visited = freeL;
        setb(layer, 0, frontier);
        bool found = false;
        int level = 0;
        while (frontier) {  // bfs(), matching.py:37-55, one SWAR step per level
          const uint32_t reach = gather_or(pref, frontier);
          found |= (reach & freeR) != 0;
          const uint32_t nxt = gather_or(mrb, reach & ~freeR) & ~visited;
          visited |= nxt;
          level++;
          if (level < 8) setb(layer, level, nxt);
          frontier = nxt;
        }
        if (!found) break;
        alive = all;
        for (int u = 0; u < n; u++)
          if ((freeL >> u) & 1u) hk_dfs(u);
      }
    }
    for (int u = 0; u < n; u++)
      if (((freeL >> u) & 1u) && !kuhn(u)) return false;
    return true;
  }
};
