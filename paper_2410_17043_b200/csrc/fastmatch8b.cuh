// n <= 8 perfect_matching (matching.py:75-112) tuned for one GPU thread: the
// same visiting order as FastMatch8 (fastmatch.cuh) with every DFS stack a
// shift register (push = shift left + or, pop = shift right: no variable
// shifts), adjacency rows / matches / BFS layers as bytes of 64-bit words read
// with byte permutes, and candidates handled as one-hot bits.
#pragma once
#include <stdint.h>

#if !defined(AUR_HD)
#if defined(__CUDACC__)
#define AUR_HD __host__ __device__ __forceinline__
#else
#define AUR_HD inline
#endif
#endif

struct FastMatch8b {
  uint64_t P, S;      // pref / sup rows: byte u = right-vertex mask of left u
  uint64_t MR;        // byte v = left vertex matched to right v (index)
  uint64_t MRB;       // byte v = one-hot left vertex matched to v (0: free)
  uint64_t MLB;       // byte u = one-hot right vertex matched to u (0: free)
  uint64_t ML;        // byte u = right vertex matched to u
  uint64_t LAY;       // byte d = BFS layer d (left vertices)
  uint32_t freeL, freeR, alive;

  AUR_HD static uint32_t byte_of(uint64_t x, uint32_t i) {
#if defined(__CUDA_ARCH__)
    return __byte_perm((uint32_t)x, (uint32_t)(x >> 32), i) & 0xFFu;
#else
    return (uint32_t)(x >> (8 * i)) & 0xFFu;
#endif
  }
  AUR_HD static uint64_t set_byte(uint64_t x, uint32_t i, uint32_t v) {
    const uint32_t sh = 8 * i;
    return (x & ~(0xFFull << sh)) | ((uint64_t)v << sh);
  }
  AUR_HD static uint32_t idx(uint32_t onehot) {
#if defined(__CUDA_ARCH__)
    return (uint32_t)(__ffs((int)onehot) - 1);
#else
    return (uint32_t)__builtin_ctz(onehot);
#endif
  }
  AUR_HD static uint32_t or_bytes(uint64_t x) {
    uint32_t r = (uint32_t)x | (uint32_t)(x >> 32);
    r |= r >> 16;
    r |= r >> 8;
    return r & 0xFFu;
  }
  // OR of the bytes of a whose index is set in mask
  AUR_HD static uint32_t gather_or(uint64_t a, uint32_t mask) {
    const uint32_t lo = ((mask & 15u) * 0x00204081u & 0x01010101u) * 0xFFu;
    const uint32_t hi = (((mask >> 4) & 15u) * 0x00204081u & 0x01010101u) * 0xFFu;
    uint32_t r = ((uint32_t)a & lo) | ((uint32_t)(a >> 32) & hi);
    r |= r >> 16;
    r |= r >> 8;
    return r & 0xFFu;
  }
  AUR_HD void match(uint32_t u, uint32_t v) {
    ML = set_byte(ML, u, v);
    MR = set_byte(MR, v, u);
    MRB = set_byte(MRB, v, 1u << u);
    MLB = set_byte(MLB, u, 1u << v);
  }
  // path: U nibbles = us[top..0] (low = top), V nibbles = vs[top-1..0], final right vertex v
  AUR_HD void augment(uint32_t U, uint32_t V, uint32_t v, int top) {
    for (int l = top; l >= 0; l--) {
      match(U & 15u, v);
      U >>= 4;
      v = V & 15u;
      V >>= 4;
    }
    // U now holds nothing; the root is the last u matched
  }

  // hopcroft_karp dfs(root), matching.py:57-65, with masked candidates: at
  // depth d only v that are free or whose partner sits on layer d+1 and is
  // alive can be taken; every other v would be skipped by the loop with no
  // side effect, and can never become viable again within this dfs (alive
  // only shrinks, layers and the matching are fixed until it augments), so
  // they are dropped up front. Viability is re-checked at every visit
  // (partners may die while a sibling is explored).
  AUR_HD bool hk_dfs(uint32_t root) {
    uint64_t L = byte_of(P, root);  // candidate stack, top at the low byte
    uint32_t U = root, V = 0;       // vertex stack / chosen right vertices
    int top = 0;
    for (;;) {
      const uint32_t nl = top + 1 < 8 ? byte_of(LAY, top + 1) & alive : 0u;
      const uint32_t m = (uint32_t)L & 0xFFu & (freeR | gather_or(MLB, nl));
      if (!m) {
        alive &= ~(1u << (U & 15u));  // dist[u] = _INF
        if (top == 0) return false;
        L >>= 8;
        U >>= 4;
        V >>= 4;
        top--;
        continue;
      }
      const uint32_t b = m & (0u - m);
      L = (L & ~0xFFull) | (m ^ b);
      const uint32_t v = idx(b);
      if (freeR & b) {
        augment(U, V, v, top);
        freeL &= ~(1u << root);
        freeR &= ~b;
        return true;
      }
      const uint32_t w = byte_of(MR, v);  // on layer top+1 and alive, by the mask
      L = (L << 8) | byte_of(P, w);
      U = (U << 4) | w;
      V = (V << 4) | v;
      top++;
    }
  }

  AUR_HD bool kuhn(uint32_t root) {
    uint32_t seen = 0;
    uint64_t L = byte_of(S, root);
    uint32_t U = root, V = 0;
    int top = 0;
    for (;;) {
      const uint32_t m = (uint32_t)L & ~seen & 0xFFu;
      if (!m) {
        if (top == 0) return false;
        L >>= 8;
        U >>= 4;
        V >>= 4;
        top--;
        continue;
      }
      const uint32_t b = m & (0u - m);
      L ^= b;
      seen |= b;
      const uint32_t v = idx(b);
      if (freeR & b) {
        augment(U, V, v, top);
        freeL &= ~(1u << root);
        freeR &= ~b;
        return true;
      }
      const uint32_t w = byte_of(MR, v);
      L = (L << 8) | byte_of(S, w);
      U = (U << 4) | w;
      V = (V << 4) | v;
      top++;
    }
  }

  // rows beyond n must be zero; result: ML bytes
  AUR_HD bool run(int n) {
    const uint32_t all = (1u << n) - 1;
    freeL = freeR = all;
    ML = MR = MRB = MLB = 0;
    if (P) {
      // first Hopcroft-Karp phase: all left free -> greedy lowest free preferred
      // vertex. The chain through freeR is four ALU ops per row; the match
      // tables are built afterwards from independent per-row results.
      uint32_t b[8];
#pragma unroll
      for (int u = 0; u < 8; u++) {
        const uint32_t m = byte_of(P, u) & freeR;
        b[u] = m & (0u - m);
        freeR &= ~b[u];
      }
      uint64_t mrb = 0, mlb = 0;
#pragma unroll
      for (int u = 0; u < 8; u++) {
        if (b[u]) {
          const uint32_t v = idx(b[u]);
          ML |= (uint64_t)v << (8 * u);
          MR |= (uint64_t)u << (8 * v);
          mrb |= (uint64_t)(1u << u) << (8 * v);
          mlb |= (uint64_t)b[u] << (8 * u);
          freeL &= ~(1u << u);
        }
      }
      MRB = mrb;
      MLB = mlb;
      for (;;) {
        uint32_t frontier = freeL, visited = freeL;
        LAY = frontier;
        bool found = false;
        int level = 0;
        while (frontier) {  // bfs(), matching.py:37-55, one SWAR step per level
          const uint32_t reach = gather_or(P, frontier);
          found |= (reach & freeR) != 0;
          const uint32_t nxt = gather_or(MRB, reach & ~freeR) & ~visited;
          visited |= nxt;
          level++;
          if (level < 8) LAY |= (uint64_t)nxt << (8 * level);
          frontier = nxt;
        }
        if (!found) break;
        alive = all;
        for (uint32_t fl = freeL; fl; fl &= fl - 1) hk_dfs(idx(fl & (0u - fl)));
      }
    }
    for (uint32_t fl = freeL; fl; fl &= fl - 1)
      if (!kuhn(idx(fl & (0u - fl)))) return false;
    return true;
  }
};
