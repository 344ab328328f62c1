// n <= 8 perfect_matching (matching.py:75-112) for one GPU thread, the K2 fast
// path. Same visiting order as FastMatch8 (fastmatch.cuh, the readable form);
// this one is arranged for the shortest dependent chains:
//  * DFS stacks are shift registers (push = shift left + or, pop = shift
//    right), so no stack access needs a variable shift;
//  * matches live as nibbles of 32-bit words (ML: left -> right, MR: right ->
//    left) plus, per right vertex v, the adjacency byte of its partner
//    (PMR / SMR: pref / sup row of mr[v]) and its one-hot partner (MRB), so a
//    DFS descent reads the next candidate row with a single byte permute;
//  * candidates are one-hot bits; an index is formed only for lookups.
#pragma once
#include <stdint.h>

#if !defined(AUR_HD)
#if defined(__CUDACC__)
#define AUR_HD __host__ __device__ __forceinline__
#else
#define AUR_HD inline
#endif
#endif

struct FastMatch8c {
  uint32_t P0, P1, S0, S1;        // pref / sup rows: byte u = right-vertex mask of left u
  uint32_t ML, MR;                // nibbles: ML[u] = right of u, MR[v] = left of v
  uint32_t MRB0, MRB1;            // bytes: one-hot left matched to v (0: free)
  uint32_t PMR0, PMR1, SMR0, SMR1;  // bytes: pref / sup row of mr[v]
  uint32_t LAY0, LAY1;            // bytes: BFS layer d
  uint32_t freeL, freeR, alive;

  AUR_HD static uint32_t byte_of(uint32_t lo, uint32_t hi, uint32_t i) {
#if defined(__CUDA_ARCH__)
    return __byte_perm(lo, hi, i) & 0xFFu;
#else
    return ((i < 4 ? lo : hi) >> (8 * (i & 3))) & 0xFFu;
#endif
  }
  AUR_HD static void set_byte(uint32_t& lo, uint32_t& hi, uint32_t i, uint32_t v) {
    const uint32_t sh = 8 * (i & 3), m = ~(0xFFu << sh), nv = v << sh;
    if (i < 4) lo = (lo & m) | nv;
    else hi = (hi & m) | nv;
  }
  AUR_HD static uint32_t nib(uint32_t w, uint32_t i) { return (w >> (4 * i)) & 15u; }
  AUR_HD static uint32_t set_nib(uint32_t w, uint32_t i, uint32_t v) {
    return (w & ~(15u << (4 * i))) | (v << (4 * i));
  }
  AUR_HD static uint32_t idx(uint32_t onehot) {
#if defined(__CUDA_ARCH__)
    return (uint32_t)(__ffs((int)onehot) - 1);
#else
    return (uint32_t)__builtin_ctz(onehot);
#endif
  }
  AUR_HD static uint32_t gather_or(uint32_t lo, uint32_t hi, uint32_t mask) {
    const uint32_t ml = ((mask & 15u) * 0x00204081u & 0x01010101u) * 0xFFu;
    const uint32_t mh = (((mask >> 4) & 15u) * 0x00204081u & 0x01010101u) * 0xFFu;
    uint32_t r = (lo & ml) | (hi & mh);
    r |= r >> 16;
    r |= r >> 8;
    return r & 0xFFu;
  }
  AUR_HD void match(uint32_t u, uint32_t v) {
    ML = set_nib(ML, u, v);
    MR = set_nib(MR, v, u);
    set_byte(MRB0, MRB1, v, 1u << u);
    set_byte(PMR0, PMR1, v, byte_of(P0, P1, u));
    set_byte(SMR0, SMR1, v, byte_of(S0, S1, u));
  }
  // path: U nibbles = us[top..0] (low = top), V nibbles = vs[top-1..0], final right vertex v
  AUR_HD void augment(uint32_t U, uint32_t V, uint32_t v, int top) {
    for (int l = top; l >= 0; l--) {
      match(U & 15u, v);
      U >>= 4;
      v = V & 15u;
      V >>= 4;
    }
  }

  AUR_HD void hk_dfs(uint32_t root) {  // matching.py:57-65
    uint64_t L = byte_of(P0, P1, root);  // candidate stack, top at the low byte
    uint32_t U = root, V = 0;
    int top = 0;
    for (;;) {
      const uint32_t m = (uint32_t)L & 0xFFu;
      if (!m) {
        alive &= ~(1u << (U & 15u));  // dist[u] = _INF
        if (top == 0) return;
        L >>= 8;
        U >>= 4;
        V >>= 4;
        top--;
        continue;
      }
      const uint32_t b = m & (0u - m);
      L ^= b;
      const uint32_t v = idx(b);
      if (freeR & b) {
        augment(U, V, v, top);
        freeL &= ~(1u << root);
        freeR &= ~b;
        return;
      }
      const uint32_t w = nib(MR, v);
      if (top + 1 < 8 && ((byte_of(LAY0, LAY1, top + 1) & alive) >> w) & 1u) {
        L = (L << 8) | byte_of(PMR0, PMR1, v);
        U = (U << 4) | w;
        V = (V << 4) | v;
        top++;
      }
    }
  }

  AUR_HD bool kuhn(uint32_t root) {  // matching.py:96-106
    uint32_t seen = 0;
    uint64_t L = byte_of(S0, S1, root);
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
      L = (L << 8) | byte_of(SMR0, SMR1, v);
      U = (U << 4) | nib(MR, v);
      V = (V << 4) | v;
      top++;
    }
  }

  // rows beyond n must be zero; result: ML nibbles
  AUR_HD bool run(int n) {
    const uint32_t all = (1u << n) - 1;
    freeL = freeR = all;
    ML = MR = 0;
    MRB0 = MRB1 = PMR0 = PMR1 = SMR0 = SMR1 = 0;
    if (P0 | P1) {
      // first Hopcroft-Karp phase: all left free -> greedy lowest free preferred vertex
#pragma unroll
      for (int u = 0; u < 8; u++) {
        const uint32_t m = byte_of(P0, P1, u) & freeR;
        if (m) {
          const uint32_t b = m & (0u - m);
          freeR &= ~b;
          freeL &= ~(1u << u);
          match(u, idx(b));
        }
      }
      for (;;) {
        uint32_t frontier = freeL, visited = freeL;
        LAY0 = frontier;
        LAY1 = 0;
        bool found = false;
        int level = 0;
        while (frontier) {  // bfs(), matching.py:37-55, one SWAR step per level
          const uint32_t reach = gather_or(P0, P1, frontier);
          found |= (reach & freeR) != 0;
          const uint32_t nxt = gather_or(MRB0, MRB1, reach & ~freeR) & ~visited;
          visited |= nxt;
          level++;
          if (level < 8) set_byte(LAY0, LAY1, level, nxt);
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
