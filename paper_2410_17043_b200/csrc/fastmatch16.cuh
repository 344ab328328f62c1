// n <= 16 perfect_matching (matching.py:75-112) for one GPU thread: FastMatch8b's
// visiting order and tricks (fastmatch8b.cuh) widened to 16-bit rows -- adjacency
// rows, one-hot match tables and BFS layers as 16-bit lanes of four 64-bit words,
// the DFS candidate stack a 256-bit shift register, vertex stacks nibbles of one
// 64-bit word, and OR-gathers over row sets done with a multiply-spread mask.
#pragma once
#include <stdint.h>

#if !defined(AUR_HD)
#if defined(__CUDACC__)
#define AUR_HD __host__ __device__ __forceinline__
#else
#define AUR_HD inline
#endif
#endif

// sixteen 16-bit lanes in four named 64-bit words: no array, so a dynamic lane
// index never sends the table to local memory (selects instead)
struct Q4 {
  uint64_t w0, w1, w2, w3;
  AUR_HD void clear() { w0 = w1 = w2 = w3 = 0; }
  AUR_HD uint64_t word(uint32_t i) const {
    const uint64_t lo = (i & 4) ? w1 : w0;
    const uint64_t hi = (i & 4) ? w3 : w2;
    return (i & 8) ? hi : lo;
  }
  AUR_HD bool any() const { return (w0 | w1 | w2 | w3) != 0; }
};

struct FastMatch16 {
  Q4 P, S;          // pref / sup rows: lane u = right-vertex mask of left u
  Q4 MRB;           // lane v = one-hot left vertex matched to right v (0: free)
  Q4 MLB;           // lane u = one-hot right vertex matched to left u (0: free)
  Q4 LAY;           // lane d = BFS layer d (left vertices)
  Q4 RLA;           // lane d = right vertices matched to alive layer-d vertices
  uint64_t ML, MR;  // nibble u = right vertex of left u / nibble v = left vertex of right v
  uint32_t freeL, freeR, alive;

  AUR_HD static uint32_t lane(const Q4& a, uint32_t i) {
    return (uint32_t)(a.word(i) >> (16 * (i & 3))) & 0xFFFFu;
  }
  AUR_HD static void set_lane(Q4& a, uint32_t i, uint32_t v) {
    const uint32_t sh = 16 * (i & 3), q = i >> 2;
    const uint64_t m = ~(0xFFFFull << sh), nv = (uint64_t)v << sh;
    a.w0 = q == 0 ? (a.w0 & m) | nv : a.w0;
    a.w1 = q == 1 ? (a.w1 & m) | nv : a.w1;
    a.w2 = q == 2 ? (a.w2 & m) | nv : a.w2;
    a.w3 = q == 3 ? (a.w3 & m) | nv : a.w3;
  }
  AUR_HD static uint32_t nib(uint64_t x, uint32_t i) { return (uint32_t)(x >> (4 * i)) & 15u; }
  AUR_HD static uint64_t set_nib(uint64_t x, uint32_t i, uint32_t v) {
    const uint32_t sh = 4 * i;
    return (x & ~(15ull << sh)) | ((uint64_t)v << sh);
  }
  AUR_HD static uint32_t idx(uint32_t onehot) {
#if defined(__CUDA_ARCH__)
    return (uint32_t)(__ffs((int)onehot) - 1);
#else
    return (uint32_t)__builtin_ctz(onehot);
#endif
  }
  // OR of the lanes of a whose index is set in mask: 4 mask bits -> 4 lane masks
  // per word (bit j times 2^(15 j) lands on bit 16 j; no carries between terms)
  AUR_HD static uint64_t spread4(uint32_t m4) {
    return (((uint64_t)m4 * 0x0000200040008001ull) & 0x0001000100010001ull) * 0xFFFFull;
  }
  AUR_HD static uint32_t gather_or(const Q4& a, uint32_t mask) {
    uint64_t r = (a.w0 & spread4(mask & 15u)) | (a.w1 & spread4((mask >> 4) & 15u)) |
                 (a.w2 & spread4((mask >> 8) & 15u)) | (a.w3 & spread4((mask >> 12) & 15u));
    r |= r >> 32;
    r |= r >> 16;
    return (uint32_t)r & 0xFFFFu;
  }
  AUR_HD void match(uint32_t u, uint32_t v) {
    ML = set_nib(ML, u, v);
    MR = set_nib(MR, v, u);
    set_lane(MRB, v, 1u << u);
    set_lane(MLB, u, 1u << v);
  }
  // path: U nibbles = us[top..0] (low = top), V nibbles = vs[top-1..0], final right vertex v
  AUR_HD void augment(uint64_t U, uint64_t V, uint32_t v, int top) {
    for (int l = top; l >= 0; l--) {
      match((uint32_t)U & 15u, v);
      U >>= 4;
      v = (uint32_t)V & 15u;
      V >>= 4;
    }
  }
  // the same, keeping RLA: the stack vertex at depth l sits on BFS layer l, so v_l
  // moves from layer l+1's set (matched to us[l+1] before) to layer l's
  AUR_HD void augment_hk(uint64_t U, uint64_t V, uint32_t v, int top) {
    for (int l = top; l >= 0; l--) {
      match((uint32_t)U & 15u, v);
      if (l < top) set_lane(RLA, (uint32_t)l + 1, lane(RLA, (uint32_t)l + 1) & ~(1u << v));
      if (l > 0) set_lane(RLA, (uint32_t)l, lane(RLA, (uint32_t)l) | (1u << v));
      U >>= 4;
      v = (uint32_t)V & 15u;
      V >>= 4;
    }
  }
  // 256-bit stack of 16-bit entries, top in the low lane of L[0]
  AUR_HD static void push(uint64_t (&L)[4], uint32_t x) {
    L[3] = (L[3] << 16) | (L[2] >> 48);
    L[2] = (L[2] << 16) | (L[1] >> 48);
    L[1] = (L[1] << 16) | (L[0] >> 48);
    L[0] = (L[0] << 16) | x;
  }
  AUR_HD static void pop(uint64_t (&L)[4]) {
    L[0] = (L[0] >> 16) | (L[1] << 48);
    L[1] = (L[1] >> 16) | (L[2] << 48);
    L[2] = (L[2] >> 16) | (L[3] << 48);
    L[3] >>= 16;
  }

  // hopcroft_karp dfs(root), matching.py:57-65, candidates masked as in FastMatch8b:
  // at depth d only v free or matched to an alive vertex of layer d+1 can be taken
  AUR_HD bool hk_dfs(uint32_t root) {
    uint64_t L[4] = {lane(P, root), 0, 0, 0};
    uint64_t U = root, V = 0;
    int top = 0;
    for (;;) {
      const uint32_t nr = top + 1 < 16 ? lane(RLA, (uint32_t)top + 1) : 0u;
      const uint32_t m = (uint32_t)L[0] & 0xFFFFu & (freeR | nr);
      if (!m) {
        const uint32_t u = (uint32_t)U & 15u;
        alive &= ~(1u << u);  // dist[u] = _INF: its partner leaves layer top's set
        set_lane(RLA, (uint32_t)top, lane(RLA, (uint32_t)top) & ~lane(MLB, u));
        if (top == 0) return false;
        pop(L);
        U >>= 4;
        V >>= 4;
        top--;
        continue;
      }
      const uint32_t b = m & (0u - m);
      L[0] = (L[0] & ~0xFFFFull) | (m ^ b);
      const uint32_t v = idx(b);
      if (freeR & b) {
        augment_hk(U, V, v, top);
        freeL &= ~(1u << root);
        freeR &= ~b;
        return true;
      }
      const uint32_t w = nib(MR, v);
      push(L, lane(P, w));
      U = (U << 4) | w;
      V = (V << 4) | v;
      top++;
    }
  }

  // perfect_matching's augment(u, seen), matching.py:96-106
  AUR_HD bool kuhn(uint32_t root) {
    uint32_t seen = 0;
    uint64_t L[4] = {lane(S, root), 0, 0, 0};
    uint64_t U = root, V = 0;
    int top = 0;
    for (;;) {
      const uint32_t m = (uint32_t)L[0] & ~seen & 0xFFFFu;
      if (!m) {
        if (top == 0) return false;
        pop(L);
        U >>= 4;
        V >>= 4;
        top--;
        continue;
      }
      const uint32_t b = m & (0u - m);
      L[0] ^= b;
      seen |= b;
      const uint32_t v = idx(b);
      if (freeR & b) {
        augment(U, V, v, top);
        freeL &= ~(1u << root);
        freeR &= ~b;
        return true;
      }
      const uint32_t w = nib(MR, v);
      push(L, lane(S, w));
      U = (U << 4) | w;
      V = (V << 4) | v;
      top++;
    }
  }

  // rows beyond n must be zero; result: ML nibbles
  AUR_HD bool run(int n) {
    const uint32_t all = n >= 32 ? ~0u : (1u << n) - 1;
    freeL = freeR = all;
    ML = MR = 0;
#pragma unroll
    MRB.clear();
    MLB.clear();
    LAY.clear();
    RLA.clear();
    if (P.any()) {
      // first Hopcroft-Karp phase: all left free -> greedy lowest free preferred vertex
#pragma unroll
      for (int u = 0; u < 16; u++) {
        const uint32_t m = lane(P, (uint32_t)u) & freeR;
        const uint32_t b = m & (0u - m);
        if (b) {
          freeR &= ~b;
          match((uint32_t)u, idx(b));
          freeL &= ~(1u << u);
        }
      }
      for (;;) {
        uint32_t frontier = freeL, visited = freeL;
        LAY.clear();
        LAY.w0 = frontier;
        bool found = false;
        int level = 0;
        while (frontier) {  // bfs(), matching.py:37-55, one gather per level
          const uint32_t reach = gather_or(P, frontier);
          found |= (reach & freeR) != 0;
          const uint32_t nxt = gather_or(MRB, reach & ~freeR) & ~visited;
          visited |= nxt;
          level++;
          if (level < 16) set_lane(LAY, (uint32_t)level, nxt);
          frontier = nxt;
        }
        if (!found) break;
        alive = all;
        RLA.clear();
        for (int d = 1; d < level && d < 16; d++) set_lane(RLA, (uint32_t)d, gather_or(MLB, lane(LAY, (uint32_t)d)));
        for (uint32_t fl = freeL; fl; fl &= fl - 1) hk_dfs(idx(fl & (0u - fl)));
      }
    }
    for (uint32_t fl = freeL; fl; fl &= fl - 1)
      if (!kuhn(idx(fl & (0u - fl)))) return false;
    return true;
  }
};
