// Experiment: FastMatch8d with lane-parallel BFS levels (warp OR-reduction + ballot).
// n <= 8 perfect_matching (matching.py:75-112) for one GPU thread, built for
// short dependent chains and few instructions. Same result as FastMatch8b
// (fastmatch8b.cuh) and the reference -- same visiting orders -- with lighter
// bookkeeping:
//
// * Greedy first Hopcroft-Karp phase: each row costs three dependent ALU ops
//   (t = P[u] & free; x = t - 1; free &= ~t | x); the match tables are built
//   from the per-row results without branches: the left->right one-hot table
//   by byte permutes, the right->left index table from three bit slices.
// * bfs(): the partners of a set R of right vertices are the rows of the
//   left->right one-hot table that meet R (a SWAR nonzero-byte test).
// * HK dfs (matching.py:57-65): no candidate stack. At depth d the viable right
//   vertices are "free, or matched to an alive vertex of BFS layer d + 1"
//   (byte d of VB); the reference loop only ever skips a candidate because its
//   partner's dfs failed, and exactly then the partner dies and the candidate
//   leaves VB, so a node's remaining candidates are always P[u] & VB[d] --
//   recomputed from the row when the search returns to it. VB is rebuilt after
//   each augmentation (partners change).
// * Kuhn extension (matching.py:96-106): no candidate stack either. `seen` is
//   shared by the whole search from one root and every candidate tried at a
//   node is marked seen, so the node's remaining candidates are S[u] & ~seen.
// Byte reads are byte permutes (prmt) of the 64-bit tables. Only nibble 0 of
// a selector has to be clean: a read whose index is itself a permute result
// needs no masking (table entries are < 8, so its nibble 1 is 0 too).
//
// Result: MR (byte v = the left vertex matched to v); left_of() / ml_of()
// read it per left vertex.
#pragma once
#include <stdint.h>

#if !defined(AUR_HD)
#if defined(__CUDACC__)
#define AUR_HD __host__ __device__ __forceinline__
#else
#define AUR_HD inline
#endif
#endif

struct FastMatch8f {
  uint64_t P, S;   // pref / sup rows: byte u = right-vertex mask of left u
  uint64_t MR;     // byte v = left vertex matched to right v (index; garbage when v is free)
  uint64_t MLB;    // byte u = one-hot right vertex matched to u (0: free)
  uint32_t freeL, freeR;

  // PTX prmt.b32, default mode (selector nibble bit 3 replicates the sign of the byte)
  AUR_HD static uint32_t prmt(uint32_t a, uint32_t b, uint32_t s) {
#if defined(__CUDA_ARCH__)
    uint32_t r;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(s));
    return r;
#else
    const uint64_t ab = ((uint64_t)b << 32) | a;
    uint32_t r = 0;
    for (int k = 0; k < 4; k++) {
      const uint32_t nib = (s >> (4 * k)) & 15u;
      uint32_t byte = (uint32_t)(ab >> (8 * (nib & 7u))) & 0xFFu;
      if (nib & 8u) byte = (byte & 0x80u) ? 0xFFu : 0u;
      r |= byte << (8 * k);
    }
    return r;
#endif
  }
  AUR_HD static uint32_t perm(uint64_t x, uint32_t i) {  // byte i in the low byte (upper bytes: garbage)
    return prmt((uint32_t)x, (uint32_t)(x >> 32), i);
  }
  AUR_HD static uint32_t idx(uint32_t m) {  // lowest set bit, m != 0
#if defined(__CUDA_ARCH__)
    return (uint32_t)(__ffs((int)m) - 1);
#else
    return (uint32_t)__builtin_ctz(m);
#endif
  }
  // 0xFF in byte k iff bit k of m (m < 16)
  AUR_HD static uint32_t bytes_of(uint32_t m) { return prmt(m * 0x10204080u, 0u, 0xBA98u); }
  // OR of the bytes of a whose index is set in mask (mask < 256)
  AUR_HD static uint32_t gather_or(uint64_t a, uint32_t mask) {
    uint32_t r = ((uint32_t)a & bytes_of(mask & 15u)) | ((uint32_t)(a >> 32) & bytes_of(mask >> 4));
    r |= r >> 16;
    r |= r >> 8;
    return r & 0xFFu;
  }
  // bit k set iff byte k of (hi:lo) is nonzero
  AUR_HD static uint32_t nz_bytes(uint32_t lo, uint32_t hi) {
    const uint32_t l = (((lo & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | lo) & 0x80808080u;
    const uint32_t h = (((hi & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | hi) & 0x80808080u;
    // bits 7, 15, 23, 31 -> 21..24 (no carries: the other product terms land elsewhere)
    return (((l >> 7) * 0x00204081u >> 21) & 15u) | (((h >> 7) * 0x00204081u >> 17) & 0xF0u);
  }
  // bit v of m in bit 0 of byte v
  AUR_HD static uint64_t spread_lsb(uint32_t m) {
    const uint32_t lo = (m & 15u) * 0x00204081u & 0x01010101u;
    const uint32_t hi = ((m >> 4) & 15u) * 0x00204081u & 0x01010101u;
    return ((uint64_t)hi << 32) | lo;
  }
  AUR_HD static uint64_t put(uint64_t x, uint32_t i, uint32_t v) {  // byte i := v
    const uint32_t sh = 8 * i;
    return (x & ~(0xFFull << sh)) | ((uint64_t)v << sh);
  }
  // right vertex matched to left u (n <= 8, perfect matching in MR): the byte of MR equal to u
  AUR_HD static uint32_t ml_of(uint64_t mr, uint32_t u, int n) {
    const uint32_t bc = u * 0x01010101u;
    const uint32_t lo = (uint32_t)mr ^ bc, hi = (uint32_t)(mr >> 32) ^ bc;
    const uint32_t valid = n >= 8 ? 0xFFu : (1u << n) - 1;
    return idx(~nz_bytes(lo, hi) & valid);
  }
  AUR_HD uint32_t ml(uint32_t u, int n) const { return ml_of(MR, u, n); }
  AUR_HD void match(uint32_t u, uint32_t v) {
    MR = put(MR, v, u);
    MLB = put(MLB, u, 1u << v);
  }

  // ---------------------------------------------------------------- HK --
  uint64_t LAY;   // byte d = BFS layer d (left vertices)
  uint64_t VB;    // byte d = right vertices viable at depth d
  uint32_t alive;
  int levels;     // number of BFS layers

  AUR_HD void build_vb() {
    uint64_t vb = (uint64_t)freeR << (8 * (levels - 1));  // deepest layer: free vertices only
    for (int d = 0; d + 1 < levels; d++)
      vb |= (uint64_t)(freeR | gather_or(MLB, perm(LAY, (uint32_t)d + 1) & alive)) << (8 * d);
    VB = vb;
  }

  // path: U nibbles = left vertices (top at the low nibble), V nibbles = the
  // right vertices chosen below each of them but the last, v = the free end
  AUR_HD void augment(uint32_t U, uint32_t V, uint32_t v, int top) {
#pragma unroll 1
    for (int l = top; l >= 0; l--) {
      match(U & 15u, v);
      U >>= 4;
      v = V & 15u;
      V >>= 4;
    }
  }

  AUR_HD bool hk_dfs(uint32_t root) {
    uint32_t U = root, V = 0, u = root;
    int top = 0;
    for (;;) {
      const uint32_t m = perm(P, u) & perm(VB, (uint32_t)top) & 0xFFu;
      if (!m) {  // dfs(u) fails: dist[u] = _INF; its partner stops being viable one level up
        const uint32_t uc = U & 15u;  // u itself may carry garbage above nibble 0
        alive &= ~(1u << uc);
        if (top == 0) return false;
        VB &= ~((uint64_t)(perm(MLB, uc) & 0xFFu) << (8 * (top - 1)));
        U >>= 4;
        V >>= 4;
        top--;
        u = U & 15u;
        continue;
      }
      const uint32_t v = idx(m);
      if ((freeR >> v) & 1u) {
        augment(U, V, v, top);
        freeL &= ~(1u << root);
        freeR &= ~(1u << v);
        build_vb();
        return true;
      }
      const uint32_t w = perm(MR, v);  // alive, on layer top + 1 (viability); clean nibble 0
      U = (U << 4) | (w & 15u);
      V = (V << 4) | v;
      top++;
      u = w;
    }
  }

  // -------------------------------------------------------------- Kuhn --
  AUR_HD bool kuhn(uint32_t root) {
    uint32_t seen = 0, U = root, V = 0, u = root;
    int top = 0;
    for (;;) {
      const uint32_t m = perm(S, u) & ~seen & 0xFFu;
      if (!m) {
        if (top == 0) return false;
        U >>= 4;
        V >>= 4;
        top--;
        u = U & 15u;
        continue;
      }
      const uint32_t v = idx(m);
      seen |= 1u << v;
      if ((freeR >> v) & 1u) {
        uint32_t vv = v;
#pragma unroll 1
        for (int l = top; l >= 0; l--) {  // the left->right table is not kept past HK
          MR = put(MR, vv, U & 15u);
          U >>= 4;
          vv = V & 15u;
          V >>= 4;
        }
        freeR &= ~(1u << v);
        kuhned = true;
        return true;
      }
      const uint32_t w = perm(MR, v);
      U = (U << 4) | (w & 15u);
      V = (V << 4) | v;
      top++;
      u = w;
    }
  }

  bool kuhned;  // the Kuhn extension augmented: MLB is stale, MR is the result

  // rows beyond n must be zero. Result: MR (every right vertex < n matched);
  // MLB too unless `kuhned`.
  AUR_HD bool run(int n) {
    const uint32_t all = (1u << n) - 1;
    freeL = freeR = all;
    MR = MLB = 0;
    kuhned = false;
    if (P) {
      // first HK phase, all left vertices free: greedy lowest free preferred vertex
      uint32_t fr = all, fl = 0;
      uint32_t b[8];
#pragma unroll
      for (int u = 0; u < 8; u++) {
        const uint32_t t = perm(P, (uint32_t)u) & fr & 0xFFu;
        const uint32_t x = t - 1u;
        b[u] = t & ~x;
        fr &= ~t | x;
        fl |= t ? 0u : (1u << u);
      }
      // left->right one-hot bytes; right->left indices from bit slices of u
      MLB = ((uint64_t)prmt(prmt(b[4], b[5], 0x3340u), prmt(b[6], b[7], 0x3340u), 0x5410u) << 32) |
            prmt(prmt(b[0], b[1], 0x3340u), prmt(b[2], b[3], 0x3340u), 0x5410u);
      const uint32_t m0 = b[1] | b[3] | b[5] | b[7], m1 = b[2] | b[3] | b[6] | b[7], m2 = b[4] | b[5] | b[6] | b[7];
      MR = spread_lsb(m0) + 2 * spread_lsb(m1) + 4 * spread_lsb(m2);
      freeR = fr;
      freeL = fl & all;
      while (freeL) {
        // bfs(), matching.py:37-55: level-synchronous, one SWAR step per level
        uint32_t frontier = freeL, visited = freeL;
        uint64_t lay = frontier;
        bool found = false;
        int level = 0;
#if defined(__CUDA_ARCH__)
        // lane u (< 8) holds row u of P and of the left->right one-hot table: a level is one
        // OR-reduction (the right vertices the frontier reaches) and one ballot (their partners)
        const uint32_t ln = threadIdx.x & 31u;
        const uint32_t pu = ln < 8 ? perm(P, ln) & 0xFFu : 0u, mu = ln < 8 ? perm(MLB, ln) & 0xFFu : 0u;
        while (frontier) {
          const uint32_t reach = __reduce_or_sync(0xffffffffu, ((frontier >> ln) & 1u) ? pu : 0u);
          found |= (reach & freeR) != 0;
          const uint32_t nxt = __ballot_sync(0xffffffffu, (mu & reach & ~freeR) != 0u) & ~visited;
          visited |= nxt;
          level++;
          if (level < 8) lay |= (uint64_t)nxt << (8 * level);
          frontier = nxt;
        }
#else
        while (frontier) {
          const uint32_t reach = gather_or(P, frontier);
          found |= (reach & freeR) != 0;
          const uint32_t bc = (reach & ~freeR) * 0x01010101u;  // partners of the matched reached vertices
          const uint32_t nxt = nz_bytes((uint32_t)MLB & bc, (uint32_t)(MLB >> 32) & bc) & ~visited;
          visited |= nxt;
          level++;
          if (level < 8) lay |= (uint64_t)nxt << (8 * level);
          frontier = nxt;
        }
#endif
        if (!found) break;
        LAY = lay;
        levels = level < 8 ? level : 8;
        alive = all;
        build_vb();
        for (uint32_t f = freeL; f; f &= f - 1) hk_dfs(idx(f));
      }
    }
    for (uint32_t f = freeL; f; f &= f - 1)
      if (!kuhn(idx(f))) return false;
    return true;
  }
};
