// k-clique counting on the rank-relabelled DAG (K6-K11).
//
// Replaces count_impl (proj/src/counting.cpp:85-200) and its recursion
// clique_rec (proj/src/clique_rec.hpp:24-62).  The reference marks
// candidates with a per-thread stamp array and filters adjacency lists;
// here every source vertex u stages the induced subgraph on N+(u) ONCE as
// a symmetric bitmap (the paper's per-source staging, counting.cpp:21-48,
// read cost sum_w indeg(w)*outdeg(w)), and then every oriented edge
// (u, w_i) is an independent task whose candidate set I = N+(u) ∩ N+(w_i)
// is row i of that bitmap restricted to higher local ids.  Because the
// DAG is relabelled by rank, local id order is a topological order, so
// "bits above x" == "out-neighbours of x" and the recursion
//     count(I, r) = sum_{x in I} count(I ∩ N+(x), r-1)
// is a sequence of AND / POPC over bitmap rows.
//
// Tiers, by d = outdeg(u):
//   warp tier   d <= 32      one warp per source; rows are single words;
//                            lane i owns edge (u, w_i) and runs the
//                            remaining k-2 levels in registers
//   CTA tier    32 < d <= D  one CTA per source; rows of ceil(d/32) words
//                            in shared memory; one warp per edge; sets
//                            larger than 32 are processed warp-
//                            cooperatively, sets of <= 32 vertices are
//                            compacted (ballot transpose) to one word per
//                            vertex and finished per lane
//   heavy tier  d > D        the same code with the bitmap, hash and warp
//                            scratch in a per-CTA slice of global memory
//                            (L2-resident)
// Per-vertex counts: each task accumulates into per-source local counters
// (u64) and flushes one global atomic per touched vertex per source.
// Totals: warp reductions, one u64 atomic per warp.
#include <cub/cub.cuh>

#include <algorithm>
#include <vector>

#include "kcg_internal.cuh"

namespace kcg {
namespace {

typedef unsigned long long ull;
constexpr uint32_t FULL = 0xffffffffu;
constexpr uint32_t EMPTY = 0xffffffffu;
constexpr uint32_t NOTFOUND = 0xffffffffu;
constexpr int CTA_THREADS = 256;
constexpr int CTA_WARPS = CTA_THREADS / 32;
constexpr int WARP_THREADS_BLOCK = 256;
constexpr int WARP_TIER_WARPS = WARP_THREADS_BLOCK / 32;
constexpr uint32_t SMEM_TIER_MAX = 1024;  // largest d staged in shared memory

__device__ __forceinline__ uint32_t above_mask(uint32_t b) {  // bits > b, b in [0,31]
  return b >= 31 ? 0u : (FULL << (b + 1));
}
__device__ __forceinline__ uint32_t hash_slot(uint32_t key, int bits) {
  return (key * 0x9E3779B1u) >> (32 - bits);
}
__device__ __forceinline__ ull warp_sum(ull v) {
  for (int s = 16; s; s >>= 1) v += __shfl_xor_sync(FULL, v, s);
  return v;
}

// ---------------------------------------------------------------------------
// Per-lane recursion over <= 32-vertex compact subproblems.
// sym[x] = neighbours of x inside the subproblem (both directions); since
// b only holds bits above the chosen x, b & sym[x] = (remaining) ∩ N+(x).
// With PV, cpv[x] accumulates the number of counted cliques containing x
// (excluding the caller's chain).
// ---------------------------------------------------------------------------
template <int R, bool PV>
__device__ __forceinline__ ull lane_cnt(uint32_t J, const uint32_t* sym, ull* cpv) {
  if constexpr (R == 1) {
    if constexpr (PV) {
      for (uint32_t b = J; b; b &= b - 1) atomicAdd(&cpv[__ffs(b) - 1], 1ull);
    }
    return __popc(J);
  } else if constexpr (R == 2) {
    ull t = 0;
    for (uint32_t b = J; b;) {
      int x = __ffs(b) - 1;
      b &= b - 1;
      uint32_t sx = sym[x];
      t += __popc(b & sx);
      if constexpr (PV) {
        uint32_t c = __popc(J & sx);
        if (c) atomicAdd(&cpv[x], ull(c));
      }
    }
    return t;
  } else {
    ull t = 0;
    for (uint32_t b = J; b;) {
      int x = __ffs(b) - 1;
      b &= b - 1;
      if (__popc(b) < R - 1) break;
      uint32_t J2 = b & sym[x];
      if (__popc(J2) >= R - 1) {
        ull c = lane_cnt<R - 1, PV>(J2, sym, cpv);
        t += c;
        if constexpr (PV) {
          if (c) atomicAdd(&cpv[x], c);
        }
      }
    }
    return t;
  }
}

// Explicit-stack variant for R beyond the templated depths.
template <bool PV>
__device__ __noinline__ ull lane_cnt_generic(uint32_t J, int R, const uint32_t* sym, ull* cpv) {
  uint32_t S[33];
  int X[33];
  ull C[33];
  int lvl = 0;
  S[0] = J;
  C[0] = 0;
  for (;;) {
    uint32_t b = S[lvl];
    const int rr = R - lvl;
    if (__popc(b) < rr) {
      if (lvl == 0) break;
      ull c = C[lvl];
      lvl--;
      C[lvl] += c;
      if (PV && c) atomicAdd(&cpv[X[lvl]], c);
      continue;
    }
    int x = __ffs(b) - 1;
    b &= b - 1;
    S[lvl] = b;
    uint32_t J2 = b & sym[x];
    const int r2 = rr - 1;
    if (__popc(J2) < r2) continue;
    if (r2 == 2) {
      ull c = lane_cnt<2, PV>(J2, sym, cpv);
      C[lvl] += c;
      if (PV && c) atomicAdd(&cpv[x], c);
    } else {
      X[lvl] = x;
      lvl++;
      S[lvl] = J2;
      C[lvl] = 0;
    }
  }
  return C[0];
}

template <bool PV>
__device__ ull lane_count(uint32_t J, int R, const uint32_t* sym, ull* cpv) {
  if (__popc(J) < R) return 0;
  switch (R) {
    case 1: return lane_cnt<1, PV>(J, sym, cpv);
    case 2: return lane_cnt<2, PV>(J, sym, cpv);
    case 3: return lane_cnt<3, PV>(J, sym, cpv);
    case 4: return lane_cnt<4, PV>(J, sym, cpv);
    case 5: return lane_cnt<5, PV>(J, sym, cpv);
    case 6: return lane_cnt<6, PV>(J, sym, cpv);
    case 7: return lane_cnt<7, PV>(J, sym, cpv);
    case 8: return lane_cnt<8, PV>(J, sym, cpv);
    default: return lane_cnt_generic<PV>(J, R, sym, cpv);
  }
}

// ---------------------------------------------------------------------------
// Warp tier: one warp per source u with 2 <= d <= 32.
// ---------------------------------------------------------------------------
template <bool PV>
__global__ void __launch_bounds__(WARP_THREADS_BLOCK)
    count_warp_kernel(const uint64_t* __restrict__ off, const uint32_t* __restrict__ adj,
                      const uint32_t* __restrict__ srcs, uint32_t nsrc, int k,
                      ull* __restrict__ total_out, ull* __restrict__ pv_rank,
                      ull* __restrict__ staged_out) {
  __shared__ uint32_t s_sym[WARP_TIER_WARPS][32];
  __shared__ uint32_t s_key[WARP_TIER_WARPS][64];
  __shared__ uint8_t s_idx[WARP_TIER_WARPS][64];
  __shared__ ull s_pv[PV ? WARP_TIER_WARPS : 1][32];
  const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  uint32_t* sym = s_sym[wib];
  uint32_t* hkey = s_key[wib];
  uint8_t* hidx = s_idx[wib];
  ull* cpv = s_pv[PV ? wib : 0];
  const int R = k - 2;
  ull my_total = 0, my_staged = 0;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t si = gw; si < nsrc; si += nw) {
    const uint32_t u = srcs[si];
    const uint64_t b = off[u];
    const uint32_t d = uint32_t(off[u + 1] - b);
    const uint32_t w = lane < d ? adj[b + lane] : 0u;
    hkey[lane] = EMPTY;
    hkey[lane + 32] = EMPTY;
    sym[lane] = 0;
    if constexpr (PV) cpv[lane] = 0;
    __syncwarp();
    if (lane < d) {
      uint32_t slot = hash_slot(w, 6);
      while (atomicCAS(&hkey[slot], EMPTY, w) != EMPTY) slot = (slot + 1) & 63;
      hidx[slot] = uint8_t(lane);
    }
    uint64_t sb = 0;
    uint32_t len = 0;
    if (lane < d) {
      sb = off[w];
      len = uint32_t(off[w + 1] - sb);
    }
    // inclusive scan of segment lengths
    uint32_t incl = len;
    for (int s = 1; s < 32; s <<= 1) {
      uint32_t t = __shfl_up_sync(FULL, incl, s);
      if (lane >= uint32_t(s)) incl += t;
    }
    const uint32_t excl = incl - len;
    const uint32_t L = __shfl_sync(FULL, incl, 31);
    my_staged += len;
    __syncwarp();
    // flattened scan of all out-lists N+(w_i): 32 consecutive entries per
    // step, each lane finds its segment by a 5-step shuffle search
    for (uint32_t c0 = 0; c0 < L; c0 += 32) {
      const uint32_t p = c0 + lane;
      uint32_t seg = 0;
#pragma unroll
      for (int step = 16; step; step >>= 1) {
        uint32_t cand = seg + step;
        uint32_t pe = __shfl_sync(FULL, excl, cand);
        if (pe <= p && cand < d) seg = cand;
      }
      const uint64_t sbase = __shfl_sync(FULL, sb, seg);
      const uint32_t sex = __shfl_sync(FULL, excl, seg);
      if (p < L) {
        const uint32_t y = adj[sbase + (p - sex)];
        uint32_t slot = hash_slot(y, 6);
        uint32_t j = NOTFOUND;
        for (;;) {
          uint32_t kk = hkey[slot];
          if (kk == y) {
            j = hidx[slot];
            break;
          }
          if (kk == EMPTY) break;
          slot = (slot + 1) & 63;
        }
        if (j != NOTFOUND) {
          atomicOr(&sym[seg], 1u << j);
          atomicOr(&sym[j], 1u << seg);
        }
      }
    }
    __syncwarp();
    ull c = 0;
    if (lane < d) {
      uint32_t row = sym[lane] & above_mask(lane);
      c = lane_count<PV>(row, R, sym, cpv);
      my_total += c;
      if constexpr (PV) {
        if (c) atomicAdd(&cpv[lane], c);
      }
    }
    if constexpr (PV) {
      __syncwarp();
      ull src_total = warp_sum(c);
      if (lane < d && cpv[lane]) atomicAdd(&pv_rank[w], cpv[lane]);
      if (lane == 0 && src_total) atomicAdd(&pv_rank[u], src_total);
    }
    __syncwarp();
  }
  my_total = warp_sum(my_total);
  if (lane == 0) {
    if (my_total) atomicAdd(total_out, my_total);
    if (my_staged) atomicAdd(staged_out, my_staged);
  }
}

// ---------------------------------------------------------------------------
// CTA / heavy tier.
// ---------------------------------------------------------------------------
struct Lvl {
  uint32_t wcur, bits, left, R, x, pad;
  ull tot;
};

// Byte layout of one CTA's working set (shared memory or a global slice).
struct Layout {
  uint32_t dmax, wpmax, tbits, levels;
  size_t sym, hkey, hidx, pvl, warp0, warp_stride;
  // per-warp offsets
  size_t w_cand, w_stack, w_csym, w_cpv, w_lvl;
  size_t total;
};

__host__ __device__ inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

__host__ __device__ inline Layout make_layout(uint32_t dmax, uint32_t levels, bool pv) {
  Layout L;
  L.dmax = dmax;
  L.wpmax = ((dmax + 31) / 32) | 1u;
  int tb = 6;
  while ((1u << tb) < 2 * dmax) tb++;
  L.tbits = tb;
  L.levels = levels;
  size_t at = 0;
  L.sym = at;
  at = align_up(at + size_t(dmax) * L.wpmax * 4, 16);
  L.hkey = at;
  at = align_up(at + (size_t(1) << tb) * 4, 16);
  L.hidx = at;
  at = align_up(at + (size_t(1) << tb) * 2, 16);
  L.pvl = at;
  at = align_up(at + (pv ? size_t(dmax) * 8 : 0), 16);
  L.warp0 = at;
  size_t w = 0;
  L.w_cand = w;
  w = align_up(w + size_t(dmax) * 2 + 64, 16);
  L.w_stack = w;
  w = align_up(w + size_t(levels) * L.wpmax * 4, 16);
  L.w_csym = w;
  w = align_up(w + 32 * 4, 16);
  L.w_cpv = w;
  w = align_up(w + (pv ? 32 * 8 : 0), 16);
  L.w_lvl = w;
  w = align_up(w + size_t(levels) * sizeof(Lvl), 16);
  L.warp_stride = w;
  L.total = align_up(at + w * CTA_WARPS, 128);
  return L;
}

struct WarpCtx {
  const uint32_t* sym;  // CTA bitmap, row stride wp
  uint32_t wp, W;
  uint16_t* cand;
  uint32_t* stack;      // levels x wp words
  uint32_t* csym;       // 32 words
  ull* cpv;             // 32 (PV)
  ull* pvl;             // d (PV)
  Lvl* lvl;
  uint32_t lane;
};

// R == 1: every member is a clique completion
template <bool PV>
__device__ ull set_members_pv(const WarpCtx& c, const uint32_t* S) {
  ull cnt = 0;
  for (uint32_t w = c.lane; w < c.W; w += 32) {
    uint32_t v = S[w];
    cnt += __popc(v);
    if constexpr (PV) {
      for (; v; v &= v - 1) atomicAdd(&c.pvl[32 * w + __ffs(v) - 1], 1ull);
    }
  }
  return warp_sum(cnt);
}

// Writes the members of S (ascending) into c.cand; returns their number.
__device__ uint32_t enumerate_members(const WarpCtx& c, const uint32_t* S, uint32_t limit) {
  uint32_t base = 0;
  for (uint32_t w0 = 0; w0 < c.W && base < limit; w0 += 32) {
    uint32_t w = w0 + c.lane;
    uint32_t v = w < c.W ? S[w] : 0u;
    uint32_t n = __popc(v);
    uint32_t incl = n;
    for (int s = 1; s < 32; s <<= 1) {
      uint32_t t = __shfl_up_sync(FULL, incl, s);
      if (c.lane >= uint32_t(s)) incl += t;
    }
    uint32_t pos = base + incl - n;
    for (; v && pos < limit; v &= v - 1) c.cand[pos++] = uint16_t(32 * w + __ffs(v) - 1);
    base += __shfl_sync(FULL, incl, 31);
  }
  __syncwarp();
  return base < limit ? base : limit;
}

// |S| <= 32: transpose S's induced rows into one word per member (ballot),
// then finish the remaining R-1 levels per lane.
template <bool PV>
__device__ ull compact_count(const WarpCtx& c, const uint32_t* S, uint32_t s, int R) {
  enumerate_members(c, S, 32);
  const uint32_t lane = c.lane;
  const uint32_t xt = lane < s ? c.cand[lane] : 0u;
  const uint32_t wofs = xt >> 5, bofs = xt & 31;
  uint32_t mine = 0;
  for (uint32_t r = 0; r < s; r++) {
    uint32_t xr = __shfl_sync(FULL, xt, r);
    uint32_t word = lane < s ? c.sym[size_t(xr) * c.wp + wofs] : 0u;
    uint32_t bal = __ballot_sync(FULL, (word >> bofs) & 1u);
    if (lane == r) mine = bal;
  }
  c.csym[lane] = mine;
  if constexpr (PV) c.cpv[lane] = 0;
  __syncwarp();
  ull ct = 0;
  if (lane < s) {
    ct = lane_count<PV>(mine & above_mask(lane), R - 1, c.csym, c.cpv);
    if constexpr (PV) {
      if (ct) atomicAdd(&c.cpv[lane], ct);
    }
  }
  __syncwarp();
  if constexpr (PV) {
    if (lane < s && c.cpv[lane]) atomicAdd(&c.pvl[xt], c.cpv[lane]);
  }
  ull tot = warp_sum(ct);
  __syncwarp();
  return tot;
}

// R == 2 with |S| > 32: sum over members x of |S ∩ N+(x)|, one member per
// lane, multi-word dot products.
template <bool PV>
__device__ ull dot_count(const WarpCtx& c, const uint32_t* S, uint32_t s) {
  uint32_t ns = enumerate_members(c, S, 0xffffffffu);
  (void)s;
  ull cnt = 0;
  for (uint32_t t = c.lane; t < ns; t += 32) {
    const uint32_t x = c.cand[t];
    const uint32_t* row = c.sym + size_t(x) * c.wp;
    const uint32_t w0 = x >> 5;
    uint32_t acc = __popc(S[w0] & row[w0] & above_mask(x & 31));
    for (uint32_t w = w0 + 1; w < c.W; w++) acc += __popc(S[w] & row[w]);
    cnt += acc;
    if constexpr (PV) {
      uint32_t all = __popc(S[w0] & row[w0] & ~above_mask(x & 31));
      for (uint32_t w = 0; w < w0; w++) all += __popc(S[w] & row[w]);
      all += acc;
      if (all) atomicAdd(&c.pvl[x], ull(all));
    }
  }
  __syncwarp();
  return warp_sum(cnt);
}

// child = S ∩ N+(x) into dst; returns |child| (warp-uniform)
__device__ uint32_t child_set(const WarpCtx& c, const uint32_t* S, uint32_t x, uint32_t* dst) {
  const uint32_t* row = c.sym + size_t(x) * c.wp;
  const uint32_t wx = x >> 5;
  uint32_t n = 0;
  for (uint32_t w = c.lane; w < c.W; w += 32) {
    uint32_t v = 0;
    if (w > wx)
      v = S[w] & row[w];
    else if (w == wx)
      v = S[w] & row[w] & above_mask(x & 31);
    dst[w] = v;
    n += __popc(v);
  }
  __syncwarp();
  return __reduce_add_sync(FULL, n);
}

// count(S, R) for a set held in stack level 0 with |S| = s.
template <bool PV>
__device__ ull warp_count(const WarpCtx& c, uint32_t s, int R) {
  const uint32_t* S0 = c.stack;
  if (uint32_t(R) > s) return 0;
  if (R == 1) return set_members_pv<PV>(c, S0);
  if (s <= 32) return compact_count<PV>(c, S0, s, R);
  if (R == 2) return dot_count<PV>(c, S0, s);
  // warp-cooperative DFS over sets larger than 32
  Lvl* st = c.lvl;
  int L = 0;
  if (c.lane == 0) st[0] = Lvl{0, S0[0], s, uint32_t(R), 0, 0, 0ull};
  __syncwarp();
  for (;;) {
    Lvl cur = st[L];
    const uint32_t* SL = c.stack + size_t(L) * c.wp;
    while (cur.bits == 0 && cur.wcur + 1 < c.W) {
      cur.wcur++;
      cur.bits = SL[cur.wcur];
    }
    if (cur.bits == 0 || cur.left < cur.R) {
      if (L == 0) {
        __syncwarp();
        return cur.tot;
      }
      ull sub = cur.tot;
      L--;
      __syncwarp();
      if (c.lane == 0) {
        st[L].tot += sub;
        if (PV && sub) atomicAdd(&c.pvl[st[L].x], sub);
      }
      __syncwarp();
      continue;
    }
    const uint32_t x = 32 * cur.wcur + __ffs(cur.bits) - 1;
    cur.bits &= cur.bits - 1;
    cur.left--;
    uint32_t* child = c.stack + size_t(L + 1) * c.wp;
    const uint32_t sc = child_set(c, SL, x, child);
    const uint32_t rc = cur.R - 1;
    ull add = 0;
    bool descend = false;
    if (sc >= rc) {
      if (rc == 1) {
        add = set_members_pv<PV>(c, child);
      } else if (sc <= 32) {
        add = compact_count<PV>(c, child, sc, int(rc));
      } else if (rc == 2) {
        add = dot_count<PV>(c, child, sc);
      } else {
        descend = true;
      }
    }
    __syncwarp();
    if (c.lane == 0) {
      cur.tot += add;
      if (PV && add) atomicAdd(&c.pvl[x], add);
      cur.x = x;
      st[L] = cur;
      if (descend) st[L + 1] = Lvl{0, child[0], sc, rc, 0, 0, 0ull};
    }
    __syncwarp();
    if (descend) L++;
  }
}

struct CtaArgs {
  const uint64_t* off;
  const uint32_t* adj;
  const uint32_t* srcs;
  uint32_t nsrc;
  int k;
  ull* total;
  ull* pv_rank;
  ull* staged;
  unsigned* work;        // source counter
  unsigned* ework;       // per-CTA edge counters (global tier)
  unsigned char* gbase;  // global working sets (heavy tier)
  Layout L;
  int global_ws;
};

template <bool PV>
__global__ void __launch_bounds__(CTA_THREADS) count_cta_kernel(CtaArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ unsigned s_src, s_edge;
  __shared__ ull s_src_total;
  const Layout& L = a.L;
  unsigned char* base = a.global_ws ? a.gbase + size_t(blockIdx.x) * L.total : smem;
  uint32_t* sym = reinterpret_cast<uint32_t*>(base + L.sym);
  uint32_t* hkey = reinterpret_cast<uint32_t*>(base + L.hkey);
  uint16_t* hidx = reinterpret_cast<uint16_t*>(base + L.hidx);
  ull* pvl = reinterpret_cast<ull*>(base + L.pvl);
  const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  unsigned char* wbase = base + L.warp0 + size_t(wib) * L.warp_stride;
  WarpCtx c;
  c.sym = sym;
  c.cand = reinterpret_cast<uint16_t*>(wbase + L.w_cand);
  c.stack = reinterpret_cast<uint32_t*>(wbase + L.w_stack);
  c.csym = reinterpret_cast<uint32_t*>(wbase + L.w_csym);
  c.cpv = reinterpret_cast<ull*>(wbase + L.w_cpv);
  c.lvl = reinterpret_cast<Lvl*>(wbase + L.w_lvl);
  c.pvl = pvl;
  c.lane = lane;
  const int R = a.k - 2;
  ull my_total = 0, my_staged = 0;
  for (;;) {
    if (threadIdx.x == 0) {
      s_src = atomicAdd(a.work, 1u);
      s_edge = 0;
      s_src_total = 0;
    }
    __syncthreads();
    const uint32_t si = s_src;
    if (si >= a.nsrc) break;
    const uint32_t u = a.srcs[si];
    const uint64_t b = a.off[u];
    const uint32_t d = uint32_t(a.off[u + 1] - b);
    const uint32_t W = (d + 31) / 32, wp = W | 1u;
    int tb = 6;
    while ((1u << tb) < 2 * d) tb++;
    const uint32_t T = 1u << tb, tmask = T - 1;
    c.wp = wp;
    c.W = W;
    for (uint32_t i = threadIdx.x; i < d * wp; i += CTA_THREADS) sym[i] = 0;
    for (uint32_t i = threadIdx.x; i < T; i += CTA_THREADS) hkey[i] = EMPTY;
    if constexpr (PV) {
      for (uint32_t i = threadIdx.x; i < d; i += CTA_THREADS) pvl[i] = 0;
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < d; i += CTA_THREADS) {
      uint32_t w = a.adj[b + i];
      uint32_t slot = hash_slot(w, tb);
      while (atomicCAS(&hkey[slot], EMPTY, w) != EMPTY) slot = (slot + 1) & tmask;
      hidx[slot] = uint16_t(i);
    }
    __syncthreads();
    // stage the induced subgraph: warp per row, lanes over N+(w_i)
    for (uint32_t i = wib; i < d; i += CTA_WARPS) {
      const uint32_t wi = a.adj[b + i];
      const uint64_t rb = a.off[wi], re = a.off[wi + 1];
      if (lane == 0) my_staged += re - rb;
      for (uint64_t p = rb + lane; p < re; p += 32) {
        const uint32_t y = a.adj[p];
        uint32_t slot = hash_slot(y, tb);
        for (;;) {
          uint32_t kk = hkey[slot];
          if (kk == y) {
            uint32_t j = hidx[slot];
            atomicOr(&sym[size_t(i) * wp + (j >> 5)], 1u << (j & 31));
            atomicOr(&sym[size_t(j) * wp + (i >> 5)], 1u << (i & 31));
            break;
          }
          if (kk == EMPTY) break;
          slot = (slot + 1) & tmask;
        }
      }
    }
    __syncthreads();
    // one warp per oriented edge (u, w_i), dynamically scheduled
    ull warp_src = 0;
    for (;;) {
      uint32_t i = 0;
      if (lane == 0) i = atomicAdd(&s_edge, 1u);
      i = __shfl_sync(FULL, i, 0);
      if (i >= d) break;
      // S0 = row i above i
      uint32_t n = 0;
      const uint32_t wi = i >> 5;
      for (uint32_t w = lane; w < W; w += 32) {
        uint32_t v = 0;
        if (w > wi)
          v = sym[size_t(i) * wp + w];
        else if (w == wi)
          v = sym[size_t(i) * wp + w] & above_mask(i & 31);
        c.stack[w] = v;
        n += __popc(v);
      }
      __syncwarp();
      const uint32_t s0 = __reduce_add_sync(FULL, n);
      ull ce = (s0 >= uint32_t(R)) ? warp_count<PV>(c, s0, R) : 0ull;
      warp_src += ce;
      if constexpr (PV) {
        if (lane == 0 && ce) atomicAdd(&pvl[i], ce);
      }
    }
    if (lane == 0) {
      my_total += warp_src;
      if (PV && warp_src) atomicAdd(&s_src_total, warp_src);
    }
    __syncthreads();
    if constexpr (PV) {
      for (uint32_t i = threadIdx.x; i < d; i += CTA_THREADS)
        if (pvl[i]) atomicAdd(&a.pv_rank[a.adj[b + i]], pvl[i]);
      if (threadIdx.x == 0 && s_src_total) atomicAdd(&a.pv_rank[u], s_src_total);
    }
    __syncthreads();
  }
  if (lane == 0) {
    if (my_total) atomicAdd(a.total, my_total);
    if (my_staged) atomicAdd(a.staged, my_staged);
  }
}

// ---------------------------------------------------------------------------
// Setup kernels
// ---------------------------------------------------------------------------
// Splits sources with d >= dmin into the warp tier list and the CTA/heavy
// candidate list (key = d for sorting).
__global__ void classify_kernel(const uint64_t* __restrict__ off, uint32_t n, uint32_t dmin,
                                uint32_t part, uint32_t nparts,
                                uint32_t* __restrict__ wlist, uint32_t* __restrict__ clist,
                                uint32_t* __restrict__ ckey, unsigned* __restrict__ cnt) {
  const uint32_t lane = threadIdx.x & 31;
  for (uint32_t base = blockIdx.x * blockDim.x; base < n; base += gridDim.x * blockDim.x) {
    const uint32_t r = base + threadIdx.x;
    uint32_t d = 0;
    if (r < n && r % nparts == part) d = uint32_t(off[r + 1] - off[r]);
    const bool inw = r < n && d >= dmin && d <= 32;
    const bool inc = r < n && d >= dmin && d > 32;
    unsigned bw = __ballot_sync(FULL, inw), bc = __ballot_sync(FULL, inc);
    unsigned ow = 0, oc = 0;
    if (lane == 0) {
      if (bw) ow = atomicAdd(&cnt[0], __popc(bw));
      if (bc) oc = atomicAdd(&cnt[1], __popc(bc));
    }
    ow = __shfl_sync(FULL, ow, 0);
    oc = __shfl_sync(FULL, oc, 0);
    const unsigned below = (1u << lane) - 1;
    if (inw) wlist[ow + __popc(bw & below)] = r;
    if (inc) {
      clist[oc + __popc(bc & below)] = r;
      ckey[oc + __popc(bc & below)] = 0xffffffffu - d;  // descending d
    }
  }
}

__global__ void k2_pv_kernel(const uint64_t* __restrict__ rdag_off,
                             const uint32_t* __restrict__ rdag_adj, uint32_t n, uint32_t part,
                             uint32_t nparts, ull* __restrict__ pv_rank) {
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    if (r % nparts != part) continue;
    const uint64_t b = rdag_off[r], e = rdag_off[r + 1];
    if (e > b) atomicAdd(&pv_rank[r], ull(e - b));
    for (uint64_t p = b; p < e; p++) atomicAdd(&pv_rank[rdag_adj[p]], 1ull);
  }
}

__global__ void gather_pv_kernel(const ull* __restrict__ pv_rank, const uint32_t* __restrict__ rank,
                                 uint32_t n, ull* __restrict__ pv) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    pv[v] = pv_rank[rank[v]];
}

template <bool PV>
void launch_cta(Graph& g, CtaArgs a, uint32_t nsrc, bool global_ws, size_t heavy_budget,
                unsigned* work_ctr) {
  a.nsrc = nsrc;
  a.work = work_ctr;
  KCG_CUDA(cudaMemsetAsync(work_ctr, 0, 4, g.stream));
  const Device& dev = device();
  unsigned grid;
  size_t smem = 0;
  if (!global_ws) {
    smem = a.L.total;
    KCG_CUDA(cudaFuncSetAttribute(count_cta_kernel<PV>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(smem)));
    int occ = 0;
    KCG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, count_cta_kernel<PV>,
                                                           CTA_THREADS, smem));
    occ = std::max(occ, 1);
    grid = std::min<uint64_t>(nsrc, uint64_t(dev.sms) * occ);
    a.global_ws = 0;
    a.gbase = nullptr;
  } else {
    size_t per = a.L.total;
    uint64_t fit = std::max<uint64_t>(1, heavy_budget / per);
    grid = unsigned(std::min<uint64_t>({nsrc, uint64_t(dev.sms) * 2, fit}));
    a.gbase = g.heavy.ensure(size_t(grid) * per, &g.bytes);
    a.global_ws = 1;
  }
  count_cta_kernel<PV><<<grid, CTA_THREADS, smem, g.stream>>>(a);
  KCG_LAUNCHED(g);
  g.stats.launches++;
}

inline ull* PVR(Graph& g) { return reinterpret_cast<ull*>(g.pv_rank.p); }

}  // namespace

uint64_t count_cliques(Graph& g, int k, bool want_pv, uint32_t part, uint32_t nparts) {
  if (nparts == 0 || part >= nparts) fail(KCG_EINVAL, "part must be < nparts");
  if (k < 2) fail(KCG_EINVAL, "k must be at least 2");
  if (!g.has_rdag) fail(KCG_EINVAL, "no DAG on the handle");
  const uint32_t n = g.n;
  g.stats = kcg_count_stats{};
  g.stats.max_out_degree = g.max_out;
  g.mark(2);
  ull* ctr = g.counters.ensure(16, &g.bytes);  // [0]=total [1]=staged [2..] work counters
  KCG_CUDA(cudaMemsetAsync(ctr, 0, 16 * 8, g.stream));
  if (want_pv) {
    g.pv_rank.ensure(size_t(n) + 1, &g.bytes);
    g.pv.ensure(size_t(n) + 1, &g.bytes);
    KCG_CUDA(cudaMemsetAsync(g.pv_rank.p, 0, size_t(n) * 8, g.stream));
  }
  uint64_t total = 0;
  if (k == 2) {
    // counting.cpp:165-173: every directed edge is a 2-clique
    total = nparts == 1 ? g.m : 0;
    if (nparts > 1) {
      std::vector<uint64_t> ro(size_t(n) + 1);
      KCG_CUDA(cudaMemcpyAsync(ro.data(), g.rdag_off.p, ro.size() * 8, cudaMemcpyDeviceToHost,
                               g.stream));
      g.sync();
      for (uint32_t r = part; r < n; r += nparts) total += ro[r + 1] - ro[r];
    }
    if (want_pv && n) {
      k2_pv_kernel<<<blocks_for(n, 256), 256, 0, g.stream>>>(g.rdag_off.p, g.rdag_adj.p, n,
                                                            part, nparts, PVR(g));
      KCG_LAUNCHED(g);
    }
    g.mark(6);
    g.mark(7);
  } else if (uint64_t(k - 1) <= g.max_out) {
    // tier lists
    const uint32_t dmin = uint32_t(k - 1);
    size_t nb = (size_t(n) * 4 + 255) & ~size_t(255);
    unsigned char* sb = g.scratch2.ensure(nb * 5 + 1024, &g.bytes);
    uint32_t* wlist = reinterpret_cast<uint32_t*>(sb);
    uint32_t* clist = reinterpret_cast<uint32_t*>(sb + nb);
    uint32_t* ckey = reinterpret_cast<uint32_t*>(sb + 2 * nb);
    uint32_t* clist2 = reinterpret_cast<uint32_t*>(sb + 3 * nb);
    uint32_t* ckey2 = reinterpret_cast<uint32_t*>(sb + 4 * nb);
    unsigned* cnt = reinterpret_cast<unsigned*>(ctr + 2);
    classify_kernel<<<blocks_for(n, 256, 148u * 16u), 256, 0, g.stream>>>(
        g.rdag_off.p, n, dmin, part, nparts, wlist, clist, ckey, cnt);
    KCG_LAUNCHED(g);
    unsigned hc[2] = {0, 0};
    KCG_CUDA(cudaMemcpyAsync(hc, cnt, 8, cudaMemcpyDeviceToHost, g.stream));
    g.sync();
    const uint32_t nw = hc[0], nc = hc[1];
    if (nc > 1) {
      size_t tb = 0;
      KCG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, ckey, ckey2, clist, clist2, nc, 0, 32,
                                               g.stream));
      KCG_CUDA(cub::DeviceRadixSort::SortPairs(cub_temp(g, tb), tb, ckey, ckey2, clist, clist2,
                                               nc, 0, 32, g.stream));
      std::swap(clist, clist2);
      std::swap(ckey, ckey2);
    }
    // host copy of the sorted degrees to cut bins
    std::vector<uint32_t> keys(nc);
    if (nc) {
      KCG_CUDA(cudaMemcpyAsync(keys.data(), ckey, size_t(nc) * 4, cudaMemcpyDeviceToHost,
                               g.stream));
    }
    g.sync();
    g.mark(6);
    const Device& dev = device();
    if (nw) {
      unsigned grid = blocks_for(uint64_t(nw) * 32, WARP_THREADS_BLOCK, dev.sms * 8u);
      if (want_pv)
        count_warp_kernel<true><<<grid, WARP_THREADS_BLOCK, 0, g.stream>>>(
            g.rdag_off.p, g.rdag_adj.p, wlist, nw, k, ctr, PVR(g), ctr + 1);
      else
        count_warp_kernel<false><<<grid, WARP_THREADS_BLOCK, 0, g.stream>>>(
            g.rdag_off.p, g.rdag_adj.p, wlist, nw, k, ctr, PVR(g), ctr + 1);
      KCG_LAUNCHED(g);
      g.stats.launches++;
    }
    g.stats.sources_warp = nw;
    if (nc) {
      // bins in descending d: [heavy] (512,1024] (256,512] (128,256] (64,128] (32,64]
      const uint32_t R = uint32_t(k - 2);
      const uint32_t bounds[] = {SMEM_TIER_MAX, 512, 256, 128, 64, 32};
      auto deg_at = [&](uint32_t i) { return 0xffffffffu - keys[i]; };
      uint32_t pos = 0;
      unsigned* work = cnt + 2;
      int wslot = 0;
      CtaArgs a{};
      a.off = g.rdag_off.p;
      a.adj = g.rdag_adj.p;
      a.k = k;
      a.total = ctr;
      a.pv_rank = PVR(g);
      a.staged = ctr + 1;
      // heavy: d > SMEM_TIER_MAX (or anything whose layout does not fit)
      uint32_t hend = 0;
      while (hend < nc && deg_at(hend) > SMEM_TIER_MAX) hend++;
      if (hend) {
        uint32_t dmax = deg_at(0);
        a.srcs = clist;
        a.L = make_layout(dmax, std::max<uint32_t>(R, 1), want_pv);
        const size_t budget = size_t(8) << 30;
        if (want_pv)
          launch_cta<true>(g, a, hend, true, budget, work + wslot++);
        else
          launch_cta<false>(g, a, hend, true, budget, work + wslot++);
        g.stats.sources_heavy = hend;
      }
      pos = hend;
      for (int bi = 0; bi < 5 && pos < nc; bi++) {
        const uint32_t hi = bounds[bi], lo = bounds[bi + 1];
        uint32_t end = pos;
        while (end < nc && deg_at(end) > lo) end++;
        if (end == pos) continue;
        Layout Lb = make_layout(hi, std::max<uint32_t>(R, 1), want_pv);
        bool global_ws = Lb.total > size_t(dev.smem_optin) - 1024;
        a.srcs = clist + pos;
        a.L = global_ws ? make_layout(deg_at(pos), std::max<uint32_t>(R, 1), want_pv) : Lb;
        const size_t budget = size_t(8) << 30;
        if (want_pv)
          launch_cta<true>(g, a, end - pos, global_ws, budget, work + wslot++);
        else
          launch_cta<false>(g, a, end - pos, global_ws, budget, work + wslot++);
        g.stats.sources_cta += end - pos;
        pos = end;
      }
    }
    g.mark(7);
  } else {
    g.mark(6);
    g.mark(7);
  }
  if (want_pv && n) {
    gather_pv_kernel<<<blocks_for(n, 256), 256, 0, g.stream>>>(PVR(g), g.rank.p, n,
                                                              reinterpret_cast<ull*>(g.pv.p));
    KCG_LAUNCHED(g);
  }
  ull hv[2] = {0, 0};
  KCG_CUDA(cudaMemcpyAsync(hv, ctr, 16, cudaMemcpyDeviceToHost, g.stream));
  g.mark(3);
  g.sync();
  if (k != 2) total = hv[0];
  g.stats.staged_elems = hv[1];
  g.times.count_ms = g.elapsed(2, 3);
  g.times.count_kernel_ms = g.elapsed(6, 7);
  return total;
}

}  // namespace kcg
