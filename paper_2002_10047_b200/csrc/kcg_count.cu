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
//   heavy tier  d > D        k = 4 (D = 512): the tiled kernel of
//                            kcg_heavy.cuh -- bitmap in a per-CTA slice of
//                            global memory (L2), counted through 128-row
//                            shared-memory tiles; k >= 5 (D = 1024): the
//                            CTA-tier code with the bitmap (and, if need be,
//                            everything else) in the global slice
// Per-vertex counts: each task accumulates into per-source local counters
// (u64) and flushes one global atomic per touched vertex per source.
// Totals: warp reductions, one u64 atomic per warp.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdlib>
#include <vector>

#include "kcg_internal.cuh"

namespace kcg {
namespace {

typedef unsigned long long ull;
constexpr uint32_t FULL = 0xffffffffu;
constexpr uint32_t EMPTY = 0xffffffffu;
constexpr int WARP_THREADS_BLOCK = 256;
constexpr int WARP_TIER_WARPS = WARP_THREADS_BLOCK / 32;
constexpr uint32_t WARP_TABLE_BITS = 7;  // 128 buckets for <= 32 keys
constexpr size_t WARP_TABLE_BYTES = 128 * 20 + 128 / 8 + 64 * 8 + 16;  // bucket_bytes(32)
constexpr uint32_t SMEM_TIER_MAX = 1024;  // largest d staged in shared memory

__device__ __forceinline__ uint32_t above_mask(uint32_t b) {  // bits > b, b in [0,31]
  return b >= 31 ? 0u : (FULL << (b + 1));
}
__device__ __forceinline__ ull warp_sum(ull v) {
  for (int s = 16; s; s >>= 1) v += __shfl_xor_sync(FULL, v, s);
  return v;
}

}  // namespace
}  // namespace kcg

#include "kcg_stage.cuh"

namespace kcg {
namespace {

}  // namespace
}  // namespace kcg

#include "kcg_dfs.cuh"

namespace kcg {
namespace {

// ---------------------------------------------------------------------------
// Warp tier: one warp per source u with 2 <= d <= 32.
// ---------------------------------------------------------------------------
template <bool PV, int MAXL>
__global__ void __launch_bounds__(WARP_THREADS_BLOCK)
    count_warp_kernel(const uint64_t* __restrict__ off, const uint32_t* __restrict__ adj,
                      const uint32_t* __restrict__ srcs, uint32_t nsrc, int k,
                      ull* __restrict__ total_out, ull* __restrict__ pv_rank,
                      ull* __restrict__ staged_out) {
  struct WarpSmem {
    alignas(16) unsigned char tbl[WARP_TABLE_BYTES];  // Buckets for <= 32 keys (B = 128)
    alignas(16) uint32_t fl[32];                      // staging flag row (one bitmap word)
    uint32_t sym[32];
    uint32_t usym[32];
    uint32_t map[32];
  };
  __shared__ WarpSmem s_w[WARP_TIER_WARPS];
  __shared__ pvc_t s_pv[PV ? WARP_TIER_WARPS : 1][32];
  extern __shared__ __align__(16) unsigned char dyn_smem[];  // per-warp DFS stacks
  const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  WarpSmem& S = s_w[wib];
  constexpr int SL = MAXL > 0 ? MAXL : 1;
  Stacks<PV, SL>* stk = reinterpret_cast<Stacks<PV, SL>*>(dyn_smem) + wib;
  uint32_t* sym = S.sym;
  pvc_t* cpv = s_pv[PV ? wib : 0];
  const int R = k - 2;
  ull my_total = 0, my_staged = 0;
  S.fl[lane] = 0;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t si = gw; si < nsrc; si += nw) {
    const uint32_t u = srcs[si];
    const uint64_t b = off[u];
    const uint32_t d = uint32_t(off[u + 1] - b);
    const uint32_t w = lane < d ? adj[b + lane] : 0u;
    sym[lane] = 0;
    if constexpr (PV) cpv[lane] = 0;
    uint64_t sb = 0;
    uint32_t len = 0;
    if (lane < d) {
      sb = off[w];
      len = uint32_t(off[w + 1] - sb);
    }
    // N+(u) in the warp's bucketed membership table (kcg_stage.cuh), index
    // field = flag position of the local index
    Buckets T = bucket_view(S.tbl, WARP_TABLE_BITS, WARP_TABLE_BITS);
    for (uint32_t attempt = 0;; attempt++) {
      T.mul = BKT_HASH + 2u * 0x632BE5ABu * attempt;
      T.ovf_mode = attempt >= BKT_TRIES;
      __syncwarp();
      bucket_clear(T, lane, 32);
      __syncwarp();
      const bool ok = lane < d ? bucket_insert(T, w, flag_pos(lane)) : true;
      if (__all_sync(FULL, ok)) break;
    }
    __syncwarp();
#if KCG_FILTER
    bucket_filter(T, lane, 32);
    __syncwarp();
#endif
    // Row i either is scanned (len entries) or searched: its d-1-i
    // candidate targets w_j (j > i) are binary-searched in N+(w_i), which
    // costs (d-1-i) * log2(len) probes -- cheaper for the long rows that
    // small sources point into.
    const uint32_t tg = lane < d ? d - 1 - lane : 0u;
    const bool srch = tg > 0 && tg * (32u - __clz(len)) < len;
    my_staged += srch ? 0u : len;
    {
      // searched rows: tasks (i, j) flattened over the lanes
      uint32_t ti = srch ? tg : 0u;
      for (int s = 1; s < 32; s <<= 1) {
        const uint32_t t = __shfl_up_sync(FULL, ti, s);
        if (lane >= uint32_t(s)) ti += t;
      }
      const uint32_t T_ = __shfl_sync(FULL, ti, 31);
      const uint32_t tex = ti - (srch ? tg : 0u);
      for (uint32_t t0 = 0; t0 < T_; t0 += 32) {
        const uint32_t t = t0 + lane;
        uint32_t r = 0;
#pragma unroll
        for (int step = 16; step; step >>= 1) {
          const uint32_t cand = r + step;
          const uint32_t pe = __shfl_sync(FULL, tex, cand);
          if (pe <= t && cand < d) r = cand;
        }
        const uint32_t rt = __shfl_sync(FULL, tex, r);
        const uint64_t rb = __shfl_sync(FULL, sb, r);
        const uint32_t rl = __shfl_sync(FULL, len, r);
        const uint32_t j = r + 1 + (t - rt);
        const uint32_t target = __shfl_sync(FULL, w, j & 31);
        if (t < T_) {
          // lower_bound(target) in the sorted row adj[rb, rb + rl)
          uint32_t lo = 0, n = rl;
          while (n > 1) {
            const uint32_t half = n >> 1;
            if (__ldg(adj + rb + lo + half - 1) < target) lo += half;
            n -= half;
          }
          if (__ldg(adj + rb + lo) == target) {
            atomicOr(&sym[r], 1u << j);
            if constexpr (PV) atomicOr(&sym[j], 1u << r);
          }
        }
      }
      my_staged += T_;
      // scanned rows, one after the other through the row scan of the CTA
      // tiers (kcg_stage.cuh: stage_scan); a row is one bitmap word, which
      // lane i keeps in a register (PV: plus the mirrored bits)
      uint32_t scanm = __ballot_sync(FULL, !srch && len > 0);
      uint32_t symr = 0;
      auto next = [&](StageRow& row) {
        if (scanm == 0) return false;
        const int r = __ffs(scanm) - 1;
        scanm &= scanm - 1;
        row.i = uint32_t(r);
        row.len = __shfl_sync(FULL, len, r);
        row.src = adj + __shfl_sync(FULL, sb, r);
        return true;
      };
      auto emit = [&](const StageRow& row) {
        const uint32_t x = S.fl[lane];
        if (x) S.fl[lane] = 0;
        const uint32_t word = __ballot_sync(FULL, x != 0);
        if (lane == row.i) symr |= word;
        if constexpr (PV) {
          if ((word >> lane) & 1u) symr |= 1u << row.i;
        }
      };
      uint8_t* fl8 = reinterpret_cast<uint8_t*>(S.fl);
      if (T.ovf_mode)
        stage_scan<true>(T, fl8, lane, next, emit);
      else
        stage_scan<false>(T, fl8, lane, next, emit);
      __syncwarp();
      sym[lane] |= symr;
    }
    __syncwarp();
    S.usym[lane] = sym[lane] & above_mask(lane);
    __syncwarp();
    ull c = 0;
    if (R == 1) {
      if (lane < d) {
        c = __popc(S.usym[lane]);
        if constexpr (PV) {
          for (uint32_t bb = S.usym[lane]; bb; bb &= bb - 1) atomicAdd(&cpv[__ffs(bb) - 1], 1u);
          if (c) atomicAdd(&cpv[lane], pvc_t(c));
        }
      }
    } else if (R == 2) {
      c = lane_pairs<PV>(lane < d, S.usym[lane], lane, S.usym, sym, cpv, lane);
    } else if (R <= 32) {
      if constexpr (MAXL > 0)
        c = steal_count<PV, SL>(lane < d, S.usym[lane], R, lane, S.usym, sym, cpv, *stk, S.map,
                                lane);
    }
    my_total += c;
    if constexpr (PV) {
      __syncwarp();
      ull src_total = warp_sum(c);
      if (lane < d && cpv[lane]) atomicAdd(&pv_rank[w], ull(cpv[lane]));
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
  uint32_t dmax, wpmax, tbits, fbits, levels;
  uint32_t lean;  // k = 4 counts: rows padded to 4 words only, warp areas = queues
                  // (tried this round: the bank-spread stride of row_stride, or
                  // power-of-two groups with an XOR swizzle of the groups -- 21%
                  // fewer shared wavefronts in the pair pass, but config 2 k=4
                  // 12.97 -> 13.7 / 15.0 ms from the lost occupancy and the
                  // extra address arithmetic)
  size_t sym, table, filter, rP, rbase, rowid, pvl, warp0, warp_stride;
  size_t sym_bytes;  // the bitmap; inside `total` unless sym_apart
  // per-warp offsets
  size_t w_cand, w_stack, w_csym, w_cusym, w_cpv, w_lvl, w_stk, w_q, w_fl;
  size_t total;
};

__host__ __device__ inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Bitmap row stride in words: a multiple of 4 (rows are read with 128-bit
// shared loads) with an odd number of 16-byte units, so lanes reading
// different rows at the same offset spread over the banks.
__host__ __device__ inline uint32_t row_stride(uint32_t W) { return 4u * (((W + 3u) >> 2) | 1u); }

// sym_apart: the bitmap is laid out separately (a per-CTA slice of global
// memory) and `total` covers the rest, which stays in shared memory.
// Row stride of a lean (k = 4 counts) layout: 16-byte rows, no bank padding
// (the flat pair pass reads unrelated rows per lane).
__host__ __device__ inline uint32_t lean_stride(uint32_t W) { return (W + 3u) & ~3u; }

// lean: k = 4 counts only -- the edge-search areas of the warps are not
// needed and the rows drop their bank padding, which buys the (256, 512]
// and (512, 724] bins one more resident CTA per SM.
__host__ __device__ inline Layout make_layout(uint32_t dmax, uint32_t levels, bool pv, int nw,
                                              size_t stk_bytes, bool sym_apart = false,
                                              bool lean = false) {
  Layout L;
  L.dmax = dmax;
  L.lean = lean;
  L.wpmax = lean ? lean_stride((dmax + 31) / 32) : row_stride((dmax + 31) / 32);
  uint32_t tb = 6;
  while ((1u << tb) < 2 * dmax) tb++;
  L.tbits = tb;
  L.fbits = tb + 4 > 14 ? (tb + 4 > 20 ? 20 : tb + 4) : 14;  // >= 8 filter bits per key
  L.levels = levels;
  size_t at = 0;
  L.sym = at;
  L.sym_bytes = align_up(size_t(dmax) * L.wpmax * 4, 128);
  if (!sym_apart) at = align_up(at + size_t(dmax) * L.wpmax * 4, 16);
  L.table = at;  // bucketed membership table (kcg_stage.cuh: Buckets)
  at = align_up(at + bucket_bytes(dmax), 16);
  L.filter = at;
  L.rP = at;
  at = align_up(at + (size_t(dmax) + 2) * 4, 16);
  L.rbase = at;
  at = align_up(at + size_t(dmax) * 8, 16);
  L.rowid = at;
  at = align_up(at + size_t(dmax) * 4, 16);
  L.pvl = at;
  at = align_up(at + (pv ? size_t(dmax) * 8 : 0), 16);
  L.warp0 = at;
  size_t w = 0;
  const size_t flb = flag_row_bytes((dmax + 31) / 32);  // staging flag row
  if (lean) {
    L.w_cand = L.w_stack = L.w_csym = L.w_cusym = L.w_cpv = L.w_lvl = L.w_stk = L.w_q = 0;
    L.w_fl = 0;
    L.warp_stride = flb;
    L.total = align_up(at + L.warp_stride * nw, 128);
    return L;
  }
  L.w_cand = w;
  w = align_up(w + 32 * 4 + 128, 16);
  L.w_stack = w;
  w = align_up(w + size_t(levels) * L.wpmax * 4, 16);
  L.w_csym = w;
  w = align_up(w + 32 * 4, 16);
  L.w_cusym = w;
  w = align_up(w + 32 * 4, 16);
  L.w_cpv = w;
  w = align_up(w + (pv ? 32 * 8 : 0), 16);
  L.w_lvl = w;
  w = align_up(w + size_t(levels) * sizeof(Lvl), 16);
  L.w_stk = w;
  w = align_up(w + stk_bytes, 16);
  L.w_q = w;
  w = align_up(w + 128 * 4, 16);
  L.w_fl = w;
  w = align_up(w + flb, 16);
  L.warp_stride = w;
  L.total = align_up(at + w * nw, 128);
  return L;
}

struct WarpCtx {
  const uint32_t* sym;  // CTA bitmap, row stride wp
  uint32_t wp, W;
  uint32_t* cand;
  uint32_t* stack;      // levels x wp words
  uint32_t* csym;       // 32 words: compact rows, both directions
  uint32_t* cusym;      // 32 words: compact rows, upper part
  void* stk;            // Stacks<PV, MAXL> of the warp's DFS engine
  uint32_t* qy;         // 128 words: staging queue (keys, rows)
  pvc_t* cpv;           // 32 (PV)
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

// Writes the first `limit` (<= 64) members of S (ascending) into c.cand,
// one word per step with lane j taking bit j; returns their number.
__device__ uint32_t enumerate_members(const WarpCtx& c, const uint32_t* S, uint32_t limit) {
  uint32_t qn = 0;
  const uint32_t lane = c.lane, lt = (1u << lane) - 1u;
  for (uint32_t w0 = 0; w0 < c.W && qn < limit; w0 += 32) {
    const uint32_t wl = w0 + lane;
    const uint32_t mine = wl < c.W ? S[wl] : 0u;
    uint32_t nz = __ballot_sync(FULL, mine != 0);
    while (nz && qn < limit) {
      const uint32_t j = __ffs(nz) - 1;
      nz &= nz - 1;
      const uint32_t v = __shfl_sync(FULL, mine, j);
      const uint32_t pos = qn + __popc(v & lt);
      if (((v >> lane) & 1u) && pos < limit) c.cand[pos] = 32 * (w0 + j) + lane;
      qn += __popc(v);
    }
  }
  __syncwarp();
  return qn < limit ? qn : limit;
}

// |S| <= 32: transpose S's induced rows into one word per member (ballot),
// then finish the remaining R-1 levels per lane.
template <bool PV, int MAXL>
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
  c.cusym[lane] = mine & above_mask(lane);
  if constexpr (PV) c.cpv[lane] = 0;
  __syncwarp();
  // R >= 3 here: every member t roots a (R-1)-clique search in its
  // compact out-neighbourhood, balanced across lanes by the DFS engine
  ull ct = 0;
  if constexpr (MAXL == 0) {
    ct = lane_pairs<PV>(lane < s, c.cusym[lane], lane, c.cusym, c.csym, c.cpv, lane);  // R == 3
  } else {
    ct = R == 3 ? lane_pairs<PV>(lane < s, c.cusym[lane], lane, c.cusym, c.csym, c.cpv, lane)
                : steal_count<PV, MAXL, true>(lane < s, c.cusym[lane], R - 1, lane, c.cusym, c.csym,
                                        c.cpv, *reinterpret_cast<Stacks<PV, MAXL>*>(c.stk),
                                        c.cand, lane);
  }
  __syncwarp();
  if constexpr (PV) {
    if (lane < s && c.cpv[lane]) atomicAdd(&c.pvl[xt], ull(c.cpv[lane]));
  }
  ull tot = warp_sum(ct);
  __syncwarp();
  return tot;
}

// |S ∩ N+(x)| above x for member x of S (128-bit loads; the bitmap's row
// padding is zero, so S's padding words never count).
template <bool PV>
__device__ __forceinline__ void dot_member(const WarpCtx& c, const uint32_t* S, uint32_t x,
                                           ull& cnt) {
  const uint32_t* row = c.sym + size_t(x) * c.wp;
  const uint4* S4 = reinterpret_cast<const uint4*>(S);
  const uint4* r4 = reinterpret_cast<const uint4*>(row);
  const uint32_t xw = x >> 5, g0 = xw >> 2, b0 = g0 * 4, G = (c.W + 3) >> 2;
  const uint32_t ax = above_mask(x & 31);
  uint4 va = S4[g0], vb = r4[g0];
  uint32_t acc = __popc(va.x & vb.x & (b0 < xw ? 0u : (b0 == xw ? ax : FULL))) +
                 __popc(va.y & vb.y & (b0 + 1 < xw ? 0u : (b0 + 1 == xw ? ax : FULL))) +
                 __popc(va.z & vb.z & (b0 + 2 < xw ? 0u : (b0 + 2 == xw ? ax : FULL))) +
                 __popc(va.w & vb.w & (b0 + 3 < xw ? 0u : (b0 + 3 == xw ? ax : FULL)));
  for (uint32_t g = g0 + 1; g < G; g++) {
    va = S4[g];
    vb = r4[g];
    acc += __popc(va.x & vb.x) + __popc(va.y & vb.y) + __popc(va.z & vb.z) + __popc(va.w & vb.w);
  }
  cnt += acc;
  if constexpr (PV) {
    uint32_t all = __popc(S[xw] & row[xw] & ~ax);
    for (uint32_t w = 0; w < xw; w++) all += __popc(S[w] & row[w]);
    all += acc;
    if (all) atomicAdd(&c.pvl[x], ull(all));
  }
}

// R == 2: sum over members x of |S ∩ N+(x)|, one member per lane.  Members
// are scattered word by word (lane j takes bit j of the current non-empty
// word) into the warp's 64-entry candidate queue, and a full batch of 32
// runs its dot products; no lane ever pops bits serially.
template <bool PV>
__device__ ull dot_count(const WarpCtx& c, const uint32_t* S, uint32_t s) {
  (void)s;
  ull cnt = 0;
  uint32_t qn = 0;
  const uint32_t lane = c.lane, lt = (1u << lane) - 1u;
  for (uint32_t w0 = 0; w0 < c.W; w0 += 32) {
    const uint32_t wl = w0 + lane;
    const uint32_t mine = wl < c.W ? S[wl] : 0u;
    uint32_t nz = __ballot_sync(FULL, mine != 0);
    while (nz) {
      const uint32_t j = __ffs(nz) - 1;
      nz &= nz - 1;
      const uint32_t v = __shfl_sync(FULL, mine, j);
      if ((v >> lane) & 1u) c.cand[qn + __popc(v & lt)] = 32 * (w0 + j) + lane;
      qn += __popc(v);
      if (qn >= 32) {
        __syncwarp();
        const uint32_t x = c.cand[lane];
        const bool mv = lane + 32 < qn;
        const uint32_t x1 = mv ? c.cand[lane + 32] : 0u;
        __syncwarp();
        if (mv) c.cand[lane] = x1;
        qn -= 32;
        dot_member<PV>(c, S, x, cnt);
      }
    }
  }
  __syncwarp();
  if (lane < qn) dot_member<PV>(c, S, c.cand[lane], cnt);
  __syncwarp();
  return warp_sum(cnt);
}

// R == 3 (k = 5), totals: for an edge set S (|S| > 32) the number of
// triangles of S's induced DAG, sum over members x and over y in
// T_x = S ∩ N+(x) above x of |S ∩ N+(x) ∩ N+(y)| above y.  The warp walks x
// in order, scatters T_x word by word into a 64-entry (x, y) queue (lane j
// takes bit j) and every full batch runs 32 three-way dot products; T_x is
// never stored and no DFS state is kept.
__device__ ull pair_dots(const WarpCtx& c, const uint32_t* S) {
  ull cnt = 0;
  uint32_t qn = 0;
  const uint32_t lane = c.lane, lt = (1u << lane) - 1u, W = c.W, G = (W + 3) >> 2;
  uint32_t* qy = c.qy;       // 64 entries
  uint32_t* qx = c.qy + 64;  // 64 entries
  const uint4* S4 = reinterpret_cast<const uint4*>(S);
  auto dot3 = [&](uint32_t x, uint32_t y) {
    const uint4* x4 = reinterpret_cast<const uint4*>(c.sym + size_t(x) * c.wp);
    const uint4* y4 = reinterpret_cast<const uint4*>(c.sym + size_t(y) * c.wp);
    const uint32_t yw = y >> 5, g0 = yw >> 2, b0 = g0 * 4, ay = above_mask(y & 31);
    uint4 va = S4[g0], vb = x4[g0], vc = y4[g0];
    uint32_t acc =
        __popc(va.x & vb.x & vc.x & (b0 < yw ? 0u : (b0 == yw ? ay : FULL))) +
        __popc(va.y & vb.y & vc.y & (b0 + 1 < yw ? 0u : (b0 + 1 == yw ? ay : FULL))) +
        __popc(va.z & vb.z & vc.z & (b0 + 2 < yw ? 0u : (b0 + 2 == yw ? ay : FULL))) +
        __popc(va.w & vb.w & vc.w & (b0 + 3 < yw ? 0u : (b0 + 3 == yw ? ay : FULL)));
    for (uint32_t g = g0 + 1; g < G; g++) {
      va = S4[g];
      vb = x4[g];
      vc = y4[g];
      acc += __popc(va.x & vb.x & vc.x) + __popc(va.y & vb.y & vc.y) +
             __popc(va.z & vb.z & vc.z) + __popc(va.w & vb.w & vc.w);
    }
    cnt += acc;
  };
  for (uint32_t s0 = 0; s0 < W; s0 += 32) {
    const uint32_t sw = s0 + lane;
    const uint32_t smine = sw < W ? S[sw] : 0u;
    uint32_t snz = __ballot_sync(FULL, smine != 0);
    while (snz) {
      const uint32_t sj = __ffs(snz) - 1;
      snz &= snz - 1;
      uint32_t xb = __shfl_sync(FULL, smine, sj);
      const uint32_t xw = s0 + sj;
      while (xb) {
        const uint32_t x = 32 * xw + __ffs(xb) - 1;
        xb &= xb - 1;
        const uint32_t* rx = c.sym + size_t(x) * c.wp;
        for (uint32_t t0 = xw & ~31u; t0 < W; t0 += 32) {
          const uint32_t tw = t0 + lane;
          uint32_t t = 0;
          if (tw < W && tw >= xw) t = S[tw] & rx[tw] & (tw == xw ? above_mask(x & 31) : FULL);
          uint32_t tnz = __ballot_sync(FULL, t != 0);
          while (tnz) {
            const uint32_t tj = __ffs(tnz) - 1;
            tnz &= tnz - 1;
            const uint32_t v = __shfl_sync(FULL, t, tj);
            if ((v >> lane) & 1u) {
              const uint32_t pos = qn + __popc(v & lt);
              qy[pos] = 32 * (t0 + tj) + lane;
              qx[pos] = x;
            }
            qn += __popc(v);
            if (qn >= 32) {
              __syncwarp();
              const uint32_t y0 = qy[lane], x0 = qx[lane];
              const bool mv = lane + 32 < qn;
              uint32_t y1 = 0, x1 = 0;
              if (mv) {
                y1 = qy[lane + 32];
                x1 = qx[lane + 32];
              }
              __syncwarp();
              if (mv) {
                qy[lane] = y1;
                qx[lane] = x1;
              }
              qn -= 32;
              dot3(x0, y0);
            }
          }
        }
      }
    }
  }
  __syncwarp();
  if (lane < qn) dot3(qx[lane], qy[lane]);
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
template <bool PV, int MAXL>
__device__ ull warp_count(const WarpCtx& c, uint32_t s, int R) {
  const uint32_t* S0 = c.stack;
  if (uint32_t(R) > s) return 0;
  if (R == 1) return set_members_pv<PV>(c, S0);
  if (R == 2) return dot_count<PV>(c, S0, s);
  if (s <= 32) return compact_count<PV, MAXL>(c, S0, s, R);
  if (!PV && R == 3) return pair_dots(c, S0);
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
      } else if (rc == 2) {
        add = dot_count<PV>(c, child, sc);
      } else if (sc <= 32) {
        add = compact_count<PV, MAXL>(c, child, sc, int(rc));
      } else if (!PV && rc == 3) {
        add = pair_dots(c, child);
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
  const uint32_t* item_src;  // source vertex (rank id) of each work item
  const uint32_t* item_sl;   // (slice << 16) | nslices: the item counts
                             // edges i with i % nslices == slice
  uint32_t nitems;
  int k;
  ull* total;
  ull* pv_rank;
  ull* staged;
  unsigned* work;        // work-item counter
  unsigned char* gbase;  // global working sets (heavy tier)
  Layout L;
};

// GWS = false: the whole working set is dynamic shared memory (the
// compiler sees shared-memory pointers and emits LDS/STS/ATOMS); true:
// per-CTA slices of a global arena (heavy tier).
// MB: minimum resident CTAs per SM the register allocation must allow (4
// caps 256-thread CTAs at 64 registers for the staging-bound k = 4 pass; 3
// gives the k >= 5 edge searches 80 registers without spills).
// GWS (working set): WS_SMEM -- everything in dynamic shared memory;
// WS_SYM_GLOBAL -- the bitmap in a per-CTA slice of global memory (L2),
// hash table, filter, row lists and warp areas in shared memory;
// WS_GLOBAL -- everything in the global slice (sources too large for the
// shared part).
constexpr int WS_SMEM = 0, WS_SYM_GLOBAL = 1, WS_GLOBAL = 2;
// WS_TILED: k = 4 counts of heavy sources (kcg_heavy.cuh) -- the bitmap in a
// global slice, counted through shared-memory tiles
constexpr int WS_TILED = 3;

template <bool PV, int GWS, int NT, int MAXL, int MB>
__global__ void __launch_bounds__(NT, MB) count_cta_kernel(CtaArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ unsigned s_src, s_edge;
  __shared__ ull s_src_total;
  typedef cub::BlockScan<ull, NT> BlockScanU64;
  __shared__ typename BlockScanU64::TempStorage s_scan;
  const Layout& L = a.L;
  unsigned char* base;
  uint32_t* sym;
  if constexpr (GWS == WS_GLOBAL) {
    base = a.gbase + size_t(blockIdx.x) * L.total;
    sym = reinterpret_cast<uint32_t*>(base + L.sym);
  } else if constexpr (GWS == WS_SYM_GLOBAL) {
    base = smem;
    sym = reinterpret_cast<uint32_t*>(a.gbase + size_t(blockIdx.x) * L.sym_bytes);
  } else {
    base = smem;
    sym = reinterpret_cast<uint32_t*>(base + L.sym);
  }
  uint32_t* rP = reinterpret_cast<uint32_t*>(base + L.rP);
  ull* rbase = reinterpret_cast<ull*>(base + L.rbase);
  uint32_t* rowid = reinterpret_cast<uint32_t*>(base + L.rowid);
  ull* pvl = reinterpret_cast<ull*>(base + L.pvl);
  // k = 4 per-vertex credits use the same area as u32 counters when the
  // source allows it (a local vertex's credit is at most C(d-1, 2) < 2^32 for
  // d <= 65536): a 32-bit shared atomic is one ATOMS.ADD where the 64-bit one
  // is a CAS loop
  constexpr uint32_t PV32_MAX_D = 65536;
  uint32_t* pvl32 = reinterpret_cast<uint32_t*>(pvl);
  const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  unsigned char* wbase = base + L.warp0 + size_t(wib) * L.warp_stride;
  WarpCtx c;
  c.sym = sym;
  c.cand = reinterpret_cast<uint32_t*>(wbase + L.w_cand);
  c.stack = reinterpret_cast<uint32_t*>(wbase + L.w_stack);
  c.csym = reinterpret_cast<uint32_t*>(wbase + L.w_csym);
  c.cusym = reinterpret_cast<uint32_t*>(wbase + L.w_cusym);
  c.stk = wbase + L.w_stk;
  c.qy = reinterpret_cast<uint32_t*>(wbase + L.w_q);
  c.cpv = reinterpret_cast<pvc_t*>(wbase + L.w_cpv);
  c.lvl = reinterpret_cast<Lvl*>(wbase + L.w_lvl);
  c.pvl = pvl;
  c.lane = lane;
  const int R = a.k - 2;
  ull my_total = 0, my_staged = 0;
  if constexpr (GWS == WS_SMEM) {  // staging flag row: zero between rows
    uint32_t* fl = reinterpret_cast<uint32_t*>(wbase + L.w_fl);
    for (uint32_t i = lane; i < flag_row_bytes((L.dmax + 31) / 32) / 4; i += 32) fl[i] = 0;
  }
  for (;;) {
    if (threadIdx.x == 0) {
      s_src = atomicAdd(a.work, 1u);
      s_edge = 0;
      s_src_total = 0;
    }
    __syncthreads();
    const uint32_t si = s_src;
    if (si >= a.nitems) break;
    const uint32_t u = a.item_src[si];
    const uint32_t slice = a.item_sl[si] >> 16, nsl = a.item_sl[si] & 0xffffu;
    const uint64_t b = a.off[u];
    const uint32_t d = uint32_t(a.off[u + 1] - b);
    const uint32_t W = (d + 31) / 32, wp = L.lean ? lean_stride(W) : row_stride(W);
    Buckets T = bucket_view(base + L.table, bucket_bits(d), bucket_bits(L.dmax));
    c.wp = wp;
    c.W = W;
    for (uint32_t i = threadIdx.x; i < d * wp; i += NT) sym[i] = 0;
    bucket_clear(T, threadIdx.x, NT);
    if constexpr (PV) {
      for (uint32_t i = threadIdx.x; i < d; i += NT) pvl[i] = 0;
    }
    __syncthreads();
    // membership table + the list of rows to scan: rows with out-neighbours
    // (row d-1 holds no bits above its index: only the symmetric per-vertex
    // bitmaps scan it); one packed (rows << 40 | elements) block scan per NT
    // rows
    uint32_t nr = 0, Lsum = 0;
    const uint32_t last = d - 1;  // row d-1 has no bits above its index
    for (uint32_t t0 = 0; t0 < d; t0 += NT) {
      const uint32_t i = t0 + threadIdx.x;
      uint32_t len = 0;
      uint64_t rb = 0;
      if (i < d) {
        const uint32_t w = a.adj[b + i];
        rb = a.off[w];
        len = uint32_t(a.off[w + 1] - rb);
        if (i >= last) len = 0;
      }
      const ull v = (len ? (1ull << 40) : 0ull) | len;
      ull excl, agg;
      BlockScanU64(s_scan).ExclusiveSum(v, excl, agg);
      if (len) {
        const uint32_t ci = nr + uint32_t(excl >> 40);
        rP[ci] = len;
        rbase[ci] = rb;
        rowid[ci] = i;
      }
      nr += uint32_t(agg >> 40);
      Lsum += uint32_t(agg & ((1ull << 40) - 1));
      __syncthreads();
    }
    bucket_build<GWS == WS_SMEM>(T, a.adj + b, d, threadIdx.x, NT);
    if (threadIdx.x == 0) my_staged += Lsum;
    // stage the induced subgraph: warps take whole rows
    if constexpr (GWS == WS_SMEM) {
      stage_rows(T, sym, wp, W, a.adj, rbase, rP, rowid, nr, &s_edge,
                 reinterpret_cast<uint8_t*>(wbase + L.w_fl), lane);
      if constexpr (PV) {
        __syncthreads();
        mirror_lower(sym, wp, d, W, wib, NT / 32, lane);
      }
    } else {
      stage_rows_atomic<PV>(T, sym, wp, a.adj, rbase, rP, rowid, nr, &s_edge, lane);
    }
    __syncthreads();
    if (threadIdx.x == 0) s_edge = 0;
    __syncthreads();
    ull warp_src = 0;
    if (R == 2) {
      // k = 4: the source's count is the number of triangles of its induced
      // DAG, sum over induced edges (i, x) of |N+(i) ∩ N+(x)|.  The edges
      // are split evenly over the threads (row edge counts -> block scan ->
      // each thread a contiguous edge range), so a dense row no longer
      // holds its warp.  Counts only: rows hold only bits above their own
      // index and the sum runs over whole 16-byte groups from x's group on.
      // Per-vertex: rows are symmetric; x is credited with its 3rd-vertex
      // cliques (cx) and its top-vertex cliques with (i, y), i < y < x
      // (`lower`), i with its 2nd-vertex cliques (flushed per row).
      uint32_t* rc = rP;  // free after staging: row edge-count prefix
      const bool p32 = d <= PV32_MAX_D;
      auto credit = [&](uint32_t idx, ull val) {
        if (p32)
          atomicAdd(&pvl32[idx], uint32_t(val));
        else
          atomicAdd(&pvl[idx], val);
      };
      const uint32_t ipt = (d + NT - 1) / NT;
      const uint32_t r0 = threadIdx.x * ipt, r1 = min(d, r0 + ipt);
      auto up_word = [&](const uint32_t* rr, uint32_t r, uint32_t w) -> uint32_t {
        const uint32_t v = rr[w];
        return (PV && w == (r >> 5)) ? v & above_mask(r & 31) : v;
      };
      ull mine = 0;
      for (uint32_t r = r0; r < r1; r++) {
        const uint32_t* rr = sym + size_t(r) * wp;
        uint32_t c = 0;
        for (uint32_t w = r >> 5; w < W; w++) c += __popc(up_word(rr, r, w));
        rc[r] = c;
        mine += c;
      }
      ull excl, E;
      BlockScanU64(s_scan).ExclusiveSum(mine, excl, E);
      {
        uint32_t run = uint32_t(excl);
        for (uint32_t r = r0; r < r1; r++) {
          const uint32_t c = rc[r];
          rc[r] = run;
          run += c;
        }
      }
      __syncthreads();
      const uint32_t e0 = uint32_t(E * threadIdx.x / NT), e1 = uint32_t(E * (threadIdx.x + 1) / NT);
      ull acc = 0;
      if (e0 < e1) {
        // row of edge e0: last r with rc[r] <= e0 (rows may be empty)
        uint32_t lo = 0, hi = d;
        while (hi - lo > 1) {
          const uint32_t mid = (lo + hi) >> 1;
          if (rc[mid] <= e0)
            lo = mid;
          else
            hi = mid;
        }
        uint32_t i = lo, skip = e0 - rc[lo];
        const uint32_t* ri = sym + size_t(i) * wp;
        uint32_t w = i >> 5, cur = up_word(ri, i, w);
        const uint32_t G = (W + 3) >> 2;
        ull ci = 0;  // PV: row i's 2nd-vertex credit
        for (uint32_t e = e0; e < e1; e++) {
          // next set bit in row order (skipping `skip` bits first)
          for (;;) {
            while (cur == 0) {
              if (++w >= W) {
                if constexpr (PV) {
                  if (ci) credit(i, ci);
                  ci = 0;
                }
                ++i;
                ri = sym + size_t(i) * wp;
                w = i >> 5;
                cur = up_word(ri, i, w);
              } else {
                cur = ri[w];
              }
            }
            if (skip == 0) break;
            cur &= cur - 1;
            skip--;
          }
          const uint32_t x = 32 * w + __ffs(cur) - 1;
          cur &= cur - 1;
          const uint4* ri4 = reinterpret_cast<const uint4*>(ri);
          const uint32_t* rx = sym + size_t(x) * wp;
          const uint4* rx4 = reinterpret_cast<const uint4*>(rx);
          uint32_t cx = 0;
          if constexpr (PV) {
            // one pass from i's group: all = |N+(i) ∩ N(x)| (x as 3rd or as
            // top vertex: bit x of row x is clear, so this is exactly
            // cx + #{y : i < y < x}), cx = the part above x
            const uint32_t wi = i >> 5, gx = w >> 2;
            uint32_t all = 0;
            for (uint32_t g = wi >> 2; g < G; g++) {
              const uint4 va = ri4[g], vb = rx4[g];
              uint32_t m[4] = {va.x & vb.x, va.y & vb.y, va.z & vb.z, va.w & vb.w};
              if (g == (wi >> 2)) {
#pragma unroll
                for (int j = 0; j < 4; j++) {
                  const uint32_t wd = 4 * g + j;
                  m[j] &= wd < wi ? 0u : wd == wi ? above_mask(i & 31) : FULL;
                }
              }
              all += __popc(m[0]) + __popc(m[1]) + __popc(m[2]) + __popc(m[3]);
              if (g >= gx) {
                if (g == gx) {
#pragma unroll
                  for (int j = 0; j < 4; j++) {
                    const uint32_t wd = 4 * g + j;
                    m[j] &= wd < w ? 0u : wd == w ? above_mask(x & 31) : FULL;
                  }
                }
                cx += __popc(m[0]) + __popc(m[1]) + __popc(m[2]) + __popc(m[3]);
              }
            }
            ci += cx;
            if (all) credit(x, all);
          } else {
            for (uint32_t g = w >> 2; g < G; g++) {
              const uint4 va = ri4[g], vb = rx4[g];
              cx += __popc(va.x & vb.x) + __popc(va.y & vb.y) + __popc(va.z & vb.z) +
                    __popc(va.w & vb.w);
            }
          }
          acc += cx;
        }
        if constexpr (PV) {
          if (ci) credit(i, ci);
        }
      }
      warp_src = warp_sum(acc);
    }
    // one warp per oriented edge (u, w_i) of this item's slice,
    // dynamically scheduled (low i first: the largest rows)
    for (; R != 2;) {
      uint32_t t = 0;
      if (lane == 0) t = atomicAdd(&s_edge, 1u);
      const uint32_t i = slice + nsl * __shfl_sync(FULL, t, 0);
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
      ull ce = (s0 >= uint32_t(R)) ? warp_count<PV, MAXL>(c, s0, R) : 0ull;
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
      // (k = 4 credited the u32 view: the u64 slots were zeroed whole)
      for (uint32_t i = threadIdx.x; i < d; i += NT) {
        const ull v = (R == 2 && d <= PV32_MAX_D) ? ull(pvl32[i]) : pvl[i];
        if (v) atomicAdd(&a.pv_rank[a.adj[b + i]], v);
      }
      if (threadIdx.x == 0 && s_src_total) atomicAdd(&a.pv_rank[u], s_src_total);
    }
    __syncthreads();
  }
  if (lane == 0) {
    if (my_total) atomicAdd(a.total, my_total);
    if (my_staged) atomicAdd(a.staged, my_staged);
  }
}

}  // namespace
}  // namespace kcg

#include "kcg_heavy.cuh"

namespace kcg {
namespace {

// ---------------------------------------------------------------------------
// Setup kernels
// ---------------------------------------------------------------------------
// Splits sources with d >= dmin into the warp tier list and the CTA/heavy
// candidate list (key = d for sorting).
// smask (rank space, optional): only sources r with smask[r] != 0 (the
// peeling updates count the region around a batch, kcg_peel.cu).
__global__ void classify_kernel(const uint64_t* __restrict__ off, uint32_t n, uint32_t dmin,
                                uint32_t r_lo, uint32_t r_hi,
                                const uint8_t* __restrict__ smask,
                                uint32_t* __restrict__ wlist, uint32_t* __restrict__ clist,
                                uint32_t* __restrict__ ckey, unsigned* __restrict__ cnt) {
  const uint32_t lane = threadIdx.x & 31;
  for (uint32_t base = blockIdx.x * blockDim.x; base < n; base += gridDim.x * blockDim.x) {
    const uint32_t r = base + threadIdx.x;
    uint32_t d = 0;
    if (r < n && r >= r_lo && r < r_hi && (!smask || smask[r])) d = uint32_t(off[r + 1] - off[r]);
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

// k = 2 (counting.cpp:165-173): every directed edge of a selected source is
// a 2-clique; the total is summed on the device so that partial and
// source-masked counts need no host pass over the offsets.
__global__ void k2_kernel(const uint64_t* __restrict__ rdag_off,
                          const uint32_t* __restrict__ rdag_adj, uint32_t n, uint32_t r_lo,
                          uint32_t r_hi, const uint8_t* __restrict__ smask,
                          ull* __restrict__ pv_rank, ull* __restrict__ total) {
  ull t = 0;
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    if (r < r_lo || r >= r_hi || (smask && !smask[r])) continue;
    const uint64_t b = rdag_off[r], e = rdag_off[r + 1];
    t += e - b;
    if (pv_rank) {
      if (e > b) atomicAdd(&pv_rank[r], ull(e - b));
      for (uint64_t p = b; p < e; p++) atomicAdd(&pv_rank[rdag_adj[p]], 1ull);
    }
  }
  t = warp_sum(t);
  if ((threadIdx.x & 31) == 0 && t) atomicAdd(total, t);
}

// Work estimate of source r for the multi-GPU split:
// w(r) = 1 + d + sum_{x in N+(r)} (1 + d+(x)) -- the staging reads of the
// per-source scheme (the B_alg term 4 * sum indeg * outdeg, source by
// source) -- plus d^2 for the k >= 5 edge searches.  One warp per source.
__global__ void source_work_kernel(const uint64_t* __restrict__ off,
                                   const uint32_t* __restrict__ adj, uint32_t n, int k,
                                   ull* __restrict__ w) {
  const uint32_t lane = threadIdx.x & 31;
  for (uint32_t r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < n;
       r += (gridDim.x * blockDim.x) >> 5) {
    const uint64_t b = off[r], e = off[r + 1];
    ull s = 0;
    for (uint64_t p = b + lane; p < e; p += 32) {
      const uint32_t x = adj[p];
      s += 1 + (off[x + 1] - off[x]);
    }
    s = warp_sum(s);
    if (lane == 0) {
      const ull d = e - b;
      w[r] = 1 + d + s + (k >= 5 ? d * d : 0ull);
    }
  }
}

// bounds[p] = #{r : excl(r) * P < T * p}, excl = exclusive prefix of w,
// T = its total; bounds[0] = 0, bounds[P] = n (shard.plan mirrors this)
__global__ void plan_bounds_kernel(const ull* __restrict__ excl, const ull* __restrict__ w,
                                   uint32_t n, uint32_t P, uint32_t* __restrict__ bounds) {
  const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p > P) return;
  if (p == 0 || n == 0) {
    bounds[p] = p == 0 ? 0u : n;
    return;
  }
  const unsigned __int128 T = (unsigned __int128)(excl[n - 1] + w[n - 1]) * p;
  uint32_t lo = 0, hi = n;  // first r with excl(r) * P >= T * p
  while (lo < hi) {
    const uint32_t mid = lo + (hi - lo) / 2;
    if ((unsigned __int128)excl[mid] * P < T)
      lo = mid + 1;
    else
      hi = mid;
  }
  bounds[p] = p == P ? n : lo;
}

__global__ void gather_pv_kernel(const ull* __restrict__ pv_rank, const uint32_t* __restrict__ rank,
                                 uint32_t n, ull* __restrict__ pv) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    pv[v] = pv_rank[rank[v]];
}

// bytes of the global arena one CTA of this working-set mode needs
inline size_t ws_global_bytes(int gws, const Layout& L) {
  return gws == WS_GLOBAL ? L.total : gws == WS_SYM_GLOBAL ? L.sym_bytes : 0;
}

template <bool PV, int GWS, int NT, int MAXL, int MB = 1>
void launch_cta_t(Graph& g, CtaArgs a, size_t heavy_budget, cudaStream_t st) {
  const Device& dev = device();
  auto kern = count_cta_kernel<PV, GWS, NT, MAXL, MB>;
  unsigned grid;
  size_t smem = 0;
  if (GWS != WS_GLOBAL) {
    smem = a.L.total;
    KCG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    int occ = 0;
    KCG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NT, smem));
    grid = unsigned(std::min<uint64_t>(a.nitems, uint64_t(dev.sms) * std::max(occ, 1)));
  }
  if (GWS == WS_SYM_GLOBAL) {
    // as many resident CTAs as the arena (sized by the caller) holds
    const uint64_t fit = std::min<uint64_t>(heavy_budget, g.heavy.n) / a.L.sym_bytes;
    if (fit == 0) fail(KCG_ERUNTIME, "heavy arena too small");
    grid = unsigned(std::min<uint64_t>(grid, fit));
    a.gbase = g.heavy.p;
  } else if (GWS == WS_GLOBAL) {
    const size_t per = a.L.total;
    const uint64_t fit = std::max<uint64_t>(1, heavy_budget / per);
    grid = unsigned(std::min<uint64_t>({a.nitems, uint64_t(dev.sms) * 2, fit}));
    a.gbase = g.heavy.p;  // sized by the caller before any launch
    if (size_t(grid) * per > g.heavy.n) fail(KCG_ERUNTIME, "heavy arena too small");
  }
  kern<<<grid, NT, smem, st>>>(a);
  KCG_LAUNCHED(g);
  g.stats.launches++;
}

template <bool PV, int MAXL>
void launch_cta(Graph& g, CtaArgs a, int gws, int nt, size_t heavy_budget, cudaStream_t st) {
  KCG_CUDA(cudaMemsetAsync(a.work, 0, 4, st));
  if (gws == WS_GLOBAL)
    launch_cta_t<PV, WS_GLOBAL, 512, MAXL>(g, a, heavy_budget, st);
  else if (gws == WS_SYM_GLOBAL)
    launch_cta_t<PV, WS_SYM_GLOBAL, 512, MAXL>(g, a, heavy_budget, st);
  else if (nt == 512) {
    if constexpr (MAXL == 0 && !PV) {  // lean k = 4: two 512-thread CTAs per SM
      if (a.k == 4) return launch_cta_t<PV, WS_SMEM, 512, MAXL, 2>(g, a, heavy_budget, st);
    }
    launch_cta_t<PV, WS_SMEM, 512, MAXL>(g, a, heavy_budget, st);
  }
  else if (nt == 128) {
    if constexpr (MAXL == 0 && !PV) {
      if (a.k == 4) return launch_cta_t<PV, WS_SMEM, 128, MAXL, 8>(g, a, heavy_budget, st);
    }
    fail(KCG_ERUNTIME, "128-thread counting CTAs are only planned for k = 4 counts");
  } else {
    if constexpr (MAXL == 0) {
      if (a.k == 4) return launch_cta_t<PV, WS_SMEM, 256, MAXL, 4>(g, a, heavy_budget, st);
    }
    launch_cta_t<PV, WS_SMEM, 256, MAXL, 3>(g, a, heavy_budget, st);
  }
}

// Tiled heavy launch (k = 4): 512-thread CTAs, two per SM when the
// shared-memory plan allows it.
constexpr int HV_NT = 512;
// Sources above d = 2047 need ~135 KB of tiles (one CTA per SM): those CTAs
// run 1024 threads so the SM still holds 32 warps.
constexpr int HV_NT_BIG = 1024;
inline int heavy_threads(uint32_t dmax) { return dmax > 2047 ? HV_NT_BIG : HV_NT; }

template <bool PV, int NT, int MB>
inline unsigned heavy_grid_t(const HeavyArgs& hv, uint32_t nitems) {
  auto kern = count_heavy4_kernel<NT, MB, PV>;
  KCG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                int(hv.smem_bytes)));
  int occ = 0;
  KCG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NT, hv.smem_bytes));
  return unsigned(std::min<uint64_t>(nitems, uint64_t(device().sms) * std::max(occ, 1)));
}
inline unsigned heavy_grid(const HeavyArgs& hv, uint32_t nitems) {
  if (hv.nthreads == HV_NT_BIG)
    return hv.pv_rank ? heavy_grid_t<true, HV_NT_BIG, 1>(hv, nitems)
                      : heavy_grid_t<false, HV_NT_BIG, 1>(hv, nitems);
  return hv.pv_rank ? heavy_grid_t<true, HV_NT, 2>(hv, nitems)
                    : heavy_grid_t<false, HV_NT, 2>(hv, nitems);
}
void launch_heavy4(Graph& g, HeavyArgs hv, cudaStream_t st) {
  const unsigned grid = heavy_grid(hv, hv.nitems);
  if (size_t(grid) * hv.slice_words * 4 > g.heavy.n) fail(KCG_ERUNTIME, "heavy arena too small");
  hv.gbase = reinterpret_cast<uint32_t*>(g.heavy.p);
  KCG_CUDA(cudaMemsetAsync(hv.work, 0, 4, st));
  if (hv.nthreads == HV_NT_BIG) {
    if (hv.pv_rank)
      count_heavy4_kernel<HV_NT_BIG, 1, true><<<grid, HV_NT_BIG, hv.smem_bytes, st>>>(hv);
    else
      count_heavy4_kernel<HV_NT_BIG, 1, false><<<grid, HV_NT_BIG, hv.smem_bytes, st>>>(hv);
  } else {
    if (hv.pv_rank)
      count_heavy4_kernel<HV_NT, 2, true><<<grid, HV_NT, hv.smem_bytes, st>>>(hv);
    else
      count_heavy4_kernel<HV_NT, 2, false><<<grid, HV_NT, hv.smem_bytes, st>>>(hv);
  }
  KCG_LAUNCHED(g);
  g.stats.launches++;
}

template <bool PV, int MAXL>
constexpr size_t stk_bytes() {
  return sizeof(Stacks<PV, MAXL>);
}
inline size_t stacks_size(bool pv, int maxl) {
  if (pv) return maxl > 8 ? stk_bytes<true, 32>() : stk_bytes<true, 8>();
  return maxl > 8 ? stk_bytes<false, 32>() : stk_bytes<false, 8>();
}

// Edge slices per source: only deep searches (k >= 8) pay for splitting a
// large source's edges over several CTAs, each re-staging its bitmap; up to
// k = 7 the per-edge warp scheduling inside one CTA balances well enough
// that re-staging costs more than it saves (config 2 k=5: 164 ms with
// d/64 slices vs 133 ms without; config 3 k=8: 463 vs 512 ms).
inline uint32_t slices_for(uint32_t d, int k) {
  if (k < 8 || d <= 128) return 1;
  return std::min<uint32_t>(64, d / 64);
}

// Smallest out-degree (exclusive) the tiled k = 4 kernel takes; a bin bound
// of the shared-memory tier.  Default 512: above that the shared-memory tier
// holds one or two CTAs per SM (bitmaps of 70-130 KB), while tiles of the
// L2-resident slice leave room for two 512-thread CTAs with any d (config 5
// k=4 count 1317 -> 1237 ms, per-vertex 2171 -> 1845 ms; config 2 9.20 ->
// 8.97 ms).  KCG_TILED_FROM overrides (256, 362, 512, 724, 1024).
inline uint32_t tiled_from() {
  static const uint32_t m = [] {
    const char* e = getenv("KCG_TILED_FROM");
    const long v = e ? atol(e) : 0;
    return uint32_t(v == 256 || v == 362 || v == 512 || v == 724 || v == 1024 ? v : 512);
  }();
  return m;
}

// KCG_TILED=0 sends heavy k = 4 sources down the older global-bitmap path
inline bool tiled_mode() {
  static const bool m = [] {
    const char* e = getenv("KCG_TILED");
    return !(e && e[0] == '0');
  }();
  return m;
}

inline ull* PVR(Graph& g) { return reinterpret_cast<ull*>(g.pv_rank.p); }

}  // namespace

void partition_plan(Graph& g, int k, uint32_t nparts, uint32_t* bounds) {
  if (nparts == 0) fail(KCG_EINVAL, "nparts must be positive");
  if (!g.has_rdag) fail(KCG_EINVAL, "no DAG on the handle");
  const uint32_t n = g.n;
  const size_t nb = (size_t(n) * 8 + 255) & ~size_t(255);
  unsigned char* sb = g.scratch2.ensure(2 * nb + size_t(nparts + 1) * 4 + 1024, &g.alloc);
  ull* w = reinterpret_cast<ull*>(sb);
  ull* excl = reinterpret_cast<ull*>(sb + nb);
  uint32_t* dbounds = reinterpret_cast<uint32_t*>(sb + 2 * nb);
  if (n) {
    source_work_kernel<<<blocks_for(uint64_t(n) * 32, 256), 256, 0, g.stream>>>(
        g.rdag_off.p, g.rdag_adj.p, n, k, w);
    KCG_LAUNCHED(g);
    size_t tb = 0;
    KCG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, w, excl, n, g.stream));
    KCG_CUDA(cub::DeviceScan::ExclusiveSum(cub_temp(g, tb), tb, w, excl, n, g.stream));
  }
  plan_bounds_kernel<<<(nparts + 1 + 127) / 128, 128, 0, g.stream>>>(excl, w, n, nparts,
                                                                      dbounds);
  KCG_LAUNCHED(g);
  KCG_CUDA(cudaMemcpyAsync(bounds, dbounds, size_t(nparts + 1) * 4, cudaMemcpyDeviceToHost,
                           g.stream));
  g.sync();
}

uint64_t dag_work(Graph& g) {
  if (!g.has_rdag) fail(KCG_EINVAL, "no DAG on the handle");
  const uint32_t n = g.n;
  if (n == 0) return 0;
  const size_t nb = (size_t(n) * 8 + 255) & ~size_t(255);
  unsigned char* sb = g.scratch2.ensure(nb + 256, &g.alloc);
  ull* w = reinterpret_cast<ull*>(sb);
  ull* sum = reinterpret_cast<ull*>(sb + nb);
  source_work_kernel<<<blocks_for(uint64_t(n) * 32, 256), 256, 0, g.stream>>>(
      g.rdag_off.p, g.rdag_adj.p, n, 4, w);
  KCG_LAUNCHED(g);
  size_t tb = 0;
  KCG_CUDA(cub::DeviceReduce::Sum(nullptr, tb, w, sum, n, g.stream));
  KCG_CUDA(cub::DeviceReduce::Sum(cub_temp(g, tb), tb, w, sum, n, g.stream));
  ull h = 0;
  KCG_CUDA(cudaMemcpyAsync(&h, sum, 8, cudaMemcpyDeviceToHost, g.stream));
  g.sync();
  // sum_r w(r) = n + 2m + sum_w indeg(w) * outdeg(w)
  return h - n - 2 * g.m;
}

uint64_t count_cliques(Graph& g, int k, bool want_pv, uint32_t r_lo, uint32_t r_hi) {
  if (r_lo > r_hi) fail(KCG_EINVAL, "source range must have r_lo <= r_hi");
  if (k < 2) fail(KCG_EINVAL, "k must be at least 2");
  if (!g.has_rdag) fail(KCG_EINVAL, "no DAG on the handle");
  const uint32_t n = g.n;
  g.stats = kcg_count_stats{};
  g.stats.max_out_degree = g.max_out;
  g.mark(2);
  ull* ctr = g.counters.ensure(16, &g.alloc);  // [0]=total [1]=staged [2..] work counters
  KCG_CUDA(cudaMemsetAsync(ctr, 0, 16 * 8, g.stream));
  if (want_pv) {
    g.pv_rank.ensure(size_t(n) + 1, &g.alloc);
    g.pv.ensure(size_t(n) + 1, &g.alloc);
    KCG_CUDA(cudaMemsetAsync(g.pv_rank.p, 0, size_t(n) * 8, g.stream));
  }
  if (k == 2) {
    g.mark(6);
    if (n) {
      k2_kernel<<<blocks_for(n, 256), 256, 0, g.stream>>>(g.rdag_off.p, g.rdag_adj.p, n, r_lo,
                                                         r_hi, g.src_mask,
                                                         want_pv ? PVR(g) : nullptr, ctr);
      KCG_LAUNCHED(g);
    }
    g.mark(7);
  } else if (uint64_t(k - 1) <= g.max_out) {
    // tier lists
    const uint32_t dmin = uint32_t(k - 1);
    size_t nb = (size_t(n) * 4 + 255) & ~size_t(255);
    unsigned char* sb = g.scratch2.ensure(nb * 5 + 1024, &g.alloc);
    uint32_t* wlist = reinterpret_cast<uint32_t*>(sb);
    uint32_t* clist = reinterpret_cast<uint32_t*>(sb + nb);
    uint32_t* ckey = reinterpret_cast<uint32_t*>(sb + 2 * nb);
    uint32_t* clist2 = reinterpret_cast<uint32_t*>(sb + 3 * nb);
    uint32_t* ckey2 = reinterpret_cast<uint32_t*>(sb + 4 * nb);
    unsigned* cnt = reinterpret_cast<unsigned*>(ctr + 2);
    classify_kernel<<<blocks_for(n, 256, 148u * 16u), 256, 0, g.stream>>>(
        g.rdag_off.p, n, dmin, r_lo, r_hi, g.src_mask, wlist, clist, ckey, cnt);
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
    // the tier launches are independent (they only add into the totals):
    // fork them over the handle's auxiliary streams and join before mark(7)
    KCG_CUDA(cudaEventRecord(g.fork_ev, g.stream));
    for (int i = 0; i < Graph::kAux; i++) KCG_CUDA(cudaStreamWaitEvent(g.aux[i], g.fork_ev, 0));
    int next_aux = 1;  // aux[0] serialises the global-memory (heavy) launches
    auto aux_stream = [&](bool gws) {
      if (gws) return g.aux[0];
      cudaStream_t s = g.aux[next_aux];
      next_aux = next_aux % (Graph::kAux - 1) + 1;
      return s;
    };
    if (nw && k <= 34) {
      const bool big = k > 10;
      const size_t dsm = k >= 5 ? size_t(WARP_TIER_WARPS) * stacks_size(want_pv, big ? 32 : 8) : 0;
      // kernels without the DFS engine when it cannot run (k <= 4): its
      // warp-synchronous loop would otherwise shape the code of the whole
      // kernel
      unsigned grid = blocks_for(uint64_t(nw) * 32, WARP_THREADS_BLOCK, dev.sms * 8u);
      auto run = [&](auto kern) {
        KCG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(dsm)));
        kern<<<grid, WARP_THREADS_BLOCK, dsm, aux_stream(false)>>>(g.rdag_off.p, g.rdag_adj.p, wlist, nw, k,
                                                          ctr, PVR(g), ctr + 1);
      };
      if (want_pv)
        k <= 4 ? run(count_warp_kernel<true, 0>)
               : big ? run(count_warp_kernel<true, 32>) : run(count_warp_kernel<true, 8>);
      else
        k <= 4 ? run(count_warp_kernel<false, 0>)
               : big ? run(count_warp_kernel<false, 32>) : run(count_warp_kernel<false, 8>);
      KCG_LAUNCHED(g);
      g.stats.launches++;
    }
    g.stats.sources_warp = nw;
    if (nc) {
      // bins in descending d: [heavy] (512,1024] (256,512] (128,256] (64,128] (32,64]
      const uint32_t R = uint32_t(k - 2);
      auto deg_at = [&](uint32_t i) { return 0xffffffffu - keys[i]; };
      std::vector<uint32_t> verts(nc);
      KCG_CUDA(cudaMemcpyAsync(verts.data(), clist, size_t(nc) * 4, cudaMemcpyDeviceToHost,
                               g.stream));
      g.sync();
      // work items (source, edge slice), heaviest sources first
      std::vector<uint32_t> isrc, isl;
      std::vector<uint32_t> first(nc + 1);
      for (uint32_t i = 0; i < nc; i++) {
        first[i] = uint32_t(isrc.size());
        const uint32_t ns = slices_for(deg_at(i), k);
        for (uint32_t s = 0; s < ns; s++) {
          isrc.push_back(verts[i]);
          isl.push_back((s << 16) | ns);
        }
      }
      first[nc] = uint32_t(isrc.size());
      const size_t ni = isrc.size();
      uint32_t* d_items = reinterpret_cast<uint32_t*>(g.scratch3.ensure(ni * 8 + 16, &g.alloc));
      KCG_CUDA(cudaMemcpyAsync(d_items, isrc.data(), ni * 4, cudaMemcpyHostToDevice, g.stream));
      KCG_CUDA(cudaMemcpyAsync(d_items + ni, isl.data(), ni * 4, cudaMemcpyHostToDevice,
                               g.stream));
      unsigned* work = cnt + 2;
      int wslot = 0;
      CtaArgs a{};
      a.off = g.rdag_off.p;
      a.adj = g.rdag_adj.p;
      a.k = k;
      a.total = ctr;
      a.pv_rank = PVR(g);
      a.staged = ctr + 1;
      const size_t budget = size_t(8) << 30;
      const uint32_t levels = std::max<uint32_t>(R, 1);
      const bool big = k > 10;  // DFS engine stack depth 32 instead of 8
      // the engine runs inside compacted edge sets only when 3+ vertices
      // remain below the compacted vertex (k >= 6)
      const size_t sbytes = k >= 6 ? stacks_size(want_pv, big ? 32 : 8) : 0;
      struct Plan {
        uint32_t lo, hi;
        Layout L;
        int gws;  // WS_*
        int nt;
        HeavyArgs hv;  // WS_TILED
      };
      std::vector<Plan> plans;
      const size_t smem_cap = size_t(dev.smem_optin) - 1024;
      // the arena is sized before the launches: the plan already says which
      // kernel (per-vertex or totals) it is for
      auto tiled_plan = [&](uint32_t dmax) {
        int nt = heavy_threads(dmax);
        HeavyArgs hv = heavy_plan(dmax, nt / 32, want_pv);
        if (hv.smem_bytes > smem_cap && nt != HV_NT) {
          // 32 flag rows of a near-4095 source no longer fit next to the table
          nt = HV_NT;
          hv = heavy_plan(dmax, nt / 32, want_pv);
        }
        if (hv.smem_bytes > smem_cap) fail(KCG_ERUNTIME, "tiled plan exceeds shared memory");
        hv.nthreads = nt;
        hv.pv_rank = want_pv ? PVR(g) : nullptr;
        return hv;
      };
      // a working set that does not fit shared memory: bitmap in global
      // memory and the rest in shared memory if that fits, else all global
      auto global_plan = [&](uint32_t lo, uint32_t hi, uint32_t dmax) {
        Layout Ls = make_layout(dmax, levels, want_pv, 16, sbytes, true);
        if (Ls.total <= smem_cap)
          plans.push_back({lo, hi, Ls, WS_SYM_GLOBAL, 512, HeavyArgs{}});
        else
          plans.push_back({lo, hi, make_layout(dmax, levels, want_pv, 16, sbytes), WS_GLOBAL,
                           512, HeavyArgs{}});
      };
      // heavy: d > smem_max (k = 4: the tiled kernel may start lower than
      // the largest bitmap shared memory can hold, see tiled_from)
      const bool tiled = k == 4 && tiled_mode();
      const uint32_t smem_max = tiled ? tiled_from() : SMEM_TIER_MAX;
      uint32_t pos = 0;
      while (pos < nc && deg_at(pos) > smem_max) pos++;
      if (pos) {
        if (tiled) {
          // tiled kernel up to HV_DMAX, binned (bucket table and tile sizes
          // follow the bin's largest source); beyond that the old path
          uint32_t p0 = 0;
          while (p0 < pos && deg_at(p0) > HV_DMAX) p0++;
          if (p0) global_plan(0, p0, deg_at(0));
          const uint32_t tb[] = {2047, 1024, 724, 512, 362, 256, 0};
          for (uint32_t lo : tb) {
            uint32_t p1 = p0;
            while (p1 < pos && deg_at(p1) > lo) p1++;
            if (p1 > p0)
              plans.push_back({p0, p1, Layout{}, WS_TILED, HV_NT, tiled_plan(deg_at(p0))});
            p0 = p1;
          }
        } else {
          global_plan(0, pos, deg_at(0));
        }
        g.stats.sources_heavy = pos;
      }
      // shared-memory bins, sqrt(2) apart so each bin's footprint (and
      // occupancy) tracks its degrees
      const uint32_t bounds[] = {SMEM_TIER_MAX, 724, 512, 362, 256, 181, 128, 90, 64, 45, 32};
      const int nbounds = sizeof(bounds) / sizeof(bounds[0]);
      for (int bi = 0; bi + 1 < nbounds && pos < nc; bi++) {
        const uint32_t hi = bounds[bi], lo = bounds[bi + 1];
        uint32_t end = pos;
        while (end < nc && deg_at(end) > lo) end++;
        if (end == pos) continue;
        const bool lean = k == 4 && !want_pv;
        // lean small sources: 128-thread CTAs (per-source barriers and
        // scans over fewer warps, more sources in flight per SM)
        const int nt = hi > 512 ? 512 : (lean && hi <= 256) ? 128 : 256;
        Layout Lb = make_layout(hi, levels, want_pv, nt / 32, sbytes, false, lean);
        if (Lb.total > smem_cap)
          global_plan(pos, end, deg_at(pos));
        else
          plans.push_back({pos, end, Lb, WS_SMEM, nt, HeavyArgs{}});
        g.stats.sources_cta += end - pos;
        pos = end;
      }
      // one heavy arena for all global-memory launches (they run in order
      // on aux[0])
      size_t arena = 0;
      for (const Plan& pl : plans)
        if (pl.gws == WS_TILED) {
          arena = std::max<size_t>(
              arena, size_t(heavy_grid(pl.hv, first[pl.hi] - first[pl.lo])) * pl.hv.slice_words * 4);
        } else if (pl.gws != WS_SMEM) {
          const size_t per = ws_global_bytes(pl.gws, pl.L);
          const uint64_t fit = std::max<uint64_t>(1, budget / per);
          // resident CTAs: <= 4 per SM at 512 threads (2 for all-global)
          const uint64_t res = uint64_t(dev.sms) * (pl.gws == WS_SYM_GLOBAL ? 4 : 2);
          const uint64_t grid =
              std::min<uint64_t>({uint64_t(first[pl.hi] - first[pl.lo]), res, fit});
          arena = std::max<size_t>(arena, grid * per);
        }
      if (arena) g.heavy.ensure(arena, &g.alloc);
      // the CTA launches read d_items and the heavy arena, which g.stream
      // only just uploaded / allocated: re-fork after that work (a wait
      // captures the event as recorded at call time, so re-recording the
      // same event is safe; the warp tier above keeps running)
      KCG_CUDA(cudaEventRecord(g.fork_ev, g.stream));
      for (int i = 0; i < Graph::kAux; i++) KCG_CUDA(cudaStreamWaitEvent(g.aux[i], g.fork_ev, 0));
      for (const Plan& pl : plans) {
        if (pl.gws == WS_TILED) {
          HeavyArgs hv = pl.hv;
          hv.off = g.rdag_off.p;
          hv.adj = g.rdag_adj.p;
          hv.item_src = d_items + first[pl.lo];
          hv.nitems = first[pl.hi] - first[pl.lo];
          hv.total = ctr;
          hv.staged = ctr + 1;
          hv.work = work + wslot++;
          launch_heavy4(g, hv, aux_stream(true));
          continue;
        }
        a.item_src = d_items + first[pl.lo];
        a.item_sl = d_items + ni + first[pl.lo];
        a.nitems = first[pl.hi] - first[pl.lo];
        a.L = pl.L;
        a.work = work + wslot++;
        cudaStream_t st = aux_stream(pl.gws != WS_SMEM);
        if (want_pv) {
          if (k <= 5)
            launch_cta<true, 0>(g, a, pl.gws, pl.nt, budget, st);
          else
            big ? launch_cta<true, 32>(g, a, pl.gws, pl.nt, budget, st)
                : launch_cta<true, 8>(g, a, pl.gws, pl.nt, budget, st);
        } else {
          if (k <= 5)
            launch_cta<false, 0>(g, a, pl.gws, pl.nt, budget, st);
          else
            big ? launch_cta<false, 32>(g, a, pl.gws, pl.nt, budget, st)
                : launch_cta<false, 8>(g, a, pl.gws, pl.nt, budget, st);
        }
      }
    }
    // join the auxiliary streams
    for (int i = 0; i < Graph::kAux; i++) {
      KCG_CUDA(cudaEventRecord(g.join_ev[i], g.aux[i]));
      KCG_CUDA(cudaStreamWaitEvent(g.stream, g.join_ev[i], 0));
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
  const uint64_t total = hv[0];
  g.stats.staged_elems = hv[1];
  g.times.count_ms = g.elapsed(2, 3);
  g.times.count_kernel_ms = g.elapsed(6, 7);
  return total;
}

}  // namespace kcg
