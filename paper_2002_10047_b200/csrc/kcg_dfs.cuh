// Warp-synchronous DFS with intra-warp work stealing over <= 32-vertex
// clique-counting problems (included by kcg_count.cu).
//
// A problem is one word per vertex: usym[v] = neighbours above v (its
// out-neighbourhood in local topological order), sym[v] = all neighbours.
// Each lane runs a depth-first search; a node holds its candidate set N
// (children are built from it) and the not-yet-chosen iteration set
// I ⊆ N.  One step pops the lowest x of I; at the last-but-one level it
// counts the completions popc(N ∩ N+(x)), otherwise it pushes the child
// N ∩ N+(x).  This is the reference's recursion clique_rec
// (proj/src/clique_rec.hpp:24-62) with its candidate filter and its
// "|cands| < remaining" pruning, on bitmaps.
//
// The current node lives in registers; only pushes and pops touch the
// shared-memory stack, so the common (leaf) step is a handful of ALU ops.
// Every STEPS steps the warp looks for idle lanes: an idle lane takes the
// upper half of the I-set of a busy lane's shallowest node with >= 2
// unchosen candidates (N stays shared), so no lane waits on another's
// subtree.
//
// Per-vertex counts (PV): inside a leaf node (two vertices still to choose)
// every v ∈ N is credited with its degree inside N; every other chosen
// vertex is credited with its subtree count when its node is done; a lane
// finishing a stolen node credits the whole chain above it.
#pragma once

namespace kcg {
namespace {

template <bool PV, int MAXL>
struct Stacks {
  uint2 ni[MAXL][32];                 // saved ancestors (N, I) per level per lane
  uint32_t X[PV ? MAXL + 1 : 1][32];  // chain: X[0] root, X[l] created node l
  ull sub[PV ? MAXL : 1][32];         // subtree counts per level
};

// Compact-problem per-vertex counters are 32-bit: within one problem of
// <= 32 vertices a vertex lies in at most C(31,15) < 2^32 cliques, and the
// counters are flushed to 64-bit per problem.
typedef uint32_t pvc_t;

// Steps between steal checks.  The per-vertex engine carries more state per
// step and profits from rebalancing sooner (config 4 k=6 per-vertex: 234 ms
// at 16, 135 at 8, 91 at 4, 99 at 1); totals are best at 8.
// CTA: the call from the CTA tier's compacted sets (short, skewed
// problems: config 3 k=6 84.4 -> 80.8 ms at 4).
template <bool PV, bool CTA>
constexpr int dfs_steps() {
  return (PV || CTA) ? 4 : 8;
}

// Per-vertex credit of leaf nodes, transposed: every lane that created a
// leaf node N this step broadcasts it and lane v adds its degree inside N
// (popc(N ∩ N(v))) to its own register accumulator `acc`.  Called by all
// 32 lanes.
__device__ __forceinline__ void leaf_pv_collect(bool made, uint32_t N, uint32_t my_sym,
                                                uint32_t lane, pvc_t& acc) {
  unsigned mk = __ballot_sync(0xffffffffu, made);
  while (mk) {
    const int c = __ffs(mk) - 1;
    mk &= mk - 1;
    const uint32_t Nc = __shfl_sync(0xffffffffu, N, c);
    if ((Nc >> lane) & 1u) acc += __popc(Nc & my_sym);
  }
}

// R == 2 needs no stack: one loop over N per lane (the last two vertices).
// Must be called by all 32 lanes (PV uses warp collectives).
template <bool PV>
__device__ __forceinline__ ull lane_pairs(bool active, uint32_t N, uint32_t root_v,
                                          const uint32_t* usym, const uint32_t* sym, pvc_t* cpv,
                                          uint32_t lane) {
  ull t = 0;
  if (active) {
    for (uint32_t b = N; b;) {
      const int x = __ffs(b) - 1;
      b &= b - 1;
      t += __popc(N & usym[x]);
    }
  }
  if constexpr (PV) {
    pvc_t acc = 0;
    leaf_pv_collect(t != 0, N, sym[lane], lane, acc);
    if (acc) atomicAdd(&cpv[lane], acc);
    if (t) atomicAdd(&cpv[root_v], pvc_t(t));
  }
  return t;
}

// Splits an iteration set with >= 2 bits at the midpoint of its lowest and
// highest bit: returns the upper part (non-empty), the caller keeps the rest.
__device__ __forceinline__ uint32_t upper_split(uint32_t I) {
  const int lo = __ffs(I) - 1, hi = 31 - __clz(I);
  const int mid = (lo + hi + 1) >> 1;  // lo < mid <= hi
  return I & (0xffffffffu << mid);
}

// Counts, summed over the warp, the R-cliques (R >= 2) inside each active
// lane's root set N0; root_v is the lane's chain vertex for PV.  Returns
// this lane's share of the total.  Must be called by all 32 lanes; `map`
// is 32 words of warp-private shared memory.
template <bool PV, int MAXL, bool CTA = false>
__device__ ull steal_count(bool active, uint32_t N0, int R, uint32_t root_v,
                           const uint32_t* usym, const uint32_t* sym, pvc_t* cpv,
                           Stacks<PV, MAXL>& st, uint32_t* map, uint32_t lane) {
  constexpr uint32_t FULLM = 0xffffffffu;
  const uint32_t lt_mask = (1u << lane) - 1u;
  int base = 0, lvl = -1;
  uint32_t cN = 0, cI = 0;  // current node
  uint32_t smask = 0;       // ancestor levels (< lvl) with >= 2 unchosen
  ull total = 0;
  ull csub = 0;  // PV: subtree count of the current node
  pvc_t acc = 0;  // PV: leaf credit of compact vertex `lane`
  const uint32_t my_sym = PV ? sym[lane] : 0u;
  if (active && __popc(N0) >= R) {
    lvl = 0;
    cN = cI = N0;
    if constexpr (PV) st.X[0][lane] = root_v;
  }
  if constexpr (PV) leaf_pv_collect(lvl == 0 && R == 2, N0, my_sym, lane, acc);
  // A node with three vertices still to choose is never pushed: choosing x
  // there leaves the leaf node lN = N ∩ N+(x), whose pairs are counted by an
  // inner loop over y ∈ lN held in registers (lJ = the y not yet visited).
  // These are most of the tree's nodes, so the stack only sees the levels
  // above them.  PV: y is credited with its degree inside lN (every pair
  // (y, z) of lN closes one clique and credits both ends), x with the
  // node's count when the loop ends.
  uint32_t lN = 0, lJ = 0, lx = 0;
  pvc_t lsum = 0;
  for (;;) {
#pragma unroll
    for (int t = 0; t < dfs_steps<PV, CTA>(); t++) {
      if (lJ) {
        const int y = __ffs(lJ) - 1;
        lJ &= lJ - 1;
        const uint32_t cs = __popc(lN & usym[y]);
        total += cs;
        if constexpr (PV) {
          lsum += cs;
          const uint32_t ca = __popc(lN & sym[y]);
          if (ca) atomicAdd(&cpv[y], pvc_t(ca));
          if (lJ == 0) {
            if (lsum) atomicAdd(&cpv[lx], lsum);
            csub += lsum;
          }
        }
      } else if (lvl >= base) {
        if (cI == 0) {
          // node exhausted: credit and pop
          if constexpr (PV) {
            if (lvl > base) {
              if (csub) atomicAdd(&cpv[st.X[lvl][lane]], pvc_t(csub));
              csub += st.sub[lvl - 1][lane];
            } else if (csub) {
              for (int l = 0; l <= base; l++) atomicAdd(&cpv[st.X[l][lane]], pvc_t(csub));
            }
          }
          if (lvl > base) {
            const uint2 nd = st.ni[lvl - 1][lane];
            cN = nd.x;
            cI = nd.y;
            smask &= ~(1u << (lvl - 1));
          }
          lvl--;
        } else {
          const int x = __ffs(cI) - 1;
          cI &= cI - 1;
          const uint32_t child = cN & usym[x];
          const uint32_t cs = __popc(child);
          const int r = R - lvl;
          if (r == 2) {
            total += cs;
            if constexpr (PV) csub += cs;
          } else if (r == 3) {
            if (cs >= 2) {
              lN = lJ = child;
              if constexpr (PV) {
                lx = x;
                lsum = 0;
              }
            }
          } else if (cs >= uint32_t(r - 1)) {
            st.ni[lvl][lane] = make_uint2(cN, cI);
            if (cI & (cI - 1)) smask |= 1u << lvl;
            if constexpr (PV) {
              st.sub[lvl][lane] = csub;
              csub = 0;
              st.X[lvl + 1][lane] = x;
            }
            lvl++;
            cN = cI = child;
          }
        }
      }
    }
    const bool busy = lvl >= base;
    const unsigned busym = __ballot_sync(FULLM, busy);
    if (busym == 0) break;
    const unsigned idle = ~busym;
    if (__popc(idle) < 4 && __popc(busym) > 4) continue;
    // work stealing: idle lanes take the upper half of a donor's
    // shallowest node with >= 2 unchosen candidates
    const bool can_give = busy && (smask != 0 || (cI & (cI - 1)) != 0);
    const unsigned don = __ballot_sync(FULLM, can_give);
    if (!don) continue;
    const uint32_t np = min(__popc(idle), __popc(don));
    const uint32_t td = __popc(don & lt_mask), ti = __popc(idle & lt_mask);
    const bool giver = can_give && td < np;
    const bool thief = !busy && ti < np;
    int gl = 0;
    uint32_t gift = 0;
    if (giver) {
      gl = smask ? __ffs(smask) - 1 : lvl;
      const uint32_t I = gl < lvl ? st.ni[gl][lane].y : cI;
      gift = upper_split(I);
      const uint32_t kept = I & ~gift;
      if (gl < lvl) {
        st.ni[gl][lane].y = kept;
        if (!(kept & (kept - 1))) smask &= ~(1u << gl);
      } else {
        cI = kept;
      }
      map[td] = lane;
    }
    // giver publishes (N, gift, level) for its thief
    const uint32_t gN = gl < lvl ? st.ni[gl][lane].x : cN;
    __syncwarp();
    const uint32_t dl = thief ? map[ti] : lane;
    const uint32_t dN = __shfl_sync(FULLM, gN, dl);
    const uint32_t dG = __shfl_sync(FULLM, gift, dl);
    const int dgl = __shfl_sync(FULLM, gl, dl);
    if (thief) {
      base = lvl = dgl;
      cN = dN;
      cI = dG;
      smask = 0;
      if constexpr (PV) {
        for (int l = 0; l <= dgl; l++) st.X[l][lane] = st.X[l][dl];
        csub = 0;
      }
    }
    __syncwarp();
  }
  if constexpr (PV) {
    if (acc) atomicAdd(&cpv[lane], acc);
  }
  return total;
}

}  // namespace
}  // namespace kcg
