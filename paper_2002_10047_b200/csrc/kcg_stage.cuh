// Staging of a source's induced subgraph (included by kcg_count.cu).
//
// For source u with out-neighbours w_0 < ... < w_{d-1} (ranks), row i of the
// symmetric bitmap gets bit j for every w_j ∈ N+(w_i).  The reference builds
// the same induced subgraph by stamping N+(v) and filtering every N+(w)
// (proj/src/counting.cpp:21-48); here N+(u) sits in a shared-memory
// open-addressing table behind a 1-bit-per-slot filter and the rows N+(w_i)
// are scanned flattened:
//
//  * long rows (>= 32 entries): a 32-element chunk spans at most two rows,
//    so a lane's row is one compare against a warp-uniform boundary;
//  * short rows: a lane finds its row from the bitmask of row starts inside
//    the chunk (one REDUX.OR);
//  * STAGE_U chunks issue their global loads before any lookup (several
//    loads in flight per lane);
//  * filter → compact → batch: lanes whose element passes the filter append
//    it to a 64-entry warp queue; probes and the two shared atomics run only
//    on full batches of 32, so the rare hits never drag the whole warp
//    through a divergent path.
#pragma once

namespace kcg {
namespace {

constexpr ull EMPTY64 = ~0ull;
constexpr int STAGE_U = 4;

// Open-addressing table of (key | local index << 32) plus a filter.
struct Member {
  ull* table;
  uint32_t* filter;
  uint32_t tbits, fbits;
};

__device__ __forceinline__ void member_insert(const Member& M, uint32_t key, uint32_t idx) {
  const uint32_t h = key * 0x9E3779B1u;
  const uint32_t fb = h >> (32 - M.fbits);
  atomicOr(&M.filter[fb >> 5], 1u << (fb & 31));
  const uint32_t mask = (1u << M.tbits) - 1;
  uint32_t slot = h >> (32 - M.tbits);
  const ull packed = ull(key) | (ull(idx) << 32);
  while (atomicCAS(&M.table[slot], EMPTY64, packed) != EMPTY64) slot = (slot + 1) & mask;
}

__device__ __forceinline__ bool member_maybe(const Member& M, uint32_t key) {
  const uint32_t fb = (key * 0x9E3779B1u) >> (32 - M.fbits);
  return (M.filter[fb >> 5] >> (fb & 31)) & 1u;
}

__device__ __forceinline__ uint32_t member_probe(const Member& M, uint32_t key) {
  const uint32_t mask = (1u << M.tbits) - 1;
  uint32_t slot = (key * 0x9E3779B1u) >> (32 - M.tbits);
  for (;;) {
    const ull e = M.table[slot];
    if (uint32_t(e) == key) return uint32_t(e >> 32);
    if (uint32_t(e) == EMPTY) return NOTFOUND;
    slot = (slot + 1) & mask;
  }
}

// Non-empty rows of a source in local order: row r is N+(w_rowid[r]),
// global elements adj[rbase[r] ..), first virtual position P[r]; P[nr] = L.
struct Rows {
  const uint32_t* P;
  const ull* rbase;
  const uint32_t* rowid;
  uint32_t nr;
};

// Warp-private batching of filter-passing candidates.  SYM: also set the
// mirrored bit (row j, column i); only the per-vertex paths read the lower
// triangle, every counting path reads rows above their own index.
template <bool SYM>
struct Stager {
  Member M;
  uint32_t* sym;
  uint32_t wp;
  uint32_t* qy;  // 64 entries
  uint32_t* qi;  // 64 entries
  uint32_t lane;
  uint32_t qn;   // warp-uniform queue length
  bool combine;  // pre-combine same-word hits before the atomic

  // Called by all 32 lanes; `valid` lanes hold a queued candidate.  With
  // `combine`, hits of one batch that land in the same bitmap word are
  // OR-ed together first -- lanes grouped by address (MATCH), one REDUX.OR
  // per group -- and only the group's first lane issues the atomic
  // (same-word lanes of one ATOMS serialise on the bank).
  __device__ __forceinline__ void set(uint32_t y, uint32_t i, bool valid) {
    const uint32_t j = valid ? member_probe(M, y) : NOTFOUND;
    const bool hit = j != NOTFOUND;
    const uint32_t addr = hit ? i * wp + (j >> 5) : 0xffffffffu;
    const uint32_t bits = hit ? 1u << (j & 31) : 0u;
    if (combine) {
      const unsigned mm = __match_any_sync(FULL, addr);
      const uint32_t word = __reduce_or_sync(mm, bits);
      if (hit && lane == uint32_t(__ffs(mm) - 1)) atomicOr(&sym[addr], word);
    } else if (hit) {
      atomicOr(&sym[addr], bits);
    }
    if constexpr (SYM) {
      if (hit) atomicOr(&sym[j * wp + (i >> 5)], 1u << (i & 31));
    }
  }
  __device__ __forceinline__ void push(bool pass, uint32_t y, uint32_t row) {
    const unsigned bal = __ballot_sync(FULL, pass);
    if (pass) {
      const uint32_t pos = qn + __popc(bal & ((1u << lane) - 1u));
      qy[pos] = y;
      qi[pos] = row;
    }
    qn += __popc(bal);
    if (qn >= 32) {
      __syncwarp();
      const uint32_t y0 = qy[lane], i0 = qi[lane];
      const bool mv = lane + 32 < qn;
      uint32_t y1 = 0, i1 = 0;
      if (mv) {
        y1 = qy[lane + 32];
        i1 = qi[lane + 32];
      }
      __syncwarp();
      if (mv) {
        qy[lane] = y1;
        qi[lane] = i1;
      }
      qn -= 32;
      set(y0, i0, true);
      __syncwarp();
    }
  }
  __device__ __forceinline__ void flush() {
    __syncwarp();
    const bool v = lane < qn;
    set(v ? qy[lane] : 0u, v ? qi[lane] : 0u, v);
    qn = 0;
    __syncwarp();
  }
};

__device__ __forceinline__ uint32_t row_search(const Rows& R, uint32_t pbeg) {
  uint32_t lo = 0, hi = R.nr;  // P[lo] <= pbeg < P[hi]
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (R.P[mid] <= pbeg)
      lo = mid;
    else
      hi = mid;
  }
  return lo;
}

// Short rows: virtual positions [pbeg, pend), 32 per chunk.
template <class ST>
__device__ __forceinline__ void stage_short(const Rows& R, ST& S,
                                            const uint32_t* __restrict__ adj, uint32_t pbeg,
                                            uint32_t pend) {
  if (pbeg >= pend) return;
  const uint32_t lane = S.lane;
  uint32_t cur = row_search(R, pbeg), pcur = R.P[cur];
  const uint32_t le_mask = (2u << lane) - 1u;
  for (uint32_t c0 = pbeg; c0 < pend; c0 += 32 * STAGE_U) {
    uint32_t y[STAGE_U], row[STAGE_U];
#pragma unroll
    for (int u = 0; u < STAGE_U; u++) {
      const uint32_t cb = c0 + 32 * u;
      const uint32_t p = cb + lane;
      const uint32_t jn = cur + 1 + lane;
      const uint32_t pn = jn <= R.nr ? R.P[jn] : 0xffffffffu;
      const uint32_t rel = pn - cb;
      const uint32_t starts = __reduce_or_sync(FULL, rel < 32u ? (1u << rel) : 0u);
      const uint32_t kk = __popc(starts & le_mask);
      const uint32_t seg = cur + kk;
      uint32_t pseg = __shfl_sync(FULL, pn, (kk - 1) & 31);
      if (kk == 0) pseg = pcur;
      const uint32_t adv = __popc(__ballot_sync(FULL, pn <= cb + 32));
      const uint32_t pnext = __shfl_sync(FULL, pn, (adv - 1) & 31);
      if (adv) pcur = pnext;
      cur += adv;
      y[u] = EMPTY;
      row[u] = 0;
      if (p < pend) {
        y[u] = __ldg(adj + R.rbase[seg] + (p - pseg));
        row[u] = R.rowid[seg];
      }
    }
#pragma unroll
    for (int u = 0; u < STAGE_U; u++)
      S.push(y[u] != EMPTY && member_maybe(S.M, y[u]), y[u], row[u]);
  }
}

// Long rows (>= 32 entries): a lane's row is one compare per chunk.
template <class ST>
__device__ __forceinline__ void stage_long(const Rows& R, ST& S,
                                           const uint32_t* __restrict__ adj, uint32_t pbeg,
                                           uint32_t pend) {
  if (pbeg >= pend) return;
  const uint32_t lane = S.lane;
  uint32_t cur = row_search(R, pbeg);
  uint32_t pnext = R.P[cur + 1];
  ull bcur = R.rbase[cur] - R.P[cur];
  uint32_t rcur = R.rowid[cur];
  ull bnxt = 0;
  uint32_t rnxt = 0;
  if (cur + 1 < R.nr) {
    bnxt = R.rbase[cur + 1] - pnext;
    rnxt = R.rowid[cur + 1];
  }
  for (uint32_t c0 = pbeg; c0 < pend; c0 += 32 * STAGE_U) {
    uint32_t y[STAGE_U], row[STAGE_U];
#pragma unroll
    for (int u = 0; u < STAGE_U; u++) {
      const uint32_t cb = c0 + 32 * u;
      const uint32_t p = cb + lane;
      const bool nx = p >= pnext;
      y[u] = EMPTY;
      row[u] = nx ? rnxt : rcur;
      if (p < pend) y[u] = __ldg(adj + (nx ? bnxt : bcur) + p);
      if (cb + 32 >= pnext && cb + 32 < pend) {  // warp-uniform row advance
        cur++;
        bcur = bnxt;
        rcur = rnxt;
        pnext = R.P[cur + 1];
        if (cur + 1 < R.nr) {
          bnxt = R.rbase[cur + 1] - pnext;
          rnxt = R.rowid[cur + 1];
        }
      }
    }
#pragma unroll
    for (int u = 0; u < STAGE_U; u++)
      S.push(y[u] != EMPTY && member_maybe(S.M, y[u]), y[u], row[u]);
  }
}

}  // namespace
}  // namespace kcg
