// Staging of a source's induced subgraph (included by kcg_count.cu).
//
// For source u with out-neighbours w_0 < ... < w_{d-1} (ranks), row i of the
// bitmap gets bit j for every w_j ∈ N+(w_i).  The reference builds the same
// induced subgraph by stamping N+(v) and filtering every N+(w)
// (proj/src/counting.cpp:21-48); here N+(u) sits in a shared-memory bucketed
// table and warps scan whole rows N+(w_i) against it.
#pragma once
#ifndef KCG_FILTER
#define KCG_FILTER 1
#endif

namespace kcg {
namespace {

__device__ __forceinline__ uint32_t popc_and4(const uint4& a, const uint4& b) {
  return __popc(a.x & b.x) + __popc(a.y & b.y) + __popc(a.z & b.z) + __popc(a.w & b.w);
}
constexpr int STAGE_U = 4;

// ---------------------------------------------------------------------------
// Row-per-warp staging with a bucketed membership table (every tier).
//
// The staging loop is bound by the LSU data pipe (shared-memory and global
// wavefronts: 75-99 % of peak before the filter words below, about two
// thirds now) together with the issue slots (profiles/r02_notes.md), so
// every element costs as few shared wavefronts and instructions as possible:
//
//  * N+(u) is hashed into B = 2^bb >= d+1 buckets of four u32 slots.  The
//    hash h = y * mul (odd mul: a bijection of u32) names the bucket by its
//    top bb bits; a slot stores h << bb (the other 32-bb bits of h) plus the
//    local index (idx < d < B fits the low bb bits).  For a probe,
//    slot - (h << bb) is the index when the slot holds y and >= B otherwise
//    (mod 2^32), so one LDS.128, four subtractions and three unsigned
//    minima give the index or a miss (empty slots are all ones and decode
//    to B-1, the miss code).  The multiplier is chosen per source so that
//    no bucket holds more than four keys (a few retries at most); only if
//    eight multipliers fail does the source fall back to an overflow list
//    (CTA-uniform flag; taken by sources whose d approaches a large B, e.g.
//    d ~ 2000 in 2048 buckets on config 5's hubs).  After the inserts the
//    insert counters become one filter word per bucket (bucket_filter): a
//    probe reads the word first and only filter-positive lanes load the
//    bucket.
//  * Warps take whole rows N+(w_i) from a shared counter (row i is then
//    written by one warp only) and read them 128 elements per step.  A hit
//    writes a byte flag at its local index in the warp's flag row (plain
//    STS.U8, no atomics: distinct indices); when the row is done, ballots
//    turn the flags into row i's words, four per LDS.32 (flag_pos), and
//    clear them.  The next 128 entries are always in flight (stage_scan).
//
// The reference's equivalent is the stamp test of counting.cpp:31-40.
// ---------------------------------------------------------------------------
constexpr uint32_t BKT_OVF_CAP = 64;
constexpr uint32_t BKT_HASH = 0x9E3779B1u;
constexpr uint32_t BKT_TRIES = 8;

struct Buckets {
  uint4* keys;      // B buckets x 4 slots (EMPTY = all ones)
  uint32_t* cnt;    // B insert counts
  uint32_t* flag;   // B bits: bucket overflowed (overflow mode)
  uint2* ovf;       // (key, local index), BKT_OVF_CAP entries
  uint32_t* ovf_n;  // overflow entries used
  uint32_t bb;      // log2 B
  uint32_t mul;     // hash multiplier (odd)
  bool ovf_mode;    // CTA-uniform: some bucket holds more than four keys
};

// Flag byte of local index j in a warp's flag row: groups of 128 indices,
// lane-major inside a group (index 128g + 32k + l is byte k of u32 32g + l),
// so one LDS.32 per lane and four ballots give the group's four bitmap words.
// A bijection of [0, B) for B >= 128 with flag_pos(B-1) = B-1, so positions
// fit the table's index field and never equal the miss code.
__host__ __device__ inline uint32_t flag_pos(uint32_t j) {
  return (j & ~127u) | ((j & 31u) << 2) | ((j >> 5) & 3u);
}
// bytes of a flag row for bitmap rows of W words
__host__ __device__ inline size_t flag_row_bytes(uint32_t W) { return size_t(128) * ((W + 3) / 4); }

// B = 2^bb >= d + 1 (index B-1 is the miss code), at least 128 (flag_pos)
__host__ __device__ inline uint32_t bucket_bits(uint32_t d) {
  uint32_t bb = 7;
  while ((1u << bb) < d + 1) bb++;
  return bb;
}
// bytes of a bucket table for sources of out-degree <= dmax
__host__ __device__ inline size_t bucket_bytes(uint32_t dmax) {
  const size_t B = size_t(1) << bucket_bits(dmax);
  return B * 16 + B * 4 + B / 8 + BKT_OVF_CAP * 8 + 16;
}
__device__ __forceinline__ Buckets bucket_view(unsigned char* p, uint32_t bb, uint32_t bbmax) {
  const size_t B = size_t(1) << bbmax;
  Buckets T;
  T.keys = reinterpret_cast<uint4*>(p);
  T.cnt = reinterpret_cast<uint32_t*>(p + B * 16);
  T.flag = reinterpret_cast<uint32_t*>(p + B * 20);
  T.ovf = reinterpret_cast<uint2*>(p + B * 20 + B / 8);
  T.ovf_n = reinterpret_cast<uint32_t*>(p + B * 20 + B / 8 + BKT_OVF_CAP * 8);
  T.bb = bb;
  T.mul = BKT_HASH;
  T.ovf_mode = false;
  return T;
}
// all threads of the CTA: EMPTY slots, zero counts and flags
__device__ __forceinline__ void bucket_clear(const Buckets& T, uint32_t t, uint32_t nt) {
  const uint32_t B = 1u << T.bb;
  for (uint32_t b = t; b < B; b += nt) {
    T.keys[b] = make_uint4(EMPTY, EMPTY, EMPTY, EMPTY);
    T.cnt[b] = 0;
  }
  for (uint32_t b = t; b < B / 32; b += nt) T.flag[b] = 0;
  if (t == 0) *T.ovf_n = 0;
}
// Inserts key with local index i.  Returns false if its bucket already
// holds four keys: in strict mode (ovf_mode off) the caller retries the
// whole table with another multiplier; in overflow mode the key goes to the
// overflow list (false only when that list is full too).
__device__ __forceinline__ bool bucket_insert(const Buckets& T, uint32_t key, uint32_t i) {
  const uint32_t h = key * T.mul;
  const uint32_t b = h >> (32 - T.bb);
  const uint32_t s = atomicAdd(&T.cnt[b], 1u);
  if (s < 4) {
    reinterpret_cast<uint32_t*>(T.keys)[4 * b + s] = (h << T.bb) | i;
    return true;
  }
  if (!T.ovf_mode) return false;
  atomicOr(&T.flag[b >> 5], 1u << (b & 31));
  const uint32_t o = atomicAdd(T.ovf_n, 1u);
  if (o >= BKT_OVF_CAP) return false;
  T.ovf[o] = make_uint2(key, i);
  return true;
}
// The local index of y, or B-1 (miss).  Warp-synchronous in overflow mode.
__device__ __forceinline__ uint32_t bucket_find(const Buckets& T, uint32_t y, bool valid) {
  const uint32_t B = 1u << T.bb;
  const uint32_t h = y * T.mul;
  const uint32_t b = h >> (32 - T.bb);
  const uint32_t t = h << T.bb;
  const uint4 q = T.keys[b];
  uint32_t j = min(min(q.x - t, q.y - t), min(q.z - t, q.w - t));
  j = valid ? min(j, B - 1) : B - 1;
  if (T.ovf_mode) {
    const bool full_miss = j == B - 1 && valid && q.w != EMPTY;
    if (__any_sync(FULL, full_miss)) {
      if (full_miss && ((T.flag[b >> 5] >> (b & 31)) & 1u)) {
        const uint32_t no = min(*T.ovf_n, BKT_OVF_CAP);
        for (uint32_t o = 0; o < no; o++) {
          const uint2 e = T.ovf[o];
          if (e.x == y) j = e.y;
        }
      }
    }
  }
  return j;
}

// The stored index of y, or a value >= B-1 (miss); y = EMPTY always misses
// (the hash is a bijection and EMPTY is no vertex id).  Warp-synchronous in
// overflow mode.
template <bool OVF>
__device__ __forceinline__ uint32_t bucket_probe(const Buckets& T, uint32_t y) {
  const uint32_t h = y * T.mul;
  const uint32_t b = h >> (32 - T.bb);
  const uint32_t t = h << T.bb;
  uint32_t j = 0xffffffffu;
#if KCG_FILTER
  // one filter word per bucket (bucket_filter): bit = the top five tag bits.
  // A scattered LDS.32 costs ~3.4 wavefronts per warp against ~8.7 for the
  // scattered LDS.128 of the buckets, which only the few filter-positive
  // lanes now issue -- the staging loops run at 86-99 % of the LSU
  // wavefront peak (profiles/r02_notes.md).
  const bool maybe = (T.cnt[b] >> (t >> 27)) & 1u;
#else
  const bool maybe = true;
#endif
  uint4 q = make_uint4(EMPTY, EMPTY, EMPTY, EMPTY);
  if (maybe) {
    q = T.keys[b];
    j = min(min(q.x - t, q.y - t), min(q.z - t, q.w - t));
  }
  if constexpr (OVF) {
    const uint32_t B = 1u << T.bb;
    const bool full_miss = maybe && j >= B - 1 && y != EMPTY && q.w != EMPTY;
    if (__any_sync(FULL, full_miss)) {
      if (full_miss && ((T.flag[b >> 5] >> (b & 31)) & 1u)) {
        const uint32_t no = min(*T.ovf_n, BKT_OVF_CAP);
        for (uint32_t o = 0; o < no; o++) {
          const uint2 e = T.ovf[o];
          if (e.x == y) j = e.y;
        }
      }
    }
  }
  return j;
}

// After the inserts (and a barrier): the insert counts become the buckets'
// filter words, one bit per key at the top five bits of its slot (the tag
// bits right below the bucket index); overflowed buckets pass everything.
// The caller synchronises afterwards.
__device__ __forceinline__ void bucket_filter(const Buckets& T, uint32_t t, uint32_t nt) {
  const uint32_t B = 1u << T.bb;
  for (uint32_t b = t; b < B; b += nt) {
    const uint4 q = T.keys[b];
    uint32_t w = 0;
    if (q.x != EMPTY) w |= 1u << (q.x >> 27);
    if (q.y != EMPTY) w |= 1u << (q.y >> 27);
    if (q.z != EMPTY) w |= 1u << (q.z >> 27);
    if (q.w != EMPTY) w |= 1u << (q.w >> 27);
    if (T.ovf_mode && ((T.flag[b >> 5] >> (b & 31)) & 1u)) w = 0xffffffffu;
    T.cnt[b] = w;
  }
}

// Builds the table for the d keys adj[0..d) (all threads of the CTA; ends
// with a barrier).  Strict multipliers first, then overflow mode.
// FLAGPOS: the stored index of key i is flag_pos(i) (stage_scan's tables).
template <bool FLAGPOS = false>
__device__ __forceinline__ void bucket_build(Buckets& T, const uint32_t* __restrict__ keys,
                                             uint32_t d, uint32_t t, uint32_t nt) {
  for (uint32_t attempt = 0;; attempt++) {
    if (attempt) {
      T.mul = BKT_HASH + 2u * 0x632BE5ABu * attempt;
      T.ovf_mode = attempt >= BKT_TRIES;
      bucket_clear(T, t, nt);
      __syncthreads();
    }
    bool ok = true;
    for (uint32_t i = t; i < d; i += nt)
      ok &= bucket_insert(T, keys[i], FLAGPOS ? flag_pos(i) : i);
    if (__syncthreads_and(ok)) break;
  }
#if KCG_FILTER
  bucket_filter(T, t, nt);
  __syncthreads();
#endif
}

// 128 entries (or the `rem` < 128 left, EMPTY beyond) at s -> z
__device__ __forceinline__ void stage_load(const uint32_t* __restrict__ s, uint32_t rem,
                                           uint32_t lane, uint32_t (&z)[STAGE_U]) {
  static_assert(STAGE_U == 4, "chunk = 128 entries");
  if (rem >= 128) {
#pragma unroll
    for (int v = 0; v < 4; v++) z[v] = __ldg(s + 32 * v + lane);
  } else {
#pragma unroll
    for (int v = 0; v < 4; v++) z[v] = 32 * v + lane < rem ? __ldg(s + 32 * v + lane) : EMPTY;
  }
}

struct StageRow {
  uint32_t i, len;      // bitmap row and |N+(w_i)|
  const uint32_t* src;  // N+(w_i)
};

// The scan of a warp's rows.  next(row) hands out the warp's next row (false:
// none left); emit(row) turns the warp's flag row into bitmap words and
// clears it.  Tables built with flag positions as indices (bucket_build<true>).
// The 128 entries after the ones being probed -- the row's next chunk, or the
// next row's first -- are always in flight.  EMPTY is no vertex id, so the
// padding of a partial chunk never hits.
template <bool OVF, class Next, class Emit>
__device__ __forceinline__ void stage_scan(const Buckets& T, uint8_t* fl, uint32_t lane, Next next,
                                           Emit emit) {
  const uint32_t NF = (1u << T.bb) - 1;
  // any non-zero byte marks a hit: NF's low byte is 0x7f or 0xff
  auto probe = [&](uint32_t y) {
    const uint32_t j = bucket_probe<OVF>(T, y);
    if (j < NF) fl[j] = uint8_t(NF);
  };
  StageRow cur{0, 0, nullptr}, nxt{0, 0, nullptr};
  uint32_t y[STAGE_U], yn[STAGE_U];
  if (!next(cur)) return;
  stage_load(cur.src, cur.len, lane, y);
  for (;;) {
    const bool have_next = next(nxt);
    if (!have_next) nxt.len = 0;
    const uint32_t* s = cur.src;
    uint32_t rem = cur.len;
    // full chunks with more of the row behind them
    while (rem > 128) {
      s += 128;
      rem -= 128;
      stage_load(s, rem, lane, yn);
#pragma unroll
      for (int v = 0; v < STAGE_U; v++) probe(y[v]);
#pragma unroll
      for (int v = 0; v < STAGE_U; v++) y[v] = yn[v];
    }
    // the row's last chunk, the next row's first chunk behind it
    stage_load(nxt.src, nxt.len, lane, yn);
    probe(y[0]);
    if (rem > 32) probe(y[1]);
    if (rem > 64) probe(y[2]);
    if (rem > 96) probe(y[3]);
#pragma unroll
    for (int v = 0; v < STAGE_U; v++) y[v] = yn[v];
    __syncwarp();
    emit(cur);
    __syncwarp();
    if (!have_next) return;
    cur = nxt;
  }
}

// Rows r in [0, nr): row rowid[r] = N+(w) at adj[rbase[r] ..+ rlen[r]),
// written as bits above the diagonal (ascending local indices).  `fl` is
// the warp's flag row (flag_row_bytes(W), zero on entry and on exit).
template <bool OVF>
__device__ __forceinline__ void stage_rows_t(const Buckets& T, uint32_t* sym, uint32_t wp,
                                             uint32_t W, const uint32_t* __restrict__ adj,
                                             const ull* rbase, const uint32_t* rlen,
                                             const uint32_t* rowid, uint32_t nr,
                                             unsigned* row_ctr, uint8_t* fl, uint32_t lane) {
  uint32_t* fl32 = reinterpret_cast<uint32_t*>(fl);
  const uint32_t G = (W + 3) >> 2;
  auto next = [&](StageRow& row) {
    uint32_t r = 0;
    if (lane == 0) r = atomicAdd(row_ctr, 1u);
    r = __shfl_sync(FULL, r, 0);
    if (r >= nr) return false;
    row.i = rowid[r];
    row.len = rlen[r];
    row.src = adj + rbase[r];
    return true;
  };
  // flags -> words of row i, four per step (lowest possible hit: i + 1)
  auto emit = [&](const StageRow& row) {
    uint32_t* dst = sym + size_t(row.i) * wp;
    for (uint32_t g = (row.i + 1) >> 7; g < G; g++) {
      const uint32_t x = fl32[32 * g + lane];
      if (x) fl32[32 * g + lane] = 0;
      const uint32_t b0 = __ballot_sync(FULL, x & 0x000000ffu);
      const uint32_t b1 = __ballot_sync(FULL, x & 0x0000ff00u);
      const uint32_t b2 = __ballot_sync(FULL, x & 0x00ff0000u);
      const uint32_t b3 = __ballot_sync(FULL, x & 0xff000000u);
      if (lane == 0) *reinterpret_cast<uint4*>(dst + 4 * g) = make_uint4(b0, b1, b2, b3);
    }
  };
  stage_scan<OVF>(T, fl, lane, next, emit);
}
__device__ __forceinline__ void stage_rows(const Buckets& T, uint32_t* sym, uint32_t wp,
                                           uint32_t W, const uint32_t* __restrict__ adj,
                                           const ull* rbase, const uint32_t* rlen,
                                           const uint32_t* rowid, uint32_t nr,
                                           unsigned* row_ctr, uint8_t* fl, uint32_t lane) {
  if (T.ovf_mode)
    stage_rows_t<true>(T, sym, wp, W, adj, rbase, rlen, rowid, nr, row_ctr, fl, lane);
  else
    stage_rows_t<false>(T, sym, wp, W, adj, rbase, rlen, rowid, nr, row_ctr, fl, lane);
}

// Heavy tier (d > 1024, the bitmap in global memory): the same row walk
// with one atomic per hit (SYM: also the mirrored bit).
template <bool SYM>
__device__ __forceinline__ void stage_rows_atomic(const Buckets& T, uint32_t* sym, uint32_t wp,
                                                  const uint32_t* __restrict__ adj,
                                                  const ull* rbase, const uint32_t* rlen,
                                                  const uint32_t* rowid, uint32_t nr,
                                                  unsigned* row_ctr, uint32_t lane) {
  const uint32_t NF = (1u << T.bb) - 1;
  for (;;) {
    uint32_t r = 0;
    if (lane == 0) r = atomicAdd(row_ctr, 1u);
    r = __shfl_sync(FULL, r, 0);
    if (r >= nr) break;
    const uint32_t i = rowid[r], len = rlen[r];
    const uint32_t* src = adj + rbase[r];
    uint32_t* dst = sym + size_t(i) * wp;
    for (uint32_t p0 = 0; p0 < len; p0 += 32 * STAGE_U) {
      uint32_t y[STAGE_U];
#pragma unroll
      for (int u = 0; u < STAGE_U; u++) {
        const uint32_t p = p0 + 32 * u + lane;
        y[u] = p < len ? __ldg(src + p) : EMPTY;
      }
#pragma unroll
      for (int u = 0; u < STAGE_U; u++) {
        const uint32_t j = bucket_find(T, y[u], p0 + 32 * u + lane < len);
        if (j != NF) {
          atomicOr(dst + (j >> 5), 1u << (j & 31));
          if constexpr (SYM) atomicOr(sym + size_t(j) * wp + (i >> 5), 1u << (i & 31));
        }
      }
    }
  }
}

// Fills the lower triangle of a bitmap whose upper triangle is staged
// (per-vertex paths read symmetric rows): 32x32 blocks (I, J), I <= J, are
// transposed with 32 ballots by one warp each.
__device__ __forceinline__ void mirror_lower(uint32_t* sym, uint32_t wp, uint32_t d, uint32_t W,
                                             uint32_t warp, uint32_t nwarps, uint32_t lane) {
  const uint32_t nblk = W * (W + 1) / 2;
  for (uint32_t blk = warp; blk < nblk; blk += nwarps) {
    // blk -> (I, J) with I <= J, row-major over the upper triangle
    uint32_t I = 0, rem = blk;
    while (rem >= W - I) {
      rem -= W - I;
      I++;
    }
    const uint32_t J = I + rem;
    const uint32_t r = 32 * I + lane;
    const uint32_t up = r < d ? sym[size_t(r) * wp + J] : 0u;
    uint32_t mine = 0;
#pragma unroll 8
    for (uint32_t c = 0; c < 32; c++) {
      const uint32_t bal = __ballot_sync(FULL, (up >> c) & 1u);
      if (lane == c) mine = bal;
    }
    // lane c: row 32J + c, word I (its bits are the rows 32I + l with bit
    // (32J + c) set)
    const uint32_t rc = 32 * J + lane;
    if (rc < d) {
      if (I == J)
        sym[size_t(rc) * wp + I] = up | mine;
      else
        sym[size_t(rc) * wp + I] = mine;
    }
  }
}

}  // namespace
}  // namespace kcg
