// k = 4 totals for heavy sources (1024 < d < 4096): included by kcg_count.cu.
//
// The induced bitmap of such a source (d rows of ceil(d/32) words, up to
// 1.5 MB) does not fit one SM's shared memory, and distributed shared memory
// is no answer on this part: a remote SM's shared memory delivers ~20
// B/clk, less than the L2 does (~66 B/clk per SM, profiles/r02_peaks.json).
// So the bitmap lives in a per-CTA slice of global memory (L2) and the
// triangle count of the induced DAG,
//     sum over induced edges (i, x) of |N+(i) ∩ N+(x)|      (counting.cpp:115-123,
//                                                            clique_rec.hpp:49-60),
// is tiled like a matrix product: column block X (128 columns = one 16-byte
// quad per row) keeps the rows x of that block resident in shared memory
// (quads from X's own on: rows hold only bits above their index, so nothing
// left of the block can count), row blocks I <= X stream through a second
// tile, and every (I, X) pair of tiles is read from L2 once instead of once
// per induced edge (config 5: 8.1 TB of L2 traffic in round 1's heavy
// launch, 3.97x the algorithmic bytes).
//
// Inside a pair of tiles a warp takes whole rows i: the members x of row i
// inside block X are the bits of the row's first quad; they go through a
// 64-entry (i, x) queue that persists across rows, so every dot-product
// step runs on 32 edges: row i is a multicast load (a batch spans few
// rows) and the rows x are consecutive members of one row, which the odd
// quad stride spreads over the bank groups.
//
// Staging is the shared-memory tiers' (kcg_stage.cuh: bucketed membership
// table, byte flags, ballots) with whole rows written to the slice --
// coalesced, no atomics, no memset -- and the next row's descriptor
// (target, offsets) loaded while the current row is probed.
#pragma once

namespace kcg {
namespace {

constexpr uint32_t HV_TB = 128;     // rows per tile = columns per quad
constexpr uint32_t HV_DMAX = 4095;  // largest out-degree the tiled kernel takes

struct HeavyArgs {
  const uint64_t* off;
  const uint32_t* adj;
  const uint32_t* item_src;
  uint32_t nitems;
  ull* total;
  ull* staged;
  unsigned* work;
  uint32_t* gbase;     // per-CTA bitmap slices
  size_t slice_words;  // words per slice
  uint32_t bbmax;      // bucket bits of the launch's largest source
  uint32_t qs;         // tile row stride in quads (odd)
  uint32_t flag_stride;  // bytes per warp flag row
  uint32_t off_flags, off_tile_x, off_tile_i, off_queue;  // dynamic smem offsets
  uint32_t off_pvl;    // per-vertex: u32 credits of the source's d local vertices
  uint32_t smem_bytes;
  int nthreads;        // CTA size the plan was made for
  ull* pv_rank;        // per-vertex: global counts (rank space)
};

// dynamic shared memory plan for sources of out-degree <= dmax, NW warps
inline HeavyArgs heavy_plan(uint32_t dmax, int nw, bool pv = false) {
  HeavyArgs a{};
  a.bbmax = bucket_bits(dmax);
  const uint32_t W = (dmax + 31) / 32, Q = (W + 3) / 4;
  a.qs = Q | 1u;
  a.flag_stride = uint32_t(flag_row_bytes(W));
  a.slice_words = size_t(dmax) * 4 * Q;
  // phase A: membership table + flag rows; phase B: two tiles + queues
  const size_t tb = align_up(bucket_bytes(dmax), 16);
  const size_t phase_a = tb + size_t(a.flag_stride) * nw;
  const size_t tile = size_t(HV_TB) * a.qs * 16;
  a.off_flags = uint32_t(tb);
  a.off_tile_x = 0;
  a.off_tile_i = uint32_t(tile);
  a.off_queue = uint32_t(2 * tile);
  const size_t phase_b = 2 * tile + size_t(nw) * 64 * 4;
  // per-vertex credits live through both phases (a source's credit per local
  // vertex is at most C(d-1, 2) < 2^32)
  a.off_pvl = uint32_t(align_up(std::max(phase_a, phase_b), 16));
  a.smem_bytes = uint32_t(align_up(a.off_pvl + (pv ? size_t(dmax) * 4 : 0), 128));
  return a;
}

// rows [row0, row0 + nrows) of the slice, quads [q0, q0 + qt) -> tile rows
// of stride qs quads (all threads of the CTA; no barrier)
// UPPER: the rows are symmetric and q0 is the quad of their own diagonal
// block: bits at or below the row's index are cleared (they sit in the first
// quad loaded).
template <int NT, bool UPPER = false>
__device__ __forceinline__ void heavy_load_tile(uint4* tile, const uint32_t* sym, uint32_t wp,
                                                uint32_t row0, uint32_t nrows, uint32_t q0,
                                                uint32_t qt, uint32_t qs) {
  const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const uint32_t rpp = qt >= 32 ? 1u : 32u / qt;  // rows per warp pass
  const uint32_t sub = lane / qt, q = lane - sub * qt;
  if (sub >= rpp) return;
  for (uint32_t r = wib * rpp + sub; r < nrows; r += (NT / 32) * rpp) {
    const uint4* src = reinterpret_cast<const uint4*>(sym + size_t(row0 + r) * wp) + q0;
    for (uint32_t c = q; c < qt; c += 32) {
      uint4 v = __ldcg(src + c);
      if (UPPER && c == 0) {
        const uint32_t wr = r >> 5, m = above_mask(r & 31);
        v.x = wr > 0 ? 0u : wr == 0 ? v.x & m : v.x;
        v.y = wr > 1 ? 0u : wr == 1 ? v.y & m : v.y;
        v.z = wr > 2 ? 0u : wr == 2 ? v.z & m : v.z;
        v.w = wr == 3 ? v.w & m : v.w;
      }
      tile[r * qs + c] = v;
    }
  }
}

template <int NT, int MB, bool PV = false>
__global__ void __launch_bounds__(NT, MB) count_heavy4_kernel(HeavyArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ unsigned s_src, s_row;
  const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const uint32_t lt = (1u << lane) - 1u;
  uint32_t* sym = a.gbase + size_t(blockIdx.x) * a.slice_words;
  uint8_t* fl = smem + a.off_flags + size_t(wib) * a.flag_stride;
  uint4* tile_x = reinterpret_cast<uint4*>(smem + a.off_tile_x);
  uint4* tile_i = reinterpret_cast<uint4*>(smem + a.off_tile_i);
  uint32_t* queue = reinterpret_cast<uint32_t*>(smem + a.off_queue) + wib * 64;
  uint32_t* pvl = reinterpret_cast<uint32_t*>(smem + a.off_pvl);
  const uint32_t qs = a.qs;
  ull my_total = 0, my_staged = 0;
  auto grab = [&]() {
    uint32_t r = 0;
    if (lane == 0) r = atomicAdd(&s_row, 1u);
    return __shfl_sync(FULL, r, 0);
  };
  for (;;) {
    if (threadIdx.x == 0) {
      s_src = atomicAdd(a.work, 1u);
      s_row = 0;
    }
    __syncthreads();
    const uint32_t si = s_src;
    if (si >= a.nitems) break;
    const uint32_t u = a.item_src[si];
    const uint64_t b = a.off[u];
    const uint32_t d = uint32_t(a.off[u + 1] - b);
    const uint32_t W = (d + 31) / 32, Q = (W + 3) / 4, wp = 4 * Q;
    Buckets T = bucket_view(smem, bucket_bits(d), a.bbmax);
    bucket_clear(T, threadIdx.x, NT);
    if constexpr (PV) {
      for (uint32_t i = threadIdx.x; i < d; i += NT) pvl[i] = 0;
    }
    for (uint32_t i = 4 * lane; i < a.flag_stride; i += 128)
      *reinterpret_cast<uint32_t*>(fl + i) = 0;  // the tiles of the last source lay here
    __syncthreads();
    bucket_build<true>(T, a.adj + b, d, threadIdx.x, NT);
    // ---- staging: warps take whole rows; row d-1 has nothing above it
    {
      uint32_t* fl32 = reinterpret_cast<uint32_t*>(fl);
      // the descriptor loads of a row are in flight while the row before it
      // is probed (stage_scan asks one row ahead)
      auto next = [&](StageRow& row) {
        const uint32_t r = grab();
        if (r >= d) return false;
        row.i = r;
        row.len = 0;
        row.src = a.adj;
        if (r + 1 < d) {
          const uint32_t w = __ldg(a.adj + b + r);
          const uint64_t rb = __ldg(a.off + w);
          row.len = uint32_t(__ldg(a.off + w + 1) - rb);
          row.src = a.adj + rb;
        }
        return true;
      };
      // flags -> the whole row (zero left of the diagonal), 32 words per store
      auto emit = [&](const StageRow& row) {
        if (lane == 0) my_staged += row.len;
        const uint32_t g_lo = (row.i + 1) >> 7;
        uint32_t* dst = sym + size_t(row.i) * wp;
        for (uint32_t w0 = 0; w0 < wp; w0 += 32) {
          uint32_t mine = 0;
          const uint32_t gend = min(w0 / 4 + 8, Q);
          for (uint32_t g = max(w0 / 4, g_lo); g < gend && row.len; g++) {
            const uint32_t x = fl32[32 * g + lane];
            if (x) fl32[32 * g + lane] = 0;
            const uint32_t b0 = __ballot_sync(FULL, x & 0x000000ffu);
            const uint32_t b1 = __ballot_sync(FULL, x & 0x0000ff00u);
            const uint32_t b2 = __ballot_sync(FULL, x & 0x00ff0000u);
            const uint32_t b3 = __ballot_sync(FULL, x & 0xff000000u);
            const uint32_t k = lane - ((4 * g) & 31u);
            if (k < 4) mine = k == 0 ? b0 : k == 1 ? b1 : k == 2 ? b2 : b3;
          }
          if (w0 + lane < wp) dst[w0 + lane] = mine;
        }
      };
      if (T.ovf_mode)
        stage_scan<true>(T, fl, lane, next, emit);
      else
        stage_scan<false>(T, fl, lane, next, emit);
    }
    __syncthreads();  // the slice's rows are visible to the whole CTA
    if constexpr (PV) {
      // ---- per-vertex: symmetric rows.  Edge (i, x), i < x, credits x with
      // all = |N+(i) ∩ N(x)| over the columns above i -- x as the middle
      // vertex of (i, x, y), y > x, and as the top vertex of (i, y, x),
      // i < y < x -- and i with cx, the part above x (clique_rec.hpp:33-36,
      // counting.cpp:191-198).  Row block I stays resident, masked to the bits
      // above each row's index; the symmetric row blocks X >= I stream
      // through the second tile, both from I's own quad on.
      mirror_lower(sym, wp, d, W, wib, NT / 32, lane);
      __syncthreads();
      ull acc = 0;
      uint32_t qn = 0;
      for (uint32_t bi = 0; bi < Q; bi++) {
        const uint32_t qt = Q - bi;
        const uint32_t ni = min(HV_TB, d - HV_TB * bi);
        heavy_load_tile<NT, true>(tile_i, sym, wp, HV_TB * bi, ni, bi, qt, qs);
        for (uint32_t bx = bi; bx < Q; bx++) {
          const uint32_t nx = min(HV_TB, d - HV_TB * bx);
          const uint32_t qx = bx - bi;
          heavy_load_tile<NT>(tile_x, sym, wp, HV_TB * bx, nx, bi, qt, qs);
          if (threadIdx.x == 0) s_row = 0;
          __syncthreads();
          auto run_batch = [&](bool valid) {
            const uint32_t e = valid ? queue[lane] : 0u;
            const uint32_t r = e >> 8, xl = e & 255u;
            const uint4* pi = tile_i + r * qs;
            const uint4* px = tile_x + xl * qs;
            uint32_t lo = 0, hi = 0;
            for (uint32_t q = 0; q < qx; q++) lo += popc_and4(pi[q], px[q]);
            for (uint32_t q = qx + 1; q < qt; q++) hi += popc_and4(pi[q], px[q]);
            // x's own quad: everything counts for `all`, bits above x for cx
            const uint4 va = pi[qx], vb = px[qx];
            const uint32_t m[4] = {va.x & vb.x, va.y & vb.y, va.z & vb.z, va.w & vb.w};
            const uint32_t wx = xl >> 5, mx = above_mask(xl & 31);
            uint32_t mid = 0, midx = 0;
#pragma unroll
            for (uint32_t j = 0; j < 4; j++) {
              mid += __popc(m[j]);
              midx += __popc(j < wx ? 0u : j == wx ? m[j] & mx : m[j]);
            }
            if (valid) {
              const uint32_t all = lo + mid + hi, cx = midx + hi;
              if (all) atomicAdd(&pvl[HV_TB * bx + xl], all);
              if (cx) atomicAdd(&pvl[HV_TB * bi + r], cx);
              acc += cx;
            }
          };
          for (;;) {
            const uint32_t r = grab();
            if (r >= ni) break;
            const uint4 m4 = tile_i[r * qs + qx];
            const uint32_t mw[4] = {m4.x, m4.y, m4.z, m4.w};
#pragma unroll
            for (int j = 0; j < 4; j++) {
              const uint32_t v = mw[j];
              if (v == 0) continue;
              if ((v >> lane) & 1u) queue[qn + __popc(v & lt)] = (r << 8) | (32u * j + lane);
              qn += __popc(v);
              if (qn >= 32) {
                __syncwarp();
                const bool mv = lane + 32 < qn;
                const uint32_t e1 = mv ? queue[lane + 32] : 0u;
                run_batch(true);
                __syncwarp();
                if (mv) queue[lane] = e1;
                qn -= 32;
                __syncwarp();
              }
            }
          }
          __syncwarp();
          if (qn) run_batch(lane < qn);
          qn = 0;
          __syncthreads();
        }
      }
      acc = warp_sum(acc);
      if (lane == 0 && acc) {
        my_total += acc;
        atomicAdd(&a.pv_rank[u], acc);
      }
      // (the last pair's closing barrier ordered every credit before this)
      for (uint32_t i = threadIdx.x; i < d; i += NT)
        if (pvl[i]) atomicAdd(&a.pv_rank[__ldg(a.adj + b + i)], ull(pvl[i]));
      continue;
    }
    // ---- tiled triangle count of the induced DAG
    ull acc = 0;
    uint32_t qn = 0;  // (i, x) queue length, warp-uniform
    for (uint32_t bx = 0; bx < Q; bx++) {
      const uint32_t qt = Q - bx;
      const uint32_t nx = min(HV_TB, d - HV_TB * bx);
      heavy_load_tile<NT>(tile_x, sym, wp, HV_TB * bx, nx, bx, qt, qs);
      // the diagonal pair first: it needs no second tile
      for (uint32_t bi = bx + 1; bi-- > 0;) {
        const uint4* ti = tile_x;
        uint32_t ni = nx;
        if (bi < bx) {
          heavy_load_tile<NT>(tile_i, sym, wp, HV_TB * bi, HV_TB, bx, qt, qs);
          ti = tile_i;
          ni = HV_TB;
        }
        if (threadIdx.x == 0) s_row = 0;
        __syncthreads();
        auto run_batch = [&](bool valid) {
          const uint32_t e = valid ? queue[lane] : 0u;
          const uint4* pi = ti + (e >> 8) * qs;
          const uint4* px = tile_x + (e & 255u) * qs;
          uint32_t c = 0;
          for (uint32_t q = 0; q < qt; q++) c += popc_and4(pi[q], px[q]);
          acc += valid ? c : 0u;
        };
        for (;;) {
          const uint32_t r = grab();
          if (r >= ni) break;
          const uint4 m4 = ti[r * qs];
          const uint32_t mw[4] = {m4.x, m4.y, m4.z, m4.w};
#pragma unroll
          for (int j = 0; j < 4; j++) {
            const uint32_t v = mw[j];
            if (v == 0) continue;
            if ((v >> lane) & 1u) queue[qn + __popc(v & lt)] = (r << 8) | (32u * j + lane);
            qn += __popc(v);
            if (qn >= 32) {
              __syncwarp();
              const bool mv = lane + 32 < qn;
              const uint32_t e1 = mv ? queue[lane + 32] : 0u;
              run_batch(true);
              __syncwarp();
              if (mv) queue[lane] = e1;
              qn -= 32;
              __syncwarp();
            }
          }
        }
        // entries name rows of this pair of tiles: drain before they change
        __syncwarp();
        if (qn) run_batch(lane < qn);
        qn = 0;
        __syncthreads();
      }
    }
    acc = warp_sum(acc);
    if (lane == 0) my_total += acc;
  }
  if (lane == 0) {
    if (my_total) atomicAdd(a.total, my_total);
    if (my_staged) atomicAdd(a.staged, my_staged);
  }
}

}  // namespace
}  // namespace kcg
