// k-clique listing on the device: list_cliques of
// proj/src/counting.cpp:214-217, which reports every clique once with its
// vertices in ascending rank (test_counting.cpp:110-123).
//
// One warp per source rank r walks the reference's recursion
// (clique_rec.hpp:24-62) over the rank-relabelled DAG: the candidate set
// of a level is the previous level's remaining candidates intersected with
// N+(x), computed 32 candidates at a time (each lane binary-searches its
// candidate in the sorted slice of x) and compacted in order with a ballot;
// sets live in a per-warp slice of global memory, the first level is the
// DAG slice itself.  At the last level every candidate completes a clique;
// the warp reserves output slots with one atomic and each lane writes its
// clique as vertex ids.
//
// Output can be far larger than memory, so the host lists in chunks of
// source ranks whose clique count -- taken with the source-masked counting
// kernels -- fits the batch, and hands each batch to the caller.
#include <algorithm>
#include <vector>

#include "kcg_internal.cuh"

namespace kcg {
namespace {

typedef unsigned long long ull;
constexpr unsigned FULLW = 0xffffffffu;
constexpr int LIST_MAXK = 34;

__device__ __forceinline__ bool in_sorted(const uint32_t* __restrict__ a, uint32_t len,
                                          uint32_t key) {
  uint32_t lo = 0, hi = len;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    const uint32_t v = a[mid];
    if (v < key)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo < len && a[lo] == key;
}

__global__ void __launch_bounds__(256)
    list_kernel(const uint64_t* __restrict__ off, const uint32_t* __restrict__ adj,
                const uint32_t* __restrict__ order, uint32_t r0, uint32_t r1, int k,
                uint32_t* __restrict__ scratch, uint32_t maxd, uint32_t* __restrict__ out,
                ull cap, ull* __restrict__ cursor) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warp = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  uint32_t* ws = scratch + warp * uint64_t(k) * maxd;
  const uint32_t* set[LIST_MAXK];
  uint32_t len[LIST_MAXK], pos[LIST_MAXK], chain[LIST_MAXK];
  for (uint64_t rr = r0 + warp; rr < r1; rr += nwarps) {
    const uint32_t r = uint32_t(rr);
    const uint64_t b = off[r];
    const uint32_t d = uint32_t(off[r + 1] - b);
    if (d + 1 < uint32_t(k)) continue;
    chain[0] = r;
    int l = 1;
    set[1] = adj + b;
    len[1] = d;
    pos[1] = 0;
    // emits chain[0..l] + each element of s[0..n)
    auto emit = [&](const uint32_t* s, uint32_t n, int depth) {
      for (uint32_t c0 = 0; c0 < n; c0 += 32) {
        const uint32_t cnt = min(32u, n - c0);
        ull base = 0;
        if (lane == 0) base = atomicAdd(cursor, ull(cnt));
        base = __shfl_sync(FULLW, base, 0);
        if (lane < cnt && base + lane < cap) {
          uint32_t* o = out + (base + lane) * uint64_t(k);
          for (int j = 0; j <= depth; j++) o[j] = order[chain[j]];
          o[depth + 1] = order[s[c0 + lane]];
        }
      }
    };
    if (k == 2) {
      emit(set[1], d, 0);
      continue;
    }
    for (;;) {
      if (len[l] - pos[l] < uint32_t(k - l)) {  // too few candidates left
        if (l == 1) break;
        l--;
        continue;
      }
      const uint32_t x = set[l][pos[l]];
      pos[l]++;
      chain[l] = x;
      // child = remaining candidates of level l that are out-neighbours of x
      const uint32_t* nx = adj + off[x];
      const uint32_t dx = uint32_t(off[x + 1] - off[x]);
      uint32_t* child = ws + uint64_t(l + 1) * maxd;
      uint32_t clen = 0;
      for (uint32_t c0 = pos[l]; c0 < len[l]; c0 += 32) {
        const uint32_t p = c0 + lane;
        bool keep = false;
        uint32_t e = 0;
        if (p < len[l]) {
          e = set[l][p];
          keep = in_sorted(nx, dx, e);
        }
        const unsigned bal = __ballot_sync(FULLW, keep);
        if (keep) child[clen + __popc(bal & ((1u << lane) - 1u))] = e;
        clen += __popc(bal);
      }
      __syncwarp();
      if (l + 2 == k) {
        emit(child, clen, l);  // chain[0..l] + one more vertex
        __syncwarp();
      } else if (clen >= uint32_t(k - l - 1)) {
        l++;
        set[l] = child;
        len[l] = clen;
        pos[l] = 0;
      }
    }
  }
}

__global__ void range_mask_kernel(uint32_t n, uint32_t r0, uint32_t r1, uint8_t* __restrict__ m) {
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x)
    m[r] = r >= r0 && r < r1;
}

}  // namespace

uint64_t list_cliques(Graph& g, int k, uint64_t batch, kcg_clique_fn fn, void* user) {
  if (k < 2) fail(KCG_EINVAL, "k must be at least 2");
  if (!g.has_rdag) {
    if (!g.has_rank) fail(KCG_EINVAL, "no DAG: call kcg_rank/kcg_direct first");
    build_dag(g, false);
  }
  if (batch == 0) batch = uint64_t(1) << 24;
  const uint32_t n = g.n;
  const uint64_t total = count_cliques(g, k, false);
  if (total == 0 || n == 0) return total;
  // any k is listed when there is nothing to list (the reference's
  // recursion simply finds no clique); a graph that does hold a clique of
  // 34+ vertices needs a deeper device stack than the listing kernel keeps
  if (k > LIST_MAXK - 1)
    fail(KCG_EINVAL, "list_cliques: the graph has " + std::to_string(total) + " " +
                         std::to_string(k) + "-cliques; device listing supports k <= 33");
  // per-range clique counts with the source-masked counter
  DevBuf<uint8_t> mask;
  mask.ensure(n, &g.alloc);
  auto range_count = [&](uint32_t a, uint32_t b) {
    range_mask_kernel<<<blocks_for(n, 256), 256, 0, g.stream>>>(n, a, b, mask.p);
    KCG_LAUNCHED(g);
    g.src_mask = mask.p;
    uint64_t c = 0;
    try {
      c = count_cliques(g, k, false);
    } catch (...) {
      g.src_mask = nullptr;
      throw;
    }
    g.src_mask = nullptr;
    return c;
  };
  // chunks [a, b) with count <= batch (a single rank may exceed it; it is
  // then listed alone with a buffer of its own size)
  std::vector<std::pair<std::pair<uint32_t, uint32_t>, uint64_t>> chunks;
  std::vector<std::pair<std::pair<uint32_t, uint32_t>, uint64_t>> todo = {{{0u, n}, total}};
  while (!todo.empty()) {
    auto [rg, c] = todo.back();
    todo.pop_back();
    if (c == 0) continue;
    if (c <= batch || rg.second - rg.first == 1) {
      chunks.push_back({rg, c});
      continue;
    }
    const uint32_t mid = rg.first + (rg.second - rg.first) / 2;
    const uint64_t cl = range_count(rg.first, mid);
    todo.push_back({{mid, rg.second}, c - cl});
    todo.push_back({{rg.first, mid}, cl});
  }
  std::sort(chunks.begin(), chunks.end());
  uint64_t maxc = 0;
  for (auto& ch : chunks) maxc = std::max(maxc, ch.second);
  const Device& dev = device();
  const uint32_t maxd = uint32_t(std::max<uint64_t>(g.max_out, 1));
  const unsigned grid = dev.sms * 8u;
  const uint64_t nwarps = uint64_t(grid) * 256 / 32;
  DevBuf<uint32_t> scratch, out;
  scratch.ensure(nwarps * uint64_t(k) * maxd, &g.alloc);
  out.ensure(maxc * uint64_t(k), &g.alloc);
  ull* cursor = reinterpret_cast<ull*>(g.counters.ensure(16, &g.alloc)) + 9;
  std::vector<uint32_t> host;
  uint64_t listed = 0;
  for (auto& ch : chunks) {
    KCG_CUDA(cudaMemsetAsync(cursor, 0, 8, g.stream));
    list_kernel<<<grid, 256, 0, g.stream>>>(g.rdag_off.p, g.rdag_adj.p, g.order.p, ch.first.first,
                                            ch.first.second, k, scratch.p, maxd, out.p, ch.second,
                                            cursor);
    KCG_LAUNCHED(g);
    ull got = 0;
    KCG_CUDA(cudaMemcpyAsync(&got, cursor, 8, cudaMemcpyDeviceToHost, g.stream));
    g.sync();
    if (got != ch.second) fail(KCG_ERUNTIME, "list_cliques: listing disagrees with the count");
    host.resize(got * uint64_t(k));
    KCG_CUDA(cudaMemcpyAsync(host.data(), out.p, host.size() * 4, cudaMemcpyDeviceToHost,
                             g.stream));
    g.sync();
    g.times.d2h_bytes += host.size() * 4;
    listed += got;
    if (fn && fn(host.data(), got, k, user) != 0) fail(KCG_ERUNTIME, "list_cliques: callback abort");
  }
  if (listed != total) fail(KCG_ERUNTIME, "list_cliques: listing disagrees with the count");
  return total;
}

}  // namespace kcg
