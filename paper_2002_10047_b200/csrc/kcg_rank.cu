// Ranking / orientation-order kernels (K1-K4 of SURVEY.md §2.3).
//
// Bulk-synchronous rounds with the whole graph in HBM.  Thresholds are
// evaluated on the host in IEEE double with exactly the reference's
// expressions and compared against (double)degree on the device, so BE
// and the arboricity estimate are bit-exact without any FMA concerns.
// Within a round the rank order is the id order, produced by an ordered
// exclusive scan over the id-sorted remaining list (never by atomic
// arrival order).
#include <cooperative_groups.h>
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <thrust/iterator/transform_iterator.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "kcg_internal.cuh"

namespace kcg {
namespace {

constexpr int kThreads = 256;

__global__ void iota_kernel(uint32_t* __restrict__ a, uint32_t n) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    a[i] = i;
}

__global__ void scatter_rank_kernel(const uint32_t* __restrict__ order, uint32_t n,
                                    uint32_t base, uint32_t* __restrict__ rank) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    rank[order[i]] = base + i;
}

// flag functors over the remaining list
struct LessThan {  // rank_barenboim_elkin: double(deg) < threshold
  const uint32_t* rem;
  const uint32_t* deg;
  double thr;
  __device__ uint32_t operator()(uint32_t i) const {
    return double(deg[rem[i]]) < thr ? 1u : 0u;
  }
};
struct AtMost {  // estimate_arboricity: double(deg) <= cutoff
  const uint32_t* rem;
  const uint32_t* deg;
  double thr;
  __device__ uint32_t operator()(uint32_t i) const {
    return double(deg[rem[i]]) <= thr ? 1u : 0u;
  }
};

template <class Flag>
__global__ void split_kernel(Flag flag, const uint32_t* __restrict__ rem, uint32_t nrem,
                             const uint32_t* __restrict__ pos, uint32_t* __restrict__ batch,
                             uint32_t* __restrict__ keep, uint8_t* __restrict__ alive,
                             uint8_t mark, uint32_t* __restrict__ rank, uint32_t placed) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nrem;
       i += gridDim.x * blockDim.x) {
    uint32_t v = rem[i];
    uint32_t p = pos[i];
    if (flag(i)) {
      batch[p] = v;
      alive[v] = mark;
      if (rank) rank[v] = placed + p;
    } else {
      keep[i - p] = v;
    }
  }
}

__global__ void invert_kernel(const uint32_t* __restrict__ rank, uint32_t n,
                              uint32_t* __restrict__ order) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    order[rank[v]] = v;
}

// Degree decrements for the survivors of a BE / GP round: one warp per
// batch vertex, lanes stride its adjacency.  Hubs (degree > kHubDeg) are
// only listed here and spread over the whole grid by decrement_hub_kernel
// (one warp walking a 50k-entry slice was the tail of the round).
constexpr uint64_t kHubDeg = 2048;

__global__ void decrement_kernel(const uint32_t* __restrict__ batch, uint32_t nb,
                                 const uint64_t* __restrict__ off,
                                 const uint32_t* __restrict__ adj,
                                 const uint8_t* __restrict__ alive,
                                 uint32_t* __restrict__ deg, uint32_t* __restrict__ hubs,
                                 unsigned* __restrict__ nhubs) {
  const uint32_t lane = threadIdx.x & 31;
  for (uint64_t w = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; w < nb;
       w += (uint64_t(gridDim.x) * blockDim.x) >> 5) {
    uint32_t v = batch[w];
    const uint64_t b = off[v], e = off[v + 1];
    if (e - b > kHubDeg) {
      if (lane == 0) hubs[atomicAdd(nhubs, 1u)] = v;
      continue;
    }
    for (uint64_t p = b + lane; p < e; p += 32) {
      uint32_t u = adj[p];
      if (alive[u] == 1) atomicSub(&deg[u], 1u);
    }
  }
}

// estimate_arboricity round: alive[] is 1 for survivors, 2 for this
// round's batch.  Reproduces the reference's sequential batch walk
// (orientation.cpp:146-154): an edge to a survivor is removed once, an
// intra-batch edge once (by its lower-id endpoint).
__device__ __forceinline__ void arb_edge(uint32_t v, uint32_t u, const uint8_t* alive,
                                         uint32_t* deg, unsigned long long& mine) {
  const uint8_t a = alive[u];
  if (a == 1) {
    atomicSub(&deg[u], 1u);
    mine++;
  } else if (a == 2 && u > v) {
    mine++;
  }
}

__global__ void arb_decrement_kernel(const uint32_t* __restrict__ batch, uint32_t nb,
                                     const uint64_t* __restrict__ off,
                                     const uint32_t* __restrict__ adj,
                                     const uint8_t* __restrict__ alive,
                                     uint32_t* __restrict__ deg,
                                     unsigned long long* __restrict__ removed,
                                     uint32_t* __restrict__ hubs, unsigned* __restrict__ nhubs) {
  const uint32_t lane = threadIdx.x & 31;
  unsigned long long mine = 0;
  for (uint64_t w = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; w < nb;
       w += (uint64_t(gridDim.x) * blockDim.x) >> 5) {
    uint32_t v = batch[w];
    const uint64_t b = off[v], e = off[v + 1];
    if (e - b > kHubDeg) {
      if (lane == 0) hubs[atomicAdd(nhubs, 1u)] = v;
      continue;
    }
    for (uint64_t p = b + lane; p < e; p += 32) arb_edge(v, adj[p], alive, deg, mine);
  }
  for (int s = 16; s; s >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, s);
  if (lane == 0 && mine) atomicAdd(removed, mine);
}

// The listed hubs: one CTA per hub, four loads in flight per thread.
// ARB: the arboricity-round semantics of arb_decrement_kernel.
template <bool ARB>
__global__ void __launch_bounds__(256)
    decrement_hub_kernel(const uint32_t* __restrict__ hubs, const unsigned* __restrict__ nhubs,
                         const uint64_t* __restrict__ off, const uint32_t* __restrict__ adj,
                         const uint8_t* __restrict__ alive, uint32_t* __restrict__ deg,
                         unsigned long long* __restrict__ removed) {
  const unsigned nh = *nhubs;
  unsigned long long mine = 0;
  for (unsigned h = blockIdx.x; h < nh; h += gridDim.x) {
    const uint32_t v = hubs[h];
    const uint64_t e = off[v + 1];
    for (uint64_t p0 = off[v] + threadIdx.x; p0 < e; p0 += 4 * 256) {
      uint32_t u[4];
#pragma unroll
      for (int j = 0; j < 4; j++) u[j] = p0 + j * 256 < e ? adj[p0 + j * 256] : 0xffffffffu;
#pragma unroll
      for (int j = 0; j < 4; j++) {
        if (u[j] == 0xffffffffu) continue;
        if constexpr (ARB) {
          arb_edge(v, u[j], alive, deg, mine);
        } else {
          if (alive[u[j]] == 1) atomicSub(&deg[u[j]], 1u);
        }
      }
    }
  }
  if constexpr (ARB) {
    for (int s = 16; s; s >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, s);
    if ((threadIdx.x & 31) == 0 && mine) atomicAdd(removed, mine);
  }
}

__global__ void kill_kernel(const uint32_t* __restrict__ batch, uint32_t nb,
                            uint8_t* __restrict__ alive) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nb; i += gridDim.x * blockDim.x)
    alive[batch[i]] = 0;
}

// k-core round: frontier vertices are already dead; a survivor whose
// degree crosses level+1 -> level joins the next frontier exactly once.
__global__ void kcore_decrement_kernel(const uint32_t* __restrict__ front, uint32_t nf,
                                       const uint64_t* __restrict__ off,
                                       const uint32_t* __restrict__ adj,
                                       const uint8_t* __restrict__ alive,
                                       uint32_t* __restrict__ deg, uint32_t level,
                                       uint32_t* __restrict__ next,
                                       unsigned long long* __restrict__ nnext) {
  const uint32_t lane = threadIdx.x & 31;
  for (uint64_t w = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; w < nf;
       w += (uint64_t(gridDim.x) * blockDim.x) >> 5) {
    uint32_t v = front[w];
    for (uint64_t p0 = off[v]; p0 < off[v + 1]; p0 += 32) {
      uint64_t p = p0 + lane;
      bool join = false;
      uint32_t u = 0;
      if (p < off[v + 1]) {
        u = adj[p];
        if (alive[u]) join = atomicSub(&deg[u], 1u) == level + 1;
      }
      // warp-aggregated append to the next frontier
      unsigned ball = __ballot_sync(0xffffffffu, join);
      if (ball) {
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(nnext, (unsigned long long)__popc(ball));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (join) next[base + __popc(ball & ((1u << lane) - 1))] = u;
      }
    }
  }
}

__global__ void kcore_kill_rank_kernel(const uint32_t* __restrict__ front, uint32_t nf,
                                       uint32_t placed, uint8_t* __restrict__ alive,
                                       uint32_t* __restrict__ rank) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nf; i += gridDim.x * blockDim.x) {
    uint32_t v = front[i];
    alive[v] = 0;
    rank[v] = placed + i;
  }
}

struct AliveDeg {  // min-degree reduction over alive remaining vertices
  const uint32_t* rem;
  const uint32_t* deg;
  const uint8_t* alive;
  __device__ uint32_t operator()(uint32_t i) const {
    uint32_t v = rem[i];
    return alive[v] ? deg[v] : 0xffffffffu;
  }
};
struct AliveSel {
  const uint8_t* alive;
  __device__ bool operator()(uint32_t v) const { return alive[v] != 0; }
};
struct AtLevel {
  const uint32_t* rem;
  const uint32_t* deg;
  const uint8_t* alive;
  uint32_t level;
  __device__ bool operator()(uint32_t v) const { return alive[v] && deg[v] <= level; }
};

__global__ void gp_keys_kernel(const uint32_t* __restrict__ rem, uint32_t nrem,
                               const uint32_t* __restrict__ deg, int idbits,
                               uint64_t* __restrict__ keys) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nrem; i += gridDim.x * blockDim.x) {
    uint32_t v = rem[i];
    keys[i] = (uint64_t(deg[v]) << idbits) | v;
  }
}
__global__ void gp_take_kernel(const uint64_t* __restrict__ keys, uint32_t nrem, uint32_t take,
                               uint64_t idmask, uint32_t placed, uint32_t* __restrict__ batch,
                               uint32_t* __restrict__ keep, uint8_t* __restrict__ alive,
                               uint32_t* __restrict__ rank) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nrem; i += gridDim.x * blockDim.x) {
    uint32_t v = uint32_t(keys[i] & idmask);
    if (i < take) {
      batch[i] = v;
      alive[v] = 0;
      rank[v] = placed + i;
    } else {
      keep[i - take] = v;
    }
  }
}

int bits_for(uint64_t x) {
  int b = 0;
  while ((uint64_t(1) << b) <= x && b < 64) b++;
  return b;
}

// Working state for a peeling run, carved from scratch2.
struct Peel {
  uint32_t* wdeg;
  uint8_t* alive;
  uint32_t* rem;
  uint32_t* rem2;
  uint32_t* batch;
  uint32_t* pos;
  uint64_t* keys;
  uint64_t* keys2;
  uint32_t* hubs;
  unsigned long long* ctr;  // [0] removed edges, [4] (as u32) hub count
};

Peel peel_state(Graph& g, bool with_keys) {
  const size_t n = g.n;
  size_t bytes = 0;
  auto carve = [&](size_t b) {
    size_t at = bytes;
    bytes += (b + 255) & ~size_t(255);
    return at;
  };
  size_t o_wdeg = carve(n * 4), o_alive = carve(n), o_rem = carve(n * 4),
         o_rem2 = carve(n * 4), o_batch = carve(n * 4), o_pos = carve(n * 4 + 4),
         o_hubs = carve(n * 4 + 4);
  size_t o_keys = with_keys ? carve(n * 8) : 0, o_keys2 = with_keys ? carve(n * 8) : 0;
  unsigned char* base = g.scratch2.ensure(bytes + 256, &g.alloc);
  Peel p;
  p.wdeg = reinterpret_cast<uint32_t*>(base + o_wdeg);
  p.alive = base + o_alive;
  p.rem = reinterpret_cast<uint32_t*>(base + o_rem);
  p.rem2 = reinterpret_cast<uint32_t*>(base + o_rem2);
  p.batch = reinterpret_cast<uint32_t*>(base + o_batch);
  p.pos = reinterpret_cast<uint32_t*>(base + o_pos);
  p.keys = with_keys ? reinterpret_cast<uint64_t*>(base + o_keys) : nullptr;
  p.keys2 = with_keys ? reinterpret_cast<uint64_t*>(base + o_keys2) : nullptr;
  p.hubs = reinterpret_cast<uint32_t*>(base + o_hubs);
  p.ctr = g.counters.ensure(8, &g.alloc);
  if (n) {
    KCG_CUDA(cudaMemcpyAsync(p.wdeg, g.deg.p, n * 4, cudaMemcpyDeviceToDevice, g.stream));
    KCG_CUDA(cudaMemsetAsync(p.alive, 1, n, g.stream));
    iota_kernel<<<blocks_for(n, kThreads), kThreads, 0, g.stream>>>(p.rem, uint32_t(n));
    KCG_LAUNCHED(g);
  }
  return p;
}

// Survivor degree decrements for batch P.batch[0..nb) (BE / GP rounds).
void decrement(Graph& g, Peel& P, uint32_t nb) {
  unsigned* nh = reinterpret_cast<unsigned*>(P.ctr + 4);
  KCG_CUDA(cudaMemsetAsync(nh, 0, 4, g.stream));
  decrement_kernel<<<blocks_for(uint64_t(nb) * 32, kThreads), kThreads, 0, g.stream>>>(
      P.batch, nb, g.und_off.p, g.und_adj.p, P.alive, P.wdeg, P.hubs, nh);
  KCG_LAUNCHED(g);
  decrement_hub_kernel<false><<<148 * 4, kThreads, 0, g.stream>>>(
      P.hubs, nh, g.und_off.p, g.und_adj.p, P.alive, P.wdeg, nullptr);
  KCG_LAUNCHED(g);
}

// Ordered flag scan: pos[i] = #flags before i; returns the batch size.
template <class Flag>
uint32_t scan_flags(Graph& g, Flag flag, uint32_t nrem, uint32_t* pos) {
  auto it = thrust::make_transform_iterator(thrust::counting_iterator<uint32_t>(0), flag);
  size_t tb = 0;
  KCG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, it, pos, nrem + 1, g.stream));
  KCG_CUDA(cub::DeviceScan::ExclusiveSum(cub_temp(g, tb), tb, it, pos, nrem + 1, g.stream));
  uint32_t nb = 0;
  KCG_CUDA(cudaMemcpyAsync(&nb, pos + nrem, 4, cudaMemcpyDeviceToHost, g.stream));
  g.sync();
  return nb;
}

// The flag functor is evaluated at index nrem by the scan above (to get
// the total in pos[nrem]); guard it.
template <class F>
struct Guard {
  F f;
  uint32_t nrem;
  __device__ uint32_t operator()(uint32_t i) const { return i < nrem ? f(i) : 0u; }
};

void rank_degree(Graph& g) {
  const uint32_t n = g.n;
  if (!n) return;
  // stable LSD radix sort of ids keyed by degree == std::stable_sort by
  // degree (orientation.cpp:10-17)
  size_t off_vals = (size_t(n) * 4 + 255) & ~size_t(255);
  unsigned char* base = g.scratch2.ensure(off_vals * 3 + 256, &g.alloc);
  uint32_t* vals_in = reinterpret_cast<uint32_t*>(base);
  uint32_t* keys_out = reinterpret_cast<uint32_t*>(base + off_vals);
  uint32_t* maxd = reinterpret_cast<uint32_t*>(base + 2 * off_vals);
  iota_kernel<<<blocks_for(n, kThreads), kThreads, 0, g.stream>>>(vals_in, n);
  KCG_LAUNCHED(g);
  size_t tb = 0;
  KCG_CUDA(cub::DeviceReduce::Max(nullptr, tb, g.deg.p, maxd, n, g.stream));
  KCG_CUDA(cub::DeviceReduce::Max(cub_temp(g, tb), tb, g.deg.p, maxd, n, g.stream));
  uint32_t mx = 0;
  KCG_CUDA(cudaMemcpyAsync(&mx, maxd, 4, cudaMemcpyDeviceToHost, g.stream));
  g.sync();
  int end_bit = std::max(1, bits_for(mx));
  g.order.ensure(n, &g.alloc);
  tb = 0;
  KCG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, g.deg.p, keys_out, vals_in, g.order.p,
                                           n, 0, end_bit, g.stream));
  KCG_CUDA(cub::DeviceRadixSort::SortPairs(cub_temp(g, tb), tb, g.deg.p, keys_out, vals_in,
                                           g.order.p, n, 0, end_bit, g.stream));
  scatter_rank_kernel<<<blocks_for(n, kThreads), kThreads, 0, g.stream>>>(g.order.p, n, 0,
                                                                          g.rank.p);
  KCG_LAUNCHED(g);
}

uint64_t rank_be(Graph& g, double eps, uint64_t alpha_hat) {
  // rank_barenboim_elkin, orientation.cpp:86-122
  if (!(eps > 0)) fail(KCG_EINVAL, "epsilon must be positive");
  if (alpha_hat < 1) fail(KCG_EINVAL, "alpha_hat must be >= 1");
  const uint32_t n = g.n;
  Peel P = peel_state(g, false);
  double threshold = (2 + eps) * double(alpha_hat);
  uint32_t nrem = n, placed = 0;
  uint64_t rounds = 0;
  while (nrem) {
    rounds++;
    Guard<LessThan> flag{LessThan{P.rem, P.wdeg, threshold}, nrem};
    uint32_t nb = scan_flags(g, flag, nrem, P.pos);
    if (nb == 0) {
      threshold *= 2;
      continue;
    }
    split_kernel<<<blocks_for(nrem, kThreads), kThreads, 0, g.stream>>>(
        flag, P.rem, nrem, P.pos, P.batch, P.rem2, P.alive, 0, g.rank.p, placed);
    KCG_LAUNCHED(g);
    decrement(g, P, nb);
    std::swap(P.rem, P.rem2);
    nrem -= nb;
    placed += nb;
  }
  return rounds;
}

uint64_t rank_gp(Graph& g, double eps) {
  // rank_goodrich_pszona, orientation.cpp:48-84
  if (!(eps > 0)) fail(KCG_EINVAL, "epsilon must be positive");
  const uint32_t n = g.n;
  Peel P = peel_state(g, true);
  const int idbits = std::max(1, bits_for(n ? n - 1 : 0));
  const uint64_t idmask = (uint64_t(1) << idbits) - 1;
  uint32_t nrem = n, placed = 0;
  uint64_t rounds = 0;
  while (nrem) {
    rounds++;
    uint64_t take = std::max<uint64_t>(
        1, uint64_t(std::floor(eps * double(nrem) / (2 + eps))));
    take = std::min<uint64_t>(take, nrem);
    gp_keys_kernel<<<blocks_for(nrem, kThreads), kThreads, 0, g.stream>>>(P.rem, nrem, P.wdeg,
                                                                         idbits, P.keys);
    KCG_LAUNCHED(g);
    size_t tb = 0;
    int end_bit = std::min(64, idbits + 32);
    KCG_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, P.keys, P.keys2, nrem, 0, end_bit,
                                            g.stream));
    KCG_CUDA(cub::DeviceRadixSort::SortKeys(cub_temp(g, tb), tb, P.keys, P.keys2, nrem, 0,
                                            end_bit, g.stream));
    gp_take_kernel<<<blocks_for(nrem, kThreads), kThreads, 0, g.stream>>>(
        P.keys2, nrem, uint32_t(take), idmask, placed, P.batch, P.rem2, P.alive, g.rank.p);
    KCG_LAUNCHED(g);
    decrement(g, P, uint32_t(take));
    std::swap(P.rem, P.rem2);
    nrem -= uint32_t(take);
    placed += uint32_t(take);
  }
  g.sync();
  return rounds;
}

// Degeneracy peel in one cooperative kernel: every alive vertex whose
// induced degree is <= level leaves in the same round; level only rises
// when the frontier empties.  Each vertex records its removal round; ranks
// are the (round, id) order, assigned afterwards by one radix sort.  Grid-
// wide syncs replace the per-round host round trips.
struct KcoreArgs {
  const uint64_t* off;
  const uint32_t* adj;
  uint32_t n;
  uint32_t* deg;     // working induced degrees
  uint32_t* rnd;     // removal round, 0xffffffff while alive
  uint32_t* front;   // two frontier buffers of n entries
  unsigned* ctr;     // [0],[1] frontier sizes, [2] min degree, [3] rounds, [4] level
};

__global__ void __launch_bounds__(256) kcore_coop_kernel(KcoreArgs a) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  const uint32_t n = a.n;
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t nthreads = gridDim.x * blockDim.x;
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t gwarp = tid >> 5, nwarps = nthreads >> 5;
  uint32_t level = 0, round = 0, placed = 0, cur = 0;
  uint32_t* fr[2] = {a.front, a.front + n};
  while (placed < n) {
    uint32_t nf = a.ctr[cur];
    if (nf == 0) {
      // level change: min alive degree, then every alive vertex at or below
      if (tid == 0) a.ctr[2] = 0xffffffffu;
      grid.sync();
      uint32_t mn = 0xffffffffu;
      for (uint32_t v = tid; v < n; v += nthreads)
        if (a.rnd[v] == 0xffffffffu) mn = min(mn, a.deg[v]);
      mn = __reduce_min_sync(0xffffffffu, mn);
      if (lane == 0 && mn != 0xffffffffu) atomicMin(&a.ctr[2], mn);
      grid.sync();
      level = max(level, a.ctr[2]);
      for (uint32_t v0 = 0; v0 < n; v0 += nthreads) {
        const uint32_t v = v0 + tid;
        const bool take = v < n && a.rnd[v] == 0xffffffffu && a.deg[v] <= level;
        const unsigned bal = __ballot_sync(0xffffffffu, take);
        uint32_t base = 0;
        if (lane == 0 && bal) base = atomicAdd(&a.ctr[cur], __popc(bal));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (take) fr[cur][base + __popc(bal & ((1u << lane) - 1))] = v;
      }
      grid.sync();
      nf = a.ctr[cur];
    }
    // this round: mark, then decrement survivors and collect the next
    // frontier (a survivor crossing level+1 -> level joins exactly once)
    for (uint32_t i = tid; i < nf; i += nthreads) a.rnd[fr[cur][i]] = round;
    if (tid == 0) a.ctr[cur ^ 1] = 0;
    grid.sync();
    for (uint32_t w = gwarp; w < nf; w += nwarps) {
      const uint32_t v = fr[cur][w];
      const uint64_t e = a.off[v + 1];
      for (uint64_t p0 = a.off[v]; p0 < e; p0 += 32) {
        const uint64_t p = p0 + lane;
        bool join = false;
        uint32_t u = 0;
        if (p < e) {
          u = a.adj[p];
          if (a.rnd[u] == 0xffffffffu) join = atomicSub(&a.deg[u], 1u) == level + 1;
        }
        const unsigned bal = __ballot_sync(0xffffffffu, join);
        if (bal) {
          uint32_t base = 0;
          if (lane == 0) base = atomicAdd(&a.ctr[cur ^ 1], __popc(bal));
          base = __shfl_sync(0xffffffffu, base, 0);
          if (join) fr[cur ^ 1][base + __popc(bal & ((1u << lane) - 1))] = u;
        }
      }
    }
    placed += nf;
    round++;
    if (tid == 0) a.ctr[cur] = 0;
    grid.sync();
    cur ^= 1;
  }
  if (tid == 0) a.ctr[3] = round;
}

__global__ void kcore_keys_kernel(const uint32_t* __restrict__ rnd, uint32_t n, int idbits,
                                  uint64_t* __restrict__ keys) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    keys[v] = (uint64_t(rnd[v]) << idbits) | v;
}

__global__ void kcore_rank_kernel(const uint64_t* __restrict__ sorted, uint32_t n,
                                  uint64_t idmask, uint32_t* __restrict__ rank,
                                  uint32_t* __restrict__ order) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint32_t v = uint32_t(sorted[i] & idmask);
    rank[v] = i;
    order[i] = v;
  }
}

uint64_t rank_kcore(Graph& g) {
  // the reference pops one (degree, id) heap minimum at a
  // time (orientation.cpp:23-46), which is inherently sequential.  This
  // order differs, its max out-degree (= degeneracy) does not.
  const uint32_t n = g.n;
  if (!n) return 0;
  Peel P = peel_state(g, true);
  unsigned* ctr = reinterpret_cast<unsigned*>(P.ctr);
  KCG_CUDA(cudaMemsetAsync(ctr, 0, 8 * 4, g.stream));
  uint32_t* rnd = P.rem;  // reuse: removal round per vertex
  KCG_CUDA(cudaMemsetAsync(rnd, 0xff, size_t(n) * 4, g.stream));
  uint32_t* front = reinterpret_cast<uint32_t*>(P.keys);  // 2n u32 fit in n u64
  KcoreArgs ka{g.und_off.p, g.und_adj.p, n, P.wdeg, rnd, front, ctr};
  int occ = 0;
  KCG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kcore_coop_kernel, 256, 0));
  const unsigned grid = unsigned(std::max(1, occ) * device().sms);
  void* args[] = {&ka};
  KCG_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(kcore_coop_kernel), grid, 256,
                                       args, 0, g.stream));
  KCG_LAUNCHED(g);
  const int idbits = std::max(1, bits_for(n - 1));
  kcore_keys_kernel<<<blocks_for(n, kThreads), kThreads, 0, g.stream>>>(rnd, n, idbits, P.keys2);
  KCG_LAUNCHED(g);
  uint64_t* sorted = P.keys;
  size_t tb = 0;
  const int end_bit = std::min(64, idbits + 32);
  KCG_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, P.keys2, sorted, n, 0, end_bit, g.stream));
  KCG_CUDA(cub::DeviceRadixSort::SortKeys(cub_temp(g, tb), tb, P.keys2, sorted, n, 0, end_bit,
                                          g.stream));
  g.order.ensure(n, &g.alloc);
  kcore_rank_kernel<<<blocks_for(n, kThreads), kThreads, 0, g.stream>>>(
      sorted, n, (uint64_t(1) << idbits) - 1, g.rank.p, g.order.p);
  KCG_LAUNCHED(g);
  unsigned rounds = 0;
  KCG_CUDA(cudaMemcpyAsync(&rounds, ctr + 3, 4, cudaMemcpyDeviceToHost, g.stream));
  g.sync();
  return rounds;
}

}  // namespace

namespace {
uint64_t estimate_impl(Graph& g, double eps) {
  // estimate_arboricity, orientation.cpp:124-155
  if (!(eps > 0)) fail(KCG_EINVAL, "epsilon must be positive");
  const uint32_t n = g.n;
  Peel P = peel_state(g, false);
  uint64_t edges_left = g.m;
  uint32_t nrem = n;
  double peak = 0;
  while (nrem) {
    double density = double(edges_left) / double(nrem);
    peak = std::max(peak, density);
    double cutoff = 2 * (1 + eps) * density;
    Guard<AtMost> flag{AtMost{P.rem, P.wdeg, cutoff}, nrem};
    uint32_t nb = scan_flags(g, flag, nrem, P.pos);
    if (nb == 0) fail(KCG_ERUNTIME, "arboricity estimate: empty batch");
    split_kernel<<<blocks_for(nrem, kThreads), kThreads, 0, g.stream>>>(
        flag, P.rem, nrem, P.pos, P.batch, P.rem2, P.alive, 2, nullptr, 0);
    KCG_LAUNCHED(g);
    KCG_CUDA(cudaMemsetAsync(P.ctr, 0, 8, g.stream));
    unsigned* nh = reinterpret_cast<unsigned*>(P.ctr + 4);
    KCG_CUDA(cudaMemsetAsync(nh, 0, 4, g.stream));
    arb_decrement_kernel<<<blocks_for(uint64_t(nb) * 32, kThreads), kThreads, 0, g.stream>>>(
        P.batch, nb, g.und_off.p, g.und_adj.p, P.alive, P.wdeg, P.ctr, P.hubs, nh);
    KCG_LAUNCHED(g);
    decrement_hub_kernel<true><<<148 * 4, kThreads, 0, g.stream>>>(
        P.hubs, nh, g.und_off.p, g.und_adj.p, P.alive, P.wdeg, P.ctr);
    KCG_LAUNCHED(g);
    kill_kernel<<<blocks_for(nb, kThreads), kThreads, 0, g.stream>>>(P.batch, nb, P.alive);
    KCG_LAUNCHED(g);
    unsigned long long removed = 0;
    KCG_CUDA(cudaMemcpyAsync(&removed, P.ctr, 8, cudaMemcpyDeviceToHost, g.stream));
    g.sync();
    edges_left -= removed;
    std::swap(P.rem, P.rem2);
    nrem -= nb;
  }
  return std::max<uint64_t>(1, uint64_t(std::ceil(peak)));
}
}  // namespace

uint64_t estimate_arboricity(Graph& g, double eps) {
  g.mark(2);
  uint64_t a = estimate_impl(g, eps);
  g.mark(3);
  g.times.rank_ms = g.elapsed(2, 3);
  return a;
}

uint64_t rank_graph(Graph& g, int strategy, double eps, uint64_t alpha_hat,
                    uint64_t* alpha_out) {
  if (strategy < KCG_DEGREE || strategy > KCG_BARENBOIM_ELKIN)
    fail(KCG_EINVAL, "unknown orientation strategy");
  if ((strategy == KCG_BARENBOIM_ELKIN || strategy == KCG_GOODRICH_PSZONA) && !(eps > 0))
    fail(KCG_EINVAL, "epsilon must be positive");
  g.rank.ensure(g.n, &g.alloc);
  g.mark(2);
  uint64_t rounds = 0;
  switch (strategy) {
    case KCG_DEGREE:
      rank_degree(g);
      break;
    case KCG_ORIGINAL:
      if (g.n) iota_kernel<<<blocks_for(g.n, kThreads), kThreads, 0, g.stream>>>(g.rank.p, g.n);
      KCG_LAUNCHED(g);
      break;
    case KCG_KCORE:
      rounds = rank_kcore(g);
      break;
    case KCG_GOODRICH_PSZONA:
      rounds = rank_gp(g, eps);
      break;
    case KCG_BARENBOIM_ELKIN: {
      uint64_t a = alpha_hat ? alpha_hat : estimate_impl(g, eps);
      if (alpha_out) *alpha_out = a;
      rounds = rank_be(g, eps, a);
      break;
    }
  }
  // order[] (inverse permutation) for the relabelled DAG
  g.order.ensure(g.n, &g.alloc);
  if (g.n && strategy != KCG_DEGREE) {
    invert_kernel<<<blocks_for(g.n, kThreads), kThreads, 0, g.stream>>>(g.rank.p, g.n, g.order.p);
    KCG_LAUNCHED(g);
  }
  g.mark(3);
  g.sync();
  g.times.rank_ms = g.elapsed(2, 3);
  return rounds;
}

}  // namespace kcg
