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
  if (tid == 0) {
    a.ctr[3] = round;
    a.ctr[4] = level;  // the degeneracy (max core number)
  }
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

uint64_t rank_kcore(Graph& g, uint32_t* degeneracy = nullptr) {
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
  unsigned hv[2] = {0, 0};
  KCG_CUDA(cudaMemcpyAsync(hv, ctr + 3, 8, cudaMemcpyDeviceToHost, g.stream));
  g.sync();
  if (degeneracy) *degeneracy = hv[1];
  return hv[0];
}

// ---- exact rank_by_kcore -----------------------------------------------------
// The reference pops the (induced degree, id) minimum one vertex at a time
// (orientation.cpp:23-46).  Reproduced exactly by one CTA: alive vertices of
// degree <= D (the degeneracy, from the parallel peel above -- the minimum
// alive degree never exceeds it) sit in per-degree hierarchical bitmaps
// (32-ary levels over the ids, top level <= 32 words), so the minimum is
// "lowest non-empty bucket, then first set bit" in one warp ballot per
// level; a pop clears its bit, decrements its live neighbours and moves
// them one bucket down (clears, barrier, sets).  The minimum bucket only
// falls by one per pop, so the search restarts one bucket below the last.
struct KcX {
  const uint64_t* off;
  const uint32_t* adj;
  uint32_t n, D, nlev;
  uint32_t lw[6];       // words per level (level 0 = ids)
  uint64_t lo[6];       // word offset of each level inside a bucket
  uint64_t bwords;      // words per bucket
  uint32_t* bits;       // (D + 1) * bwords
  uint32_t* deg;
  uint8_t* done;
  uint32_t* rank;
  uint32_t* order;
  unsigned* err;
};

__device__ __forceinline__ void kx_clear(const KcX& a, uint32_t b, uint32_t v) {
  uint32_t* B = a.bits + uint64_t(b) * a.bwords;
  uint32_t idx = v;
  for (uint32_t l = 0; l < a.nlev; l++) {
    const uint32_t bit = 1u << (idx & 31);
    const uint32_t old = atomicAnd(&B[a.lo[l] + (idx >> 5)], ~bit);
    if ((old & ~bit) != 0) break;  // word still non-empty
    idx >>= 5;
  }
}

__device__ __forceinline__ void kx_set(const KcX& a, uint32_t b, uint32_t v) {
  uint32_t* B = a.bits + uint64_t(b) * a.bwords;
  uint32_t idx = v;
  for (uint32_t l = 0; l < a.nlev; l++) {
    const uint32_t old = atomicOr(&B[a.lo[l] + (idx >> 5)], 1u << (idx & 31));
    if (old != 0) break;  // upper levels already mark this word
    idx >>= 5;
  }
}

__global__ void kx_fill_kernel(KcX a) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < a.n; v += gridDim.x * blockDim.x) {
    const uint32_t d = uint32_t(a.off[v + 1] - a.off[v]);
    a.deg[v] = d;
    if (d <= a.D) kx_set(a, d, v);
  }
}

constexpr int kKxThreads = 1024;

__global__ void __launch_bounds__(kKxThreads) kx_peel_kernel(KcX a) {
  __shared__ uint32_t s_v, s_b;
  const uint32_t lane = threadIdx.x & 31;
  uint32_t b = 0;
  for (uint32_t step = 0; step < a.n; step++) {
    if (threadIdx.x < 32) {
      // lowest non-empty bucket at or above b, then its first set bit
      const uint32_t top = a.nlev - 1;
      uint32_t w = 0;
      for (; b <= a.D; b++) {
        const uint32_t* B = a.bits + uint64_t(b) * a.bwords;
        w = lane < a.lw[top] ? B[a.lo[top] + lane] : 0u;
        if (__ballot_sync(0xffffffffu, w != 0)) break;
      }
      if (b > a.D) {  // cannot happen while D is the degeneracy
        if (lane == 0) {
          *a.err = 1;
          s_v = 0xffffffffu;
        }
      } else {
        const uint32_t* B = a.bits + uint64_t(b) * a.bwords;
        const unsigned nz = __ballot_sync(0xffffffffu, w != 0);
        const uint32_t f = __ffs(nz) - 1;
        uint32_t word = __shfl_sync(0xffffffffu, w, f);
        uint32_t idx = f * 32 + __ffs(word) - 1;
        for (int l = int(top) - 1; l >= 0; l--) {
          word = B[a.lo[l] + idx];  // warp-uniform load
          idx = idx * 32 + __ffs(word) - 1;
        }
        if (lane == 0) {
          s_v = idx;
          s_b = b;
        }
      }
    }
    __syncthreads();
    if (s_v == 0xffffffffu) return;
    const uint32_t v = s_v, bv = s_b;
    if (threadIdx.x == 0) {
      a.done[v] = 1;
      a.rank[v] = step;
      a.order[step] = v;
      kx_clear(a, bv, v);
    }
    b = bv ? bv - 1 : 0;
    // neighbours, kKxThreads at a time: clear from old bucket, then set
    const uint64_t e = a.off[v + 1];
    for (uint64_t p0 = a.off[v]; p0 < e; p0 += kKxThreads) {
      const uint64_t p = p0 + threadIdx.x;
      uint32_t u = 0xffffffffu, nd = 0xffffffffu;
      if (p < e) {
        u = a.adj[p];
        if (u != v && !a.done[u]) {
          const uint32_t od = a.deg[u];
          nd = od - 1;
          a.deg[u] = nd;
          if (od <= a.D) kx_clear(a, od, u);
        } else {
          u = 0xffffffffu;
        }
      }
      __syncthreads();
      if (u != 0xffffffffu && nd <= a.D) kx_set(a, nd, u);
      __syncthreads();
    }
  }
}

uint64_t rank_kcore_exact(Graph& g) {
  const uint32_t n = g.n;
  if (!n) return 0;
  uint32_t D = 0;
  rank_kcore(g, &D);  // the degeneracy bounds every bucket we need
  KcX a{};
  a.off = g.und_off.p;
  a.adj = g.und_adj.p;
  a.n = n;
  a.D = D;
  uint64_t words = 0;
  uint32_t len = n;
  uint32_t l = 0;
  do {
    len = (len + 31) / 32;
    if (l >= 6) fail(KCG_ERUNTIME, "exact k-core: graph too large for the bucket levels");
    a.lw[l] = len;
    a.lo[l] = words;
    words += len;
    l++;
  } while (len > 32);
  a.nlev = l;
  a.bwords = (words + 31) & ~uint64_t(31);
  const uint64_t total_words = a.bwords * (uint64_t(D) + 1);
  DevBuf<uint32_t> bits;
  bits.ensure(total_words, &g.alloc);
  KCG_CUDA(cudaMemsetAsync(bits.p, 0, total_words * 4, g.stream));
  a.bits = bits.p;
  Peel P = peel_state(g, false);
  a.deg = P.wdeg;
  a.done = P.alive;  // reused as the done flags
  KCG_CUDA(cudaMemsetAsync(a.done, 0, n, g.stream));
  a.rank = g.rank.p;
  g.order.ensure(n, &g.alloc);
  a.order = g.order.p;
  kx_fill_kernel<<<blocks_for(n, kThreads), kThreads, 0, g.stream>>>(a);
  KCG_LAUNCHED(g);
  a.err = reinterpret_cast<unsigned*>(P.ctr + 5);
  KCG_CUDA(cudaMemsetAsync(a.err, 0, 4, g.stream));
  kx_peel_kernel<<<1, kKxThreads, 0, g.stream>>>(a);
  KCG_LAUNCHED(g);
  unsigned err = 0;
  KCG_CUDA(cudaMemcpyAsync(&err, a.err, 4, cudaMemcpyDeviceToHost, g.stream));
  g.sync();
  if (err) fail(KCG_ERUNTIME, "exact k-core: no bucket at or below the degeneracy");
  return 0;
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
  if (strategy < KCG_DEGREE || strategy > KCG_KCORE_PARALLEL)
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
      rounds = rank_kcore_exact(g);
      break;
    case KCG_KCORE_PARALLEL:
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
