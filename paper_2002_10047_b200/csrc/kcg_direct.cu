// DAG CSR construction (K5 of SURVEY.md §2.3): direct_by_ranking
// (proj/src/graph.cpp:94-114) on the device, plus the rank-relabelled copy
// the counter works on.
//
//  pass 1  one warp per vertex: out-degree = #{v in N(u) : rank v > rank u}
//          (ballot/popc over 32-wide coalesced chunks of the slice)
//  scan    u64 exclusive scans -> id-space offsets and rank-space offsets
//  pass 2  one warp per vertex: ordered (ballot-prefix) compaction of the
//          slice -> id-space targets, ascending by id exactly like the
//          reference; the same pass writes rank[v] into the relabelled
//          slice of vertex rank[u]
//  sort    segmented sort of the relabelled slices (ascending rank), so
//          every out-neighbourhood is in topological order
#include <cub/cub.cuh>
#include <thrust/iterator/transform_iterator.h>

#include <algorithm>

#include "kcg_internal.cuh"

namespace kcg {
namespace {

constexpr int kThreads = 256;

// Hubs (undirected degree > kHubDeg) are listed by the warp kernels and
// handled by one CTA each (outdeg_hub_kernel, fill_hub_kernel): a single warp
// walking a 50k-entry slice with dependent gathers was the long tail of
// both passes on the skewed configs.
constexpr uint32_t kHubDeg = 2048;
// Hub CTAs are latency-bound on the rank gathers: four 512-thread CTAs per SM
// (one per SM left three quarters of the warp slots empty: config 5 hub passes
// 2.9 + 4.6 ms).
constexpr unsigned kHubGrid = 148 * 4;

__global__ void outdeg_kernel(const uint64_t* __restrict__ off, const uint32_t* __restrict__ adj,
                              const uint32_t* __restrict__ rank, uint32_t n,
                              uint64_t* __restrict__ outdeg, uint64_t* __restrict__ rdeg,
                              uint32_t* __restrict__ hubs, unsigned* __restrict__ nhubs) {
  const uint32_t lane = threadIdx.x & 31;
  for (uint64_t u = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; u < n;
       u += (uint64_t(gridDim.x) * blockDim.x) >> 5) {
    const uint32_t ru = rank[u];
    const uint64_t b = off[u], e = off[u + 1];
    if (e - b > kHubDeg) {
      if (lane == 0) hubs[atomicAdd(nhubs, 1u)] = uint32_t(u);
      continue;
    }
    // four 32-entry chunks per step: the adjacency loads, then the rank
    // gathers, are all in flight together (a 2048-entry slice was 64
    // dependent load pairs in a row)
    uint32_t c = 0;
    for (uint64_t p0 = b + lane; p0 < e; p0 += 128) {
      uint32_t v[4];
#pragma unroll
      for (int j = 0; j < 4; j++) v[j] = p0 + 32 * j < e ? adj[p0 + 32 * j] : 0xffffffffu;
#pragma unroll
      for (int j = 0; j < 4; j++) c += v[j] != 0xffffffffu && rank[v[j]] > ru;
    }
    c = __reduce_add_sync(0xffffffffu, c);
    if (lane == 0) {
      if (outdeg) outdeg[u] = c;
      rdeg[ru] = c;
    }
  }
}

// One CTA per hub: the slice is read 4 x 512 entries per step (loads in
// flight), out-neighbours counted with a block reduction.
__global__ void __launch_bounds__(512)
    outdeg_hub_kernel(const uint64_t* __restrict__ off, const uint32_t* __restrict__ adj,
                      const uint32_t* __restrict__ rank, const uint32_t* __restrict__ hubs,
                      const unsigned* __restrict__ nhubs, uint64_t* __restrict__ outdeg,
                      uint64_t* __restrict__ rdeg) {
  typedef cub::BlockReduce<uint32_t, 512> Red;
  __shared__ typename Red::TempStorage tmp;
  const unsigned nh = *nhubs;
  for (unsigned hi = blockIdx.x; hi < nh; hi += gridDim.x) {
    const uint32_t u = hubs[hi];
    const uint32_t ru = rank[u];
    const uint64_t b = off[u], e = off[u + 1];
    uint32_t c = 0;
    for (uint64_t p0 = b + threadIdx.x; p0 < e; p0 += 4 * 512) {
      uint32_t a[4];
#pragma unroll
      for (int j = 0; j < 4; j++) a[j] = p0 + j * 512 < e ? adj[p0 + j * 512] : 0xffffffffu;
#pragma unroll
      for (int j = 0; j < 4; j++) c += a[j] != 0xffffffffu && rank[a[j]] > ru;
    }
    c = Red(tmp).Sum(c);
    if (threadIdx.x == 0) {
      if (outdeg) outdeg[u] = c;
      rdeg[ru] = c;
    }
    __syncthreads();
  }
}

constexpr uint32_t kMidSortL = 256;

__device__ __forceinline__ uint32_t warp_bitonic_sort(uint32_t x, uint32_t lane) {
#pragma unroll
  for (uint32_t k = 2; k <= 32; k <<= 1) {
#pragma unroll
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      const uint32_t y = __shfl_xor_sync(0xffffffffu, x, j);
      const bool keep_min = ((lane & j) == 0) == ((lane & k) == 0);
      x = keep_min ? min(x, y) : max(x, y);
    }
  }
  return x;
}

// Pass 2: ordered compaction of each slice into the id-space DAG (ascending
// ids, like graph.cpp:102-112) and the relabelled slice of rank[u].
// Relabelled slices of <= 32 targets are sorted in registers (warp bitonic
// sort); longer ones are listed for sort_long_kernel.
__global__ void __launch_bounds__(256)
    fill_kernel(const uint64_t* __restrict__ off, const uint32_t* __restrict__ adj,
                const uint32_t* __restrict__ rank, uint32_t n,
                const uint64_t* __restrict__ dag_off, uint32_t* __restrict__ dag_adj,
                const uint64_t* __restrict__ rdag_off, uint32_t* __restrict__ rdag_adj,
                uint32_t* __restrict__ long_list, unsigned* __restrict__ nlong) {
  __shared__ uint32_t buf[8][32];
  const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  for (uint64_t u = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; u < n;
       u += (uint64_t(gridDim.x) * blockDim.x) >> 5) {
    const uint32_t ru = rank[u];
    const uint64_t b = off[u], e = off[u + 1];
    if (e - b > kHubDeg) continue;  // fill_hub_kernel
    uint64_t wid = dag_adj ? dag_off[u] : 0;
    const uint64_t wr0 = rdag_off[ru];
    const uint32_t dout = uint32_t(rdag_off[ru + 1] - wr0);
    const bool shortl = dout <= 32;
    uint32_t got = 0;
    // four chunks per step, loads and gathers in flight together
    for (uint64_t p0 = b + lane; p0 < e + lane && got < dout; p0 += 128) {
      uint32_t v[4], rv[4];
#pragma unroll
      for (int j = 0; j < 4; j++) v[j] = p0 + 32 * j < e ? adj[p0 + 32 * j] : 0xffffffffu;
#pragma unroll
      for (int j = 0; j < 4; j++) rv[j] = v[j] != 0xffffffffu ? rank[v[j]] : 0u;
#pragma unroll
      for (int j = 0; j < 4; j++) {
        const bool out = rv[j] > ru;  // ranks of real targets only: padding has rank 0 <= ru
        const unsigned ball = __ballot_sync(0xffffffffu, out);
        if (out) {
          const uint32_t at = got + __popc(ball & ((1u << lane) - 1));
          if (dag_adj) dag_adj[wid + at] = v[j];
          if (shortl)
            buf[wib][at] = rv[j];
          else
            rdag_adj[wr0 + at] = rv[j];
        }
        got += __popc(ball);
      }
    }
    if (shortl) {
      if (dout) {
        __syncwarp();
        uint32_t x = lane < dout ? buf[wib][lane] : 0xffffffffu;
        x = warp_bitonic_sort(x, lane);
        if (lane < dout) rdag_adj[wr0 + lane] = x;
      }
      __syncwarp();
    } else if (lane == 0) {
      // mid slices from the front of long_list, longer ones from the back
      if (dout <= kMidSortL)
        long_list[atomicAdd(&nlong[0], 1u)] = ru;
      else
        long_list[n - 1 - atomicAdd(&nlong[1], 1u)] = ru;
    }
  }
}

// fill_kernel for the hubs: one CTA each, ordered compaction of 512
// entries per step with a block scan; the relabelled slice goes to the
// sort lists like the warp path's (<= 32 targets: sorted here by warp 0).
__global__ void __launch_bounds__(512)
    fill_hub_kernel(const uint64_t* __restrict__ off, const uint32_t* __restrict__ adj,
                    const uint32_t* __restrict__ rank, uint32_t n,
                    const uint32_t* __restrict__ hubs, const unsigned* __restrict__ nhubs,
                    const uint64_t* __restrict__ dag_off, uint32_t* __restrict__ dag_adj,
                    const uint64_t* __restrict__ rdag_off, uint32_t* __restrict__ rdag_adj,
                    uint32_t* __restrict__ long_list, unsigned* __restrict__ nlong) {
  typedef cub::BlockScan<uint32_t, 512> Scan;
  __shared__ typename Scan::TempStorage tmp;
  const unsigned nh = *nhubs;
  for (unsigned hi = blockIdx.x; hi < nh; hi += gridDim.x) {
    const uint32_t u = hubs[hi];
    const uint32_t ru = rank[u];
    const uint64_t b = off[u], e = off[u + 1];
    const uint64_t wid = dag_adj ? dag_off[u] : 0;
    const uint64_t wr0 = rdag_off[ru];
    const uint32_t dout = uint32_t(rdag_off[ru + 1] - wr0);
    uint32_t got = 0;
    // 2048 entries per step, four consecutive ones per thread (blocked
    // arrangement, loads in flight before the gathers)
    for (uint64_t p0 = b; p0 < e && got < dout; p0 += 4 * 512) {
      const uint64_t pb = p0 + 4 * threadIdx.x;
      uint32_t v[4], rv[4], out[4], at[4];
#pragma unroll
      for (int j = 0; j < 4; j++) v[j] = pb + j < e ? adj[pb + j] : 0xffffffffu;
#pragma unroll
      for (int j = 0; j < 4; j++) {
        rv[j] = v[j] != 0xffffffffu ? rank[v[j]] : 0u;
        out[j] = v[j] != 0xffffffffu && rv[j] > ru;
      }
      uint32_t tot;
      Scan(tmp).ExclusiveSum(out, at, tot);
#pragma unroll
      for (int j = 0; j < 4; j++) {
        if (out[j]) {
          if (dag_adj) dag_adj[wid + got + at[j]] = v[j];
          rdag_adj[wr0 + got + at[j]] = rv[j];
        }
      }
      got += tot;
      __syncthreads();
    }
    if (dout <= 32) {
      __syncthreads();
      if (threadIdx.x < 32 && dout) {
        uint32_t x = threadIdx.x < dout ? rdag_adj[wr0 + threadIdx.x] : 0xffffffffu;
        x = warp_bitonic_sort(x, threadIdx.x);
        if (threadIdx.x < dout) rdag_adj[wr0 + threadIdx.x] = x;
      }
    } else if (threadIdx.x == 0) {
      if (dout <= kMidSortL)
        long_list[atomicAdd(&nlong[0], 1u)] = ru;
      else
        long_list[n - 1 - atomicAdd(&nlong[1], 1u)] = ru;
    }
    __syncthreads();
  }
}

// Bitonic sort of a[0..np2) in shared memory by `nthreads` cooperating
// threads (index t); the caller synchronises between stages via `sync`.
template <class Sync>
__device__ __forceinline__ void smem_bitonic(uint32_t* a, uint32_t np2, uint32_t t,
                                             uint32_t nthreads, Sync sync) {
  for (uint32_t k = 2; k <= np2; k <<= 1)
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      for (uint32_t i = t; i < np2; i += nthreads) {
        const uint32_t l = i ^ j;
        if (l > i) {
          const uint32_t x = a[i], y = a[l];
          if ((x > y) == ((i & k) == 0)) {
            a[i] = y;
            a[l] = x;
          }
        }
      }
      sync();
    }
}

// Bitonic sort of 32*E keys held E per lane (key index = lane*E + r): the
// j < E stages exchange registers of one lane, the others one shuffle per
// key; no shared memory, no barriers.
template <int E>
__device__ __forceinline__ void warp_sort_regs(uint32_t (&a)[E], uint32_t lane) {
#pragma unroll
  for (uint32_t k = 2; k <= 32u * E; k <<= 1) {
#pragma unroll
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      if (j < uint32_t(E)) {
#pragma unroll
        for (uint32_t r = 0; r < uint32_t(E); r++) {
          if ((r & j) == 0) {
            const bool asc = k < uint32_t(E) ? (r & k) == 0 : ((lane * E + r) & k) == 0;
            const uint32_t lo = min(a[r], a[r ^ j]), hi = max(a[r], a[r ^ j]);
            a[r] = asc ? lo : hi;
            a[r ^ j] = asc ? hi : lo;
          }
        }
      } else {
        const uint32_t lj = j / E;
        const bool keep_min = ((lane & lj) == 0) == (((lane * E) & k) == 0);
#pragma unroll
        for (uint32_t r = 0; r < uint32_t(E); r++) {
          const uint32_t y = __shfl_xor_sync(0xffffffffu, a[r], lj);
          a[r] = keep_min ? min(a[r], y) : max(a[r], y);
        }
      }
    }
  }
}

template <int E>
__device__ __forceinline__ void warp_sort_slice(uint32_t* __restrict__ p, uint32_t len,
                                                uint32_t lane) {
  uint32_t a[E];
#pragma unroll
  for (int r = 0; r < E; r++) a[r] = 32 * r + lane < len ? p[32 * r + lane] : 0xffffffffu;
  warp_sort_regs<E>(a, lane);
#pragma unroll
  for (int r = 0; r < E; r++)
    if (lane * E + r < len) p[lane * E + r] = a[r];
}

// Relabelled slices of 33..1024 targets: one warp each, sorted in registers
// (8, 16 or 32 keys per lane).  Longer slices are left to sort_big_kernel.
constexpr uint32_t kWarpSortMax = 1024;
// EMAX = 8: the list holds slices of <= 256 targets only (the kernel then
// needs few registers and runs at full occupancy); 32: up to kWarpSortMax.
template <int EMAX>
__global__ void __launch_bounds__(256)
    sort_warp_kernel(const uint32_t* __restrict__ list, uint32_t nl,
                     const uint64_t* __restrict__ off, uint32_t* __restrict__ adj) {
  const uint32_t lane = threadIdx.x & 31;
  for (uint32_t li = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; li < nl;
       li += (gridDim.x * blockDim.x) >> 5) {
    const uint32_t r = list[li];
    const uint64_t b = off[r];
    const uint32_t len = uint32_t(off[r + 1] - b);
    if (len <= 256) {
      warp_sort_slice<8>(adj + b, len, lane);
    } else if constexpr (EMAX > 8) {
      if (len <= 512)
        warp_sort_slice<16>(adj + b, len, lane);
      else if (len <= kWarpSortMax)
        warp_sort_slice<32>(adj + b, len, lane);
    }
    __syncwarp();
  }
}

constexpr uint32_t kBigSort = 8192;

// Slices of 1025..8192 targets: one CTA each.
__global__ void __launch_bounds__(512)
    sort_big_kernel(const uint32_t* __restrict__ list, uint32_t nl,
                    const uint64_t* __restrict__ off, uint32_t* __restrict__ adj) {
  __shared__ uint32_t sm[kBigSort];
  for (uint32_t li = blockIdx.x; li < nl; li += gridDim.x) {
    const uint32_t r = list[li];
    const uint64_t b = off[r];
    const uint32_t len = uint32_t(off[r + 1] - b);
    if (len <= kWarpSortMax) continue;  // sort_warp_kernel
    uint32_t np2 = 512;
    while (np2 < len) np2 <<= 1;
    for (uint32_t i = threadIdx.x; i < np2; i += blockDim.x)
      sm[i] = i < len ? adj[b + i] : 0xffffffffu;
    __syncthreads();
    smem_bitonic(sm, np2, threadIdx.x, blockDim.x, [] __device__() { __syncthreads(); });
    for (uint32_t i = threadIdx.x; i < len; i += blockDim.x) adj[b + i] = sm[i];
    __syncthreads();
  }
}

// Copies the listed slices from the sort output back into rdag_adj.
__global__ void copy_slices_kernel(const uint32_t* __restrict__ list, uint32_t nl,
                                   const uint64_t* __restrict__ off,
                                   const uint32_t* __restrict__ src, uint32_t* __restrict__ dst) {
  for (uint32_t li = blockIdx.x; li < nl; li += gridDim.x) {
    const uint32_t r = list[li];
    for (uint64_t p = off[r] + threadIdx.x; p < off[r + 1]; p += blockDim.x) dst[p] = src[p];
  }
}

// Offsets of the listed (long) relabelled slices, for CUB.
struct SliceBegin {
  const uint32_t* list;
  const uint64_t* off;
  __host__ __device__ uint64_t operator()(uint32_t i) const { return off[list[i]]; }
};
struct SliceEnd {
  const uint32_t* list;
  const uint64_t* off;
  __host__ __device__ uint64_t operator()(uint32_t i) const { return off[list[i] + 1]; }
};

// Relabel an adopted id-space DAG: slice of u becomes slice rank[u] with
// targets mapped to ranks; flags edges that do not point up in rank.
__global__ void relabel_kernel(const uint64_t* __restrict__ dag_off,
                               const uint32_t* __restrict__ dag_adj,
                               const uint32_t* __restrict__ rank, uint32_t n,
                               const uint64_t* __restrict__ rdag_off,
                               uint32_t* __restrict__ rdag_adj,
                               unsigned long long* __restrict__ bad) {
  const uint32_t lane = threadIdx.x & 31;
  for (uint64_t u = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; u < n;
       u += (uint64_t(gridDim.x) * blockDim.x) >> 5) {
    const uint32_t ru = rank[u];
    const uint64_t b = dag_off[u], e = dag_off[u + 1], w = rdag_off[ru];
    for (uint64_t p = b + lane; p < e; p += 32) {
      uint32_t v = dag_adj[p];
      uint32_t rv = v < n ? rank[v] : 0;
      if (v >= n || rv <= ru) atomicAdd(bad, 1ull);
      rdag_adj[w + (p - b)] = rv;
    }
  }
}

__global__ void dag_deg_kernel(const uint64_t* __restrict__ dag_off,
                               const uint32_t* __restrict__ rank, uint32_t n,
                               uint64_t* __restrict__ rdeg) {
  for (uint32_t u = blockIdx.x * blockDim.x + threadIdx.x; u < n; u += gridDim.x * blockDim.x)
    rdeg[rank[u]] = dag_off[u + 1] - dag_off[u];
}

void exclusive_scan_u64(Graph& g, uint64_t* in, uint64_t* out, size_t count) {
  size_t tb = 0;
  KCG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, in, out, count, g.stream));
  KCG_CUDA(cub::DeviceScan::ExclusiveSum(cub_temp(g, tb), tb, in, out, count, g.stream));
}

void max_out_degree(Graph& g, const uint64_t* rdeg) {
  uint64_t* mx = reinterpret_cast<uint64_t*>(g.counters.ensure(4, &g.alloc));
  size_t tb = 0;
  KCG_CUDA(cub::DeviceReduce::Max(nullptr, tb, rdeg, mx, g.n, g.stream));
  KCG_CUDA(cub::DeviceReduce::Max(cub_temp(g, tb), tb, rdeg, mx, g.n, g.stream));
  KCG_CUDA(cudaMemcpyAsync(&g.max_out, mx, 8, cudaMemcpyDeviceToHost, g.stream));
}

// ascending-rank slices for every vertex (CUB segmented sort)
void sort_all_slices(Graph& g) {
  const uint32_t n = g.n;
  size_t tb = 0;
  if (g.m) {
    uint32_t* tmp = reinterpret_cast<uint32_t*>(g.scratch2.ensure(g.m * 4 + 16, &g.alloc));
    tb = 0;
    KCG_CUDA(cub::DeviceSegmentedSort::SortKeys(nullptr, tb, g.rdag_adj.p, tmp, g.m, n,
                                                g.rdag_off.p, g.rdag_off.p + 1, g.stream));
    KCG_CUDA(cub::DeviceSegmentedSort::SortKeys(cub_temp(g, tb), tb, g.rdag_adj.p, tmp, g.m,
                                                n, g.rdag_off.p, g.rdag_off.p + 1, g.stream));
    KCG_CUDA(cudaMemcpyAsync(g.rdag_adj.p, tmp, g.m * 4, cudaMemcpyDeviceToDevice, g.stream));
  }
}

}  // namespace

void build_dag(Graph& g, bool want_id_dag) {
  if (!g.has_und) fail(KCG_EINVAL, "handle holds no undirected graph");
  const uint32_t n = g.n;
  g.mark(2);
  g.rdag_off.ensure(size_t(n) + 1, &g.alloc);
  g.rdag_adj.ensure(g.m, &g.alloc);
  if (want_id_dag) {
    g.dag_off.ensure(size_t(n) + 1, &g.alloc);
    g.dag_adj.ensure(g.m, &g.alloc);
  }
  // degree arrays live in pv_rank / pv (n+1 u64 each) until counting
  uint64_t* rdeg = g.pv_rank.ensure(size_t(n) + 1, &g.alloc);
  uint64_t* odeg = want_id_dag ? g.pv.ensure(size_t(n) + 1, &g.alloc) : nullptr;
  KCG_CUDA(cudaMemsetAsync(rdeg + n, 0, 8, g.stream));
  if (odeg) KCG_CUDA(cudaMemsetAsync(odeg + n, 0, 8, g.stream));
  unsigned grid = blocks_for(uint64_t(n) * 32, kThreads, 148u * 64u);
  uint32_t* lists = reinterpret_cast<uint32_t*>(g.scratch3.ensure(size_t(n) * 8 + 64, &g.alloc));
  uint32_t* hubs = lists + n;
  unsigned* cnt = reinterpret_cast<unsigned*>(g.counters.ensure(8, &g.alloc) + 3);
  KCG_CUDA(cudaMemsetAsync(cnt, 0, 12, g.stream));  // [0,1] sort lists, [2] hubs
  if (n) {
    outdeg_kernel<<<grid, kThreads, 0, g.stream>>>(g.und_off.p, g.und_adj.p, g.rank.p, n, odeg,
                                                   rdeg, hubs, cnt + 2);
    KCG_LAUNCHED(g);
    outdeg_hub_kernel<<<kHubGrid, 512, 0, g.stream>>>(g.und_off.p, g.und_adj.p, g.rank.p, hubs,
                                                 cnt + 2, odeg, rdeg);
    KCG_LAUNCHED(g);
  }
  exclusive_scan_u64(g, rdeg, g.rdag_off.p, size_t(n) + 1);
  if (odeg) exclusive_scan_u64(g, odeg, g.dag_off.p, size_t(n) + 1);
  if (n) {
    fill_kernel<<<grid, kThreads, 0, g.stream>>>(g.und_off.p, g.und_adj.p, g.rank.p, n,
                                                 want_id_dag ? g.dag_off.p : nullptr,
                                                 want_id_dag ? g.dag_adj.p : nullptr,
                                                 g.rdag_off.p, g.rdag_adj.p, lists, cnt);
    KCG_LAUNCHED(g);
    fill_hub_kernel<<<kHubGrid, 512, 0, g.stream>>>(g.und_off.p, g.und_adj.p, g.rank.p, n, hubs,
                                               cnt + 2, want_id_dag ? g.dag_off.p : nullptr,
                                               want_id_dag ? g.dag_adj.p : nullptr, g.rdag_off.p,
                                               g.rdag_adj.p, lists, cnt);
    KCG_LAUNCHED(g);
  }
  max_out_degree(g, rdeg);
  unsigned hcnt[2] = {0, 0};
  KCG_CUDA(cudaMemcpyAsync(hcnt, cnt, 8, cudaMemcpyDeviceToHost, g.stream));
  g.sync();
  if (hcnt[0]) {  // 33..256 targets: a warp per slice
    sort_warp_kernel<8><<<std::min<unsigned>((hcnt[0] + 7) / 8, 148u * 16u), 256, 0, g.stream>>>(
        lists, hcnt[0], g.rdag_off.p, g.rdag_adj.p);
    KCG_LAUNCHED(g);
  }
  if (hcnt[1]) {  // longer slices, listed from the back of `lists`
    const uint32_t* big = lists + n - hcnt[1];
    uint32_t maxlen = uint32_t(std::min<uint64_t>(g.max_out, 0xffffffffu));
    sort_warp_kernel<32><<<std::min<unsigned>((hcnt[1] + 7) / 8, 148u * 16u), 256, 0, g.stream>>>(
        big, hcnt[1], g.rdag_off.p, g.rdag_adj.p);  // 257..1024 targets
    KCG_LAUNCHED(g);
    if (maxlen <= kWarpSortMax) {
      // nothing longer than the warp sort takes
    } else if (maxlen <= kBigSort) {
      sort_big_kernel<<<std::min<unsigned>(hcnt[1], 148u * 4u), 512, 0, g.stream>>>(
          big, hcnt[1], g.rdag_off.p, g.rdag_adj.p);
      KCG_LAUNCHED(g);
    } else {
      // CUB segmented sort over just those slices
      auto cnt_it = thrust::counting_iterator<uint32_t>(0);
      auto beg = thrust::make_transform_iterator(cnt_it, SliceBegin{big, g.rdag_off.p});
      auto end = thrust::make_transform_iterator(cnt_it, SliceEnd{big, g.rdag_off.p});
      uint32_t* tmp = reinterpret_cast<uint32_t*>(g.scratch2.ensure(g.m * 4 + 16, &g.alloc));
      size_t tb = 0;
      KCG_CUDA(cub::DeviceSegmentedSort::SortKeys(nullptr, tb, g.rdag_adj.p, tmp, g.m, hcnt[1],
                                                  beg, end, g.stream));
      KCG_CUDA(cub::DeviceSegmentedSort::SortKeys(cub_temp(g, tb), tb, g.rdag_adj.p, tmp, g.m,
                                                  hcnt[1], beg, end, g.stream));
      copy_slices_kernel<<<std::min<unsigned>(hcnt[1], 148u * 8u), 256, 0, g.stream>>>(
          big, hcnt[1], g.rdag_off.p, tmp, g.rdag_adj.p);
      KCG_LAUNCHED(g);
    }
  }
  g.mark(3);
  g.times.direct_ms = g.elapsed(2, 3);
  g.has_rdag = true;
  if (want_id_dag) g.has_dag = true;
}

void relabel_from_dag(Graph& g) {
  const uint32_t n = g.n;
  g.mark(2);
  g.rdag_off.ensure(size_t(n) + 1, &g.alloc);
  g.rdag_adj.ensure(g.m, &g.alloc);
  uint64_t* rdeg = g.pv_rank.ensure(size_t(n) + 1, &g.alloc);
  KCG_CUDA(cudaMemsetAsync(rdeg + n, 0, 8, g.stream));
  if (n)
    dag_deg_kernel<<<blocks_for(n, kThreads), kThreads, 0, g.stream>>>(g.dag_off.p, g.rank.p, n,
                                                                       rdeg);
  KCG_LAUNCHED(g);
  exclusive_scan_u64(g, rdeg, g.rdag_off.p, size_t(n) + 1);
  unsigned long long* bad = g.counters.ensure(4, &g.alloc) + 2;
  KCG_CUDA(cudaMemsetAsync(bad, 0, 8, g.stream));
  if (n)
    relabel_kernel<<<blocks_for(uint64_t(n) * 32, kThreads, 148u * 64u), kThreads, 0, g.stream>>>(
        g.dag_off.p, g.dag_adj.p, g.rank.p, n, g.rdag_off.p, g.rdag_adj.p, bad);
  KCG_LAUNCHED(g);
  unsigned long long nbad = 0;
  KCG_CUDA(cudaMemcpyAsync(&nbad, bad, 8, cudaMemcpyDeviceToHost, g.stream));
  max_out_degree(g, rdeg);
  sort_all_slices(g);
  g.sync();
  if (nbad) fail(KCG_EINVAL, "DAG edge does not point toward higher rank");
  g.mark(3);
  g.times.direct_ms = g.elapsed(2, 3);
  g.has_rdag = true;
}

}  // namespace kcg
