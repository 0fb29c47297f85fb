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

#include <algorithm>

#include "kcg_internal.cuh"

namespace kcg {
namespace {

constexpr int kThreads = 256;

__global__ void outdeg_kernel(const uint64_t* __restrict__ off, const uint32_t* __restrict__ adj,
                              const uint32_t* __restrict__ rank, uint32_t n,
                              uint64_t* __restrict__ outdeg, uint64_t* __restrict__ rdeg) {
  const uint32_t lane = threadIdx.x & 31;
  for (uint64_t u = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; u < n;
       u += (uint64_t(gridDim.x) * blockDim.x) >> 5) {
    const uint32_t ru = rank[u];
    const uint64_t b = off[u], e = off[u + 1];
    uint32_t c = 0;
    for (uint64_t p0 = b; p0 < e; p0 += 32) {
      uint64_t p = p0 + lane;
      bool out = p < e && rank[adj[p]] > ru;
      c += __popc(__ballot_sync(0xffffffffu, out));
    }
    if (lane == 0) {
      if (outdeg) outdeg[u] = c;
      rdeg[ru] = c;
    }
  }
}

__global__ void fill_kernel(const uint64_t* __restrict__ off, const uint32_t* __restrict__ adj,
                            const uint32_t* __restrict__ rank, uint32_t n,
                            const uint64_t* __restrict__ dag_off, uint32_t* __restrict__ dag_adj,
                            const uint64_t* __restrict__ rdag_off,
                            uint32_t* __restrict__ rdag_adj) {
  const uint32_t lane = threadIdx.x & 31;
  for (uint64_t u = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; u < n;
       u += (uint64_t(gridDim.x) * blockDim.x) >> 5) {
    const uint32_t ru = rank[u];
    const uint64_t b = off[u], e = off[u + 1];
    uint64_t wid = dag_adj ? dag_off[u] : 0;
    uint64_t wr = rdag_off[ru];
    for (uint64_t p0 = b; p0 < e; p0 += 32) {
      uint64_t p = p0 + lane;
      uint32_t v = 0, rv = 0;
      bool out = false;
      if (p < e) {
        v = adj[p];
        rv = rank[v];
        out = rv > ru;
      }
      unsigned ball = __ballot_sync(0xffffffffu, out);
      if (out) {
        uint32_t at = __popc(ball & ((1u << lane) - 1));
        if (dag_adj) dag_adj[wid + at] = v;
        rdag_adj[wr + at] = rv;
      }
      wid += __popc(ball);
      wr += __popc(ball);
    }
  }
}

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

void sort_rdag_and_max(Graph& g, const uint64_t* rdeg) {
  const uint32_t n = g.n;
  // max out-degree
  uint64_t* mx = reinterpret_cast<uint64_t*>(g.counters.ensure(4, &g.bytes));
  size_t tb = 0;
  KCG_CUDA(cub::DeviceReduce::Max(nullptr, tb, rdeg, mx, n, g.stream));
  KCG_CUDA(cub::DeviceReduce::Max(cub_temp(g, tb), tb, rdeg, mx, n, g.stream));
  KCG_CUDA(cudaMemcpyAsync(&g.max_out, mx, 8, cudaMemcpyDeviceToHost, g.stream));
  // ascending-rank slices
  if (g.m) {
    uint32_t* tmp = reinterpret_cast<uint32_t*>(g.scratch2.ensure(g.m * 4 + 16, &g.bytes));
    tb = 0;
    KCG_CUDA(cub::DeviceSegmentedSort::SortKeys(nullptr, tb, g.rdag_adj.p, tmp, g.m, n,
                                                g.rdag_off.p, g.rdag_off.p + 1, g.stream));
    KCG_CUDA(cub::DeviceSegmentedSort::SortKeys(cub_temp(g, tb), tb, g.rdag_adj.p, tmp, g.m,
                                                n, g.rdag_off.p, g.rdag_off.p + 1, g.stream));
    KCG_CUDA(cudaMemcpyAsync(g.rdag_adj.p, tmp, g.m * 4, cudaMemcpyDeviceToDevice, g.stream));
  }
  g.sync();
}

}  // namespace

void build_dag(Graph& g, bool want_id_dag) {
  if (!g.has_und) fail(KCG_EINVAL, "handle holds no undirected graph");
  const uint32_t n = g.n;
  g.mark(2);
  g.rdag_off.ensure(size_t(n) + 1, &g.bytes);
  g.rdag_adj.ensure(g.m, &g.bytes);
  if (want_id_dag) {
    g.dag_off.ensure(size_t(n) + 1, &g.bytes);
    g.dag_adj.ensure(g.m, &g.bytes);
  }
  // degree arrays live in pv_rank / pv (n+1 u64 each) until counting
  uint64_t* rdeg = g.pv_rank.ensure(size_t(n) + 1, &g.bytes);
  uint64_t* odeg = want_id_dag ? g.pv.ensure(size_t(n) + 1, &g.bytes) : nullptr;
  KCG_CUDA(cudaMemsetAsync(rdeg + n, 0, 8, g.stream));
  if (odeg) KCG_CUDA(cudaMemsetAsync(odeg + n, 0, 8, g.stream));
  unsigned grid = blocks_for(uint64_t(n) * 32, kThreads, 148u * 64u);
  if (n) outdeg_kernel<<<grid, kThreads, 0, g.stream>>>(g.und_off.p, g.und_adj.p, g.rank.p, n,
                                                        odeg, rdeg);
  KCG_LAUNCHED(g);
  exclusive_scan_u64(g, rdeg, g.rdag_off.p, size_t(n) + 1);
  if (odeg) exclusive_scan_u64(g, odeg, g.dag_off.p, size_t(n) + 1);
  if (n)
    fill_kernel<<<grid, kThreads, 0, g.stream>>>(g.und_off.p, g.und_adj.p, g.rank.p, n,
                                                 want_id_dag ? g.dag_off.p : nullptr,
                                                 want_id_dag ? g.dag_adj.p : nullptr,
                                                 g.rdag_off.p, g.rdag_adj.p);
  KCG_LAUNCHED(g);
  sort_rdag_and_max(g, rdeg);
  g.mark(3);
  g.times.direct_ms = g.elapsed(2, 3);
  g.has_rdag = true;
  if (want_id_dag) g.has_dag = true;
}

void relabel_from_dag(Graph& g) {
  const uint32_t n = g.n;
  g.mark(2);
  g.rdag_off.ensure(size_t(n) + 1, &g.bytes);
  g.rdag_adj.ensure(g.m, &g.bytes);
  uint64_t* rdeg = g.pv_rank.ensure(size_t(n) + 1, &g.bytes);
  KCG_CUDA(cudaMemsetAsync(rdeg + n, 0, 8, g.stream));
  if (n)
    dag_deg_kernel<<<blocks_for(n, kThreads), kThreads, 0, g.stream>>>(g.dag_off.p, g.rank.p, n,
                                                                       rdeg);
  KCG_LAUNCHED(g);
  exclusive_scan_u64(g, rdeg, g.rdag_off.p, size_t(n) + 1);
  unsigned long long* bad = g.counters.ensure(4, &g.bytes) + 2;
  KCG_CUDA(cudaMemsetAsync(bad, 0, 8, g.stream));
  if (n)
    relabel_kernel<<<blocks_for(uint64_t(n) * 32, kThreads, 148u * 64u), kThreads, 0, g.stream>>>(
        g.dag_off.p, g.dag_adj.p, g.rank.p, n, g.rdag_off.p, g.rdag_adj.p, bad);
  KCG_LAUNCHED(g);
  unsigned long long nbad = 0;
  KCG_CUDA(cudaMemcpyAsync(&nbad, bad, 8, cudaMemcpyDeviceToHost, g.stream));
  sort_rdag_and_max(g, rdeg);
  if (nbad) fail(KCG_EINVAL, "DAG edge does not point toward higher rank");
  g.mark(3);
  g.times.direct_ms = g.elapsed(2, 3);
  g.has_rdag = true;
}

}  // namespace kcg
