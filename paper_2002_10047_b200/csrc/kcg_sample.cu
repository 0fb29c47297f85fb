// Colour-sparsified approximate counting on the device (SURVEY.md §8(f)
// row 3): colorful_sparsify and approx_count of proj/src/sampling.cpp.
//
// Every vertex gets colour floor(h(seed, v) * colors / 2^64) with the
// reference's counter-based hash (sampling.cpp:10-24); an edge survives iff
// its endpoints share a colour.  One warp per vertex filters its CSR slice
// with an ordered ballot compaction (slices stay ascending), so the result
// is exactly Graph::from_edges of the kept pairs (sampling.cpp:28-40).
#include <cub/cub.cuh>

#include <algorithm>

#include "kcg_internal.cuh"

namespace kcg {
namespace {

typedef unsigned long long ull;

__host__ __device__ __forceinline__ ull splitmix64(ull x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

__global__ void color_kernel(uint32_t n, ull seed_mix, ull colors, ull* __restrict__ color) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    const ull h = splitmix64(seed_mix + 0x9e3779b97f4a7c15ull * (ull(v) + 1));
    color[v] = __umul64hi(h, colors);
  }
}

// pass 1 (write == false): kept-degree per vertex into cnt[v] (cnt[n] = 0);
// pass 2: ordered compaction into the new adjacency at off2[v]
template <bool WRITE>
__global__ void mono_kernel(const uint64_t* __restrict__ off, const uint32_t* __restrict__ adj,
                            const ull* __restrict__ color, uint32_t n, ull* __restrict__ cnt,
                            const uint64_t* __restrict__ off2, uint32_t* __restrict__ adj2) {
  const uint32_t lane = threadIdx.x & 31;
  for (uint64_t v = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; v <= n;
       v += (uint64_t(gridDim.x) * blockDim.x) >> 5) {
    if (v == n) {
      if (!WRITE && lane == 0) cnt[n] = 0;
      continue;
    }
    const ull cv = color[v];
    const uint64_t b = off[v], e = off[v + 1];
    uint64_t w = WRITE ? off2[v] : 0;
    uint32_t c = 0;
    for (uint64_t p0 = b; p0 < e; p0 += 32) {
      const uint64_t p = p0 + lane;
      uint32_t u = 0;
      bool keep = false;
      if (p < e) {
        u = adj[p];
        keep = color[u] == cv;
      }
      const unsigned bal = __ballot_sync(0xffffffffu, keep);
      if (WRITE && keep) adj2[w + __popc(bal & ((1u << lane) - 1u))] = u;
      w += __popc(bal);
      c += __popc(bal);
    }
    if (!WRITE && lane == 0) cnt[v] = c;
  }
}

__global__ void degree_kernel2(const uint64_t* __restrict__ off, uint32_t n,
                               uint32_t* __restrict__ deg) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    deg[v] = uint32_t(off[v + 1] - off[v]);
}

}  // namespace

void colorful_sparsify(const Graph& src, Graph& dst, uint64_t colors, uint64_t seed) {
  if (colors < 1) fail(KCG_EINVAL, "colors must be at least 1");
  if (!src.has_und) fail(KCG_EINVAL, "handle holds no undirected graph");
  const uint32_t n = src.n;
  dst.n = n;
  dst.mark(0);
  // wait for the source handle's queued work before reading its CSR
  KCG_CUDA(cudaStreamSynchronize(src.stream));
  dst.und_off.ensure(size_t(n) + 1, &dst.alloc);
  if (colors == 1) {  // sampling.cpp:31: the graph itself
    dst.m = src.m;
    dst.und_adj.ensure(std::max<uint64_t>(2 * src.m, 1), &dst.alloc);
    KCG_CUDA(cudaMemcpyAsync(dst.und_off.p, src.und_off.p, (size_t(n) + 1) * 8,
                             cudaMemcpyDeviceToDevice, dst.stream));
    if (src.m)
      KCG_CUDA(cudaMemcpyAsync(dst.und_adj.p, src.und_adj.p, 2 * src.m * 4,
                               cudaMemcpyDeviceToDevice, dst.stream));
  } else {
    const size_t b64 = ((size_t(n) + 1) * 8 + 255) & ~size_t(255);
    unsigned char* ws = dst.scratch2.ensure(2 * b64, &dst.alloc);
    ull* color = reinterpret_cast<ull*>(ws);
    ull* cnt = reinterpret_cast<ull*>(ws + b64);
    if (n) {
      color_kernel<<<blocks_for(n, 256), 256, 0, dst.stream>>>(n, splitmix64(seed), colors, color);
      KCG_LAUNCHED(dst);
    }
    mono_kernel<false><<<blocks_for((uint64_t(n) + 1) * 32, 256), 256, 0, dst.stream>>>(
        src.und_off.p, src.und_adj.p, color, n, cnt, nullptr, nullptr);
    KCG_LAUNCHED(dst);
    size_t tb = 0;
    KCG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, dst.und_off.p, n + 1, dst.stream));
    KCG_CUDA(cub::DeviceScan::ExclusiveSum(cub_temp(dst, tb), tb, cnt, dst.und_off.p, n + 1,
                                           dst.stream));
    uint64_t two_m = 0;
    KCG_CUDA(cudaMemcpyAsync(&two_m, dst.und_off.p + n, 8, cudaMemcpyDeviceToHost, dst.stream));
    dst.sync();
    dst.m = two_m / 2;
    dst.und_adj.ensure(std::max<uint64_t>(two_m, 1), &dst.alloc);
    mono_kernel<true><<<blocks_for(uint64_t(n) * 32, 256), 256, 0, dst.stream>>>(
        src.und_off.p, src.und_adj.p, color, n, nullptr, dst.und_off.p, dst.und_adj.p);
    KCG_LAUNCHED(dst);
  }
  dst.deg.ensure(n, &dst.alloc);
  if (n) {
    degree_kernel2<<<blocks_for(n, 256), 256, 0, dst.stream>>>(dst.und_off.p, n, dst.deg.p);
    KCG_LAUNCHED(dst);
  }
  dst.has_und = true;
  dst.has_rank = dst.has_dag = dst.has_rdag = false;
  dst.mark(1);
  dst.times.upload_ms = dst.elapsed(0, 1);
}

}  // namespace kcg
