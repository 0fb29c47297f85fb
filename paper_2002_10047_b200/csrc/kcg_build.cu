// Input construction on the device:
// Graph::from_edges normalisation (proj/src/graph.cpp:11-41) and the R-MAT
// generator of the benchmark configs, so a whole pipeline -- samples ->
// CSR -> ranking -> DAG -> counts -> peeling -- stays in HBM.
//
//  canon   one thread per input edge: key = (min << 32 | max), self-loops
//          -> ~0 (sorts last), endpoint >= n -> error flag
//  sort    CUB radix sort of the keys on the 32 + ceil(log2 n) live bits
//  unique  CUB DeviceSelect::Unique; the ~0 tail (loops) is dropped
//  count   per vertex: edges where it is the smaller endpoint (hi) and the
//          larger one (lo), atomics; CSR offsets = scan(lo + hi)
//  fill    forward-sorted keys write the upper slice of u in order; a
//          STABLE radix sort on the v bits only turns the same list into
//          (v, u ascending) order, which writes the lower slice of v.  The
//          lower slice precedes the upper one and both ascend, exactly the
//          reference's cursor fill order.
//
// The R-MAT kernel reproduces the host generator (gen/kcgen.cpp
// kcgen_rmat) bit for bit: same counter-based splitmix64 stream and the
// same integer quadrant thresholds, so device-built and host-built configs
// have identical digests.
#include <cub/cub.cuh>
#include <thrust/iterator/transform_iterator.h>

#include <algorithm>
#include <vector>

#include "kcg_internal.cuh"

namespace kcg {
namespace {

typedef unsigned long long ull;
constexpr ull LOOP = ~0ull;

__device__ __forceinline__ ull fmix(ull z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
constexpr ull kGolden = 0x9E3779B97F4A7C15ull;

ull host_fmix(ull z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
ull stream_key(ull seed, ull stream) {
  return host_fmix(seed * 0xD6E8FEB86659FD93ull + host_fmix(stream + kGolden));
}

__global__ void canon_kernel(const uint32_t* __restrict__ us, const uint32_t* __restrict__ vs,
                             uint64_t cnt, uint32_t n, ull* __restrict__ keys,
                             ull* __restrict__ bad) {
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < cnt;
       i += uint64_t(gridDim.x) * blockDim.x) {
    uint32_t u = us[i], v = vs[i];
    if (u >= n || v >= n) {
      atomicAdd(bad, 1ull);
      keys[i] = LOOP;
      continue;
    }
    if (u > v) {
      const uint32_t t = u;
      u = v;
      v = t;
    }
    keys[i] = u == v ? LOOP : (ull(u) << 32 | v);
  }
}

// R-MAT samples (kcgen_rmat): sample e uses draws e*scale .. e*scale+scale-1
__global__ void rmat_kernel(int scale, uint64_t samples, ull key, ull t1, ull t2, ull t3,
                            const uint32_t* __restrict__ perm, ull* __restrict__ keys) {
  for (uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < samples;
       e += uint64_t(gridDim.x) * blockDim.x) {
    uint32_t u = 0, v = 0;
    const ull base = e * ull(scale);
    for (int l = 0; l < scale; l++) {
      const ull r = fmix(key + (base + l + 1) * kGolden) >> 11;
      const uint32_t bit = 1u << (scale - 1 - l);
      if (r < t1) {
      } else if (r < t2) {
        v |= bit;
      } else if (r < t3) {
        u |= bit;
      } else {
        u |= bit;
        v |= bit;
      }
    }
    if (perm) {
      u = perm[u];
      v = perm[v];
    }
    if (u > v) {
      const uint32_t t = u;
      u = v;
      v = t;
    }
    keys[e] = u == v ? LOOP : (ull(u) << 32 | v);
  }
}

__global__ void degree_from_off_kernel(const uint64_t* __restrict__ off, uint32_t n,
                                       uint32_t* __restrict__ deg) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    deg[v] = uint32_t(off[v + 1] - off[v]);
}

__global__ void endpoint_count_kernel(const ull* __restrict__ keys, uint64_t m,
                                      uint32_t* __restrict__ hi, uint32_t* __restrict__ lo) {
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < m;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const ull k = keys[i];
    atomicAdd(&hi[k >> 32], 1u);
    atomicAdd(&lo[uint32_t(k)], 1u);
  }
}

__global__ void degree_sum_kernel(const uint32_t* __restrict__ hi, const uint32_t* __restrict__ lo,
                                  uint32_t n, uint64_t* __restrict__ deg) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v <= n; v += gridDim.x * blockDim.x)
    deg[v] = v < n ? uint64_t(hi[v]) + lo[v] : 0;
}

// forward order (u asc, v asc): entry i is the (i - first_u)-th upper
// neighbour of u; first_u = hi_start[u]
__global__ void fill_upper_kernel(const ull* __restrict__ keys, uint64_t m,
                                  const uint64_t* __restrict__ off,
                                  const uint32_t* __restrict__ lo,
                                  const uint64_t* __restrict__ hi_start,
                                  uint32_t* __restrict__ adj) {
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < m;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const ull k = keys[i];
    const uint32_t u = uint32_t(k >> 32);
    adj[off[u] + lo[u] + (i - hi_start[u])] = uint32_t(k);
  }
}

// (v asc, u asc) order: entry j is the (j - first_v)-th lower neighbour of v
__global__ void fill_lower_kernel(const ull* __restrict__ keys, uint64_t m,
                                  const uint64_t* __restrict__ off,
                                  const uint64_t* __restrict__ lo_start,
                                  uint32_t* __restrict__ adj) {
  for (uint64_t j = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < m;
       j += uint64_t(gridDim.x) * blockDim.x) {
    const ull k = keys[j];
    const uint32_t v = uint32_t(k);
    adj[off[v] + (j - lo_start[v])] = uint32_t(k >> 32);
  }
}

int bits_for(uint64_t x) {
  int b = 0;
  while ((uint64_t(1) << b) < x) b++;
  return b;
}

template <class T>
T fetch(Graph& g, const T* d) {
  T h;
  KCG_CUDA(cudaMemcpyAsync(&h, d, sizeof(T), cudaMemcpyDeviceToHost, g.stream));
  g.sync();
  return h;
}

struct Widen {
  __device__ uint64_t operator()(uint32_t x) const { return x; }
};

// keys[0..cnt) (u < v, LOOP for dropped samples) -> g.und_off / g.und_adj
// and g.m.  `alt` is a second key buffer of cnt entries; both are consumed.
void csr_from_keys(Graph& g, ull* keys, ull* alt, uint64_t cnt) {
  const uint32_t n = g.n;
  const int vb = std::max(1, bits_for(n));
  ull* cnts = g.counters.ensure(16, &g.alloc);
  uint64_t m = 0;
  size_t tb = 0;
  if (cnt) {
    // valid keys live in bits [0, 32 + vb); LOOP has all of them set and
    // sorts last (v <= 2^32 - 2 < LOOP's low word)
    const int end_bit = std::min(64, 32 + vb);
    KCG_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, keys, alt, cnt, 0, end_bit, g.stream));
    KCG_CUDA(cub::DeviceRadixSort::SortKeys(cub_temp(g, tb), tb, keys, alt, cnt, 0, end_bit,
                                            g.stream));
    KCG_CUDA(cub::DeviceSelect::Unique(nullptr, tb, alt, keys, cnts, cnt, g.stream));
    KCG_CUDA(cub::DeviceSelect::Unique(cub_temp(g, tb), tb, alt, keys, cnts, cnt, g.stream));
    m = fetch(g, cnts);
    if (m && fetch(g, keys + (m - 1)) == LOOP) m--;
  }
  g.m = m;
  auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
  const size_t b32 = al((size_t(n) + 1) * 4), b64 = al((size_t(n) + 1) * 8);
  unsigned char* ws = g.scratch2.ensure(2 * b32 + 3 * b64, &g.alloc);
  uint32_t* hi = reinterpret_cast<uint32_t*>(ws);
  uint32_t* lo = reinterpret_cast<uint32_t*>(ws + b32);
  uint64_t* deg = reinterpret_cast<uint64_t*>(ws + 2 * b32);
  uint64_t* hi_start = reinterpret_cast<uint64_t*>(ws + 2 * b32 + b64);
  uint64_t* lo_start = reinterpret_cast<uint64_t*>(ws + 2 * b32 + 2 * b64);
  KCG_CUDA(cudaMemsetAsync(hi, 0, (size_t(n) + 1) * 4, g.stream));
  KCG_CUDA(cudaMemsetAsync(lo, 0, (size_t(n) + 1) * 4, g.stream));
  g.und_off.ensure(size_t(n) + 1, &g.alloc);
  g.und_adj.ensure(std::max<uint64_t>(2 * m, 1), &g.alloc);
  if (m) {
    endpoint_count_kernel<<<blocks_for(m, 256), 256, 0, g.stream>>>(keys, m, hi, lo);
    KCG_LAUNCHED(g);
  }
  degree_sum_kernel<<<blocks_for(uint64_t(n) + 1, 256), 256, 0, g.stream>>>(hi, lo, n, deg);
  KCG_LAUNCHED(g);
  KCG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, deg, g.und_off.p, n + 1, g.stream));
  KCG_CUDA(cub::DeviceScan::ExclusiveSum(cub_temp(g, tb), tb, deg, g.und_off.p, n + 1,
                                         g.stream));
  if (m) {
    // run starts of the forward (by u) and lower (by v) orders
    auto scan_u32 = [&](const uint32_t* c, uint64_t* out) {
      auto it = thrust::make_transform_iterator(c, Widen());
      size_t t2 = 0;
      KCG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, t2, it, out, n + 1, g.stream));
      KCG_CUDA(cub::DeviceScan::ExclusiveSum(cub_temp(g, t2), t2, it, out, n + 1, g.stream));
    };
    scan_u32(hi, hi_start);
    scan_u32(lo, lo_start);
    fill_upper_kernel<<<blocks_for(m, 256), 256, 0, g.stream>>>(keys, m, g.und_off.p, lo,
                                                                hi_start, g.und_adj.p);
    KCG_LAUNCHED(g);
    // stable sort on the v bits only: (u asc, v asc) -> (v asc, u asc)
    KCG_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, keys, alt, m, 0, vb, g.stream));
    KCG_CUDA(cub::DeviceRadixSort::SortKeys(cub_temp(g, tb), tb, keys, alt, m, 0, vb,
                                            g.stream));
    fill_lower_kernel<<<blocks_for(m, 256), 256, 0, g.stream>>>(alt, m, g.und_off.p, lo_start,
                                                                g.und_adj.p);
    KCG_LAUNCHED(g);
  }
}

void finish(Graph& g) {
  g.deg.ensure(g.n, &g.alloc);
  if (g.n) {
    const uint32_t n = g.n;
    // degree from the offsets (same as kcg_graph_create's finish_und)
    degree_from_off_kernel<<<blocks_for(n, 256), 256, 0, g.stream>>>(g.und_off.p, n, g.deg.p);
    KCG_LAUNCHED(g);
  }
  g.has_und = true;
  g.has_rank = g.has_dag = g.has_rdag = false;
}

}  // namespace

void build_from_edges(Graph& g, uint32_t n, const uint32_t* us, const uint32_t* vs,
                      uint64_t cnt) {
  g.n = n;
  g.mark(0);
  DevBuf<ull> keys, alt;
  keys.ensure(std::max<uint64_t>(cnt, 1), &g.alloc);
  alt.ensure(std::max<uint64_t>(cnt, 1), &g.alloc);
  if (cnt) {
    // stage the two endpoint arrays in the key buffers' storage
    uint32_t* d_us = reinterpret_cast<uint32_t*>(alt.p);
    uint32_t* d_vs = d_us + cnt;
    KCG_CUDA(cudaMemcpyAsync(d_us, us, cnt * 4, cudaMemcpyHostToDevice, g.stream));
    KCG_CUDA(cudaMemcpyAsync(d_vs, vs, cnt * 4, cudaMemcpyHostToDevice, g.stream));
    g.times.h2d_bytes += cnt * 8;
    ull* bad = g.counters.ensure(16, &g.alloc) + 8;
    KCG_CUDA(cudaMemsetAsync(bad, 0, 8, g.stream));
    canon_kernel<<<blocks_for(cnt, 256), 256, 0, g.stream>>>(d_us, d_vs, cnt, n, keys.p, bad);
    KCG_LAUNCHED(g);
    if (fetch(g, bad)) fail(KCG_EINVAL, "edge endpoint out of range");
  }
  csr_from_keys(g, keys.p, alt.p, cnt);
  finish(g);
  g.mark(1);
  g.times.upload_ms = g.elapsed(0, 1);
}

void build_rmat(Graph& g, int scale, uint64_t samples, double a, double b, double c,
                uint64_t seed, bool permute) {
  if (scale < 1 || scale > 31) fail(KCG_EINVAL, "scale must be in [1, 31]");
  const uint32_t n = uint32_t(1) << scale;
  g.n = n;
  g.mark(0);
  // integer thresholds on the 53-bit uniform, exactly as kcgen_rmat
  const double two53 = 0x1.0p53;
  const ull t1 = ull(a * two53), t2 = ull((a + b) * two53), t3 = ull((a + b + c) * two53);
  DevBuf<uint32_t> perm;
  if (permute) {
    // seeded Fisher-Yates (inherently sequential; n draws on the host)
    std::vector<uint32_t> p(n);
    for (uint32_t i = 0; i < n; i++) p[i] = i;
    const ull pk = stream_key(seed, 2);
    for (uint32_t i = n - 1; i > 0; i--) {
      const uint32_t j = uint32_t(host_fmix(pk + (ull(i) + 1) * kGolden) % (ull(i) + 1));
      std::swap(p[i], p[j]);
    }
    perm.ensure(n, &g.alloc);
    KCG_CUDA(cudaMemcpyAsync(perm.p, p.data(), size_t(n) * 4, cudaMemcpyHostToDevice,
                             g.stream));
    g.sync();  // p goes out of scope
  }
  DevBuf<ull> keys, alt;
  keys.ensure(std::max<uint64_t>(samples, 1), &g.alloc);
  alt.ensure(std::max<uint64_t>(samples, 1), &g.alloc);
  if (samples) {
    rmat_kernel<<<blocks_for(samples, 256, 148u * 64u), 256, 0, g.stream>>>(
        scale, samples, stream_key(seed, 1), t1, t2, t3, permute ? perm.p : nullptr, keys.p);
    KCG_LAUNCHED(g);
  }
  csr_from_keys(g, keys.p, alt.p, samples);
  finish(g);
  g.mark(1);
  g.times.upload_ms = g.elapsed(0, 1);
}

}  // namespace kcg
