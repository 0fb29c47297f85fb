// extern "C" surface of libkcg.so (include/kcg.h): handle lifecycle,
// transfers, status-code mapping.  The compute phases live in
// kcg_rank.cu, kcg_direct.cu and kcg_count.cu.
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <vector>

#include "kcg_internal.cuh"

namespace kcg {

namespace {
thread_local std::string g_last_error;
std::once_flag g_dev_once;
Device g_dev;
bool g_dev_ok = false;
std::string g_dev_err;

__global__ void degree_kernel(const uint64_t* __restrict__ off, uint32_t n,
                              uint32_t* __restrict__ deg) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += gridDim.x * blockDim.x)
    deg[v] = uint32_t(off[v + 1] - off[v]);
}

// Validates a bijection: seen[r] counts hits; any r >= n or a repeat
// raises the flag.
__global__ void bijection_kernel(const uint32_t* __restrict__ rank, uint32_t n,
                                 uint32_t* __restrict__ seen,
                                 uint32_t* __restrict__ order,
                                 unsigned long long* __restrict__ bad) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += gridDim.x * blockDim.x) {
    uint32_t r = rank[v];
    if (r >= n || atomicAdd(&seen[r], 1u) != 0) {
      atomicAdd(bad, 1ull);
    } else {
      order[r] = v;
    }
  }
}

}  // namespace

void fail(int status, const std::string& msg) { throw Error(status, msg); }

cudaError_t alloc_async(void** p, size_t bytes, cudaStream_t s) {
  const Device& d = device();
  if (d.pool) return cudaMallocFromPoolAsync(p, bytes, d.pool, s);
  return cudaMallocAsync(p, bytes, s);
}
void set_last_error(const std::string& msg) { g_last_error = msg; }

const Device& device() {
  std::call_once(g_dev_once, [] {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) {
      g_dev_err = std::string("no CUDA device: ") + cudaGetErrorString(e);
      (void)cudaGetLastError();
      return;
    }
    cudaDeviceProp p;
    e = cudaGetDeviceProperties(&p, dev);
    if (e != cudaSuccess) {
      g_dev_err = cudaGetErrorString(e);
      (void)cudaGetLastError();
      return;
    }
    g_dev.id = dev;
    g_dev.sms = p.multiProcessorCount;
    g_dev.smem_optin = int(p.sharedMemPerBlockOptin);
    g_dev.l2 = p.l2CacheSize;
    g_dev.major = p.major;
    g_dev.minor = p.minor;
    // a library-owned pool that keeps freed memory cached (handles come and
    // go on every drop-in call); the host application's default pool is
    // left as it was
    cudaMemPoolProps pp{};
    pp.allocType = cudaMemAllocationTypePinned;
    pp.handleTypes = cudaMemHandleTypeNone;
    pp.location.type = cudaMemLocationTypeDevice;
    pp.location.id = dev;
    if (cudaMemPoolCreate(&g_dev.pool, &pp) == cudaSuccess) {
      uint64_t thr = ~0ull;
      cudaMemPoolSetAttribute(g_dev.pool, cudaMemPoolAttrReleaseThreshold, &thr);
    } else {
      g_dev.pool = nullptr;
    }
    (void)cudaGetLastError();
    if (p.major != 10) {
      g_dev_err = "libkcg is built for sm_100a (B200); found compute capability " +
                  std::to_string(p.major) + "." + std::to_string(p.minor);
      return;
    }
    g_dev_ok = true;
  });
  if (!g_dev_ok) fail(KCG_ERUNTIME, g_dev_err);
  return g_dev;
}

// Streams and events of finished handles are kept for the next one: the
// drop-in and e2e paths create a handle per call, and creating 7 streams
// and 15 events each time cost ~0.3 ms per call.
namespace {
struct StreamSet {
  cudaStream_t stream;
  cudaStream_t aux[Graph::kAux];
  cudaEvent_t ev[8];
  cudaEvent_t fork_ev;
  cudaEvent_t join_ev[Graph::kAux];
};
std::mutex g_sets_mu;
std::vector<StreamSet> g_sets;
}  // namespace

Graph::Graph() {
  device();
  {
    std::lock_guard<std::mutex> lk(g_sets_mu);
    if (!g_sets.empty()) {
      const StreamSet ss = g_sets.back();
      g_sets.pop_back();
      stream = ss.stream;
      for (int i = 0; i < kAux; i++) aux[i] = ss.aux[i], join_ev[i] = ss.join_ev[i];
      for (int i = 0; i < 8; i++) ev[i] = ss.ev[i];
      fork_ev = ss.fork_ev;
      alloc.stream = stream;
      return;
    }
  }
  KCG_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
  alloc.stream = stream;
  for (auto& e : ev) KCG_CUDA(cudaEventCreate(&e));
  for (auto& s : aux) KCG_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  KCG_CUDA(cudaEventCreateWithFlags(&fork_ev, cudaEventDisableTiming));
  for (auto& e : join_ev) KCG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
}

void Graph::release_all() {
  und_off.release();
  und_adj.release();
  deg.release();
  rank.release();
  order.release();
  dag_off.release();
  dag_adj.release();
  rdag_off.release();
  rdag_adj.release();
  pv_rank.release();
  pv.release();
  scratch.release();
  scratch2.release();
  scratch3.release();
  heavy.release();
  counters.release();
  live_off.release();
  live_adj.release();
  peel_ws.release();
}

Graph::~Graph() {
  for (auto& s : aux)
    if (s) cudaStreamSynchronize(s);
  if (stream) cudaStreamSynchronize(stream);
  release_all();
  if (stream) cudaStreamSynchronize(stream);
  for (auto& s : aux)
    if (s) cudaStreamSynchronize(s);
  bool complete = stream && fork_ev;
  for (int i = 0; i < kAux; i++) complete = complete && aux[i] && join_ev[i];
  for (int i = 0; i < 8; i++) complete = complete && ev[i];
  if (complete && cudaGetLastError() == cudaSuccess) {
    StreamSet ss;
    ss.stream = stream;
    for (int i = 0; i < kAux; i++) ss.aux[i] = aux[i], ss.join_ev[i] = join_ev[i];
    for (int i = 0; i < 8; i++) ss.ev[i] = ev[i];
    ss.fork_ev = fork_ev;
    std::lock_guard<std::mutex> lk(g_sets_mu);
    g_sets.push_back(ss);
    return;
  }
  for (auto& e : ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : join_ev)
    if (e) cudaEventDestroy(e);
  if (fork_ev) cudaEventDestroy(fork_ev);
  for (auto& s : aux)
    if (s) cudaStreamDestroy(s);
  if (stream) cudaStreamDestroy(stream);
}

void Graph::sync() { KCG_CUDA(cudaStreamSynchronize(stream)); }

double Graph::elapsed(int a, int b) {
  float ms = 0;
  KCG_CUDA(cudaEventSynchronize(ev[b]));
  KCG_CUDA(cudaEventElapsedTime(&ms, ev[a], ev[b]));
  return ms;
}

void* cub_temp(Graph& g, size_t bytes) { return g.scratch.ensure(bytes, &g.alloc); }

namespace {

template <class F>
int guarded(F&& f) {
  try {
    f();
    return KCG_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.status;
  } catch (const std::bad_alloc&) {
    set_last_error("host allocation failed");
    return KCG_ENOMEM;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return KCG_ERUNTIME;
  }
}

Graph* G(kcg_graph* h) {
  if (!h) fail(KCG_EINVAL, "null kcg_graph handle");
  return reinterpret_cast<Graph*>(h);
}
const Graph* G(const kcg_graph* h) {
  if (!h) fail(KCG_EINVAL, "null kcg_graph handle");
  return reinterpret_cast<const Graph*>(h);
}

// Large transfers between the device and PAGEABLE host memory (the drop-in
// API's std::vectors) can pin the host range for the duration of the copy
// (cudaHostRegister) so that it runs as one direct DMA instead of the
// driver's staged pageable path.  Off by default: on the B200 box pinning and
// unpinning cost more than they save (api_bench, config 2: warm sequence
// 41.3 ms registered vs 27.1 ms pageable; config 5: 1962 vs 1581 ms).
// KCG_REGISTER=1 turns it on; memory the caller already pinned is used as is.
bool register_host() {
  static const bool on = [] {
    const char* e = getenv("KCG_REGISTER");
    return e && e[0] == '1';
  }();
  return on;
}
constexpr size_t kRegisterMin = size_t(8) << 20;

bool is_pinned(const void* p) {
  cudaPointerAttributes attr;
  const bool pinned = cudaPointerGetAttributes(&attr, p) == cudaSuccess &&
                      attr.type == cudaMemoryTypeHost;
  (void)cudaGetLastError();
  return pinned;
}

void transfer(Graph& g, void* dst, const void* src, size_t bytes, cudaMemcpyKind kind) {
  void* host = kind == cudaMemcpyHostToDevice ? const_cast<void*>(src) : dst;
  if (bytes >= kRegisterMin && register_host() && !is_pinned(host)) {
    const unsigned flags = kind == cudaMemcpyHostToDevice ? cudaHostRegisterReadOnly
                                                          : cudaHostRegisterDefault;
    if (cudaHostRegister(host, bytes, flags) == cudaSuccess) {
      const cudaError_t e = cudaMemcpyAsync(dst, src, bytes, kind, g.stream);
      const cudaError_t s = e == cudaSuccess ? cudaStreamSynchronize(g.stream) : e;
      cudaHostUnregister(host);
      KCG_CUDA(s);
      return;
    }
    (void)cudaGetLastError();  // not registrable: the staged copy below
  }
  KCG_CUDA(cudaMemcpyAsync(dst, src, bytes, kind, g.stream));
}

// Stream-ordered host <-> device copies on the handle's stream (a pageable
// source is staged or registered before the call returns).
void upload(Graph& g, void* dst, const void* src, size_t bytes) {
  if (!bytes) return;
  transfer(g, dst, src, bytes, cudaMemcpyHostToDevice);
  g.times.h2d_bytes += bytes;
}

void download(Graph& g, void* dst, const void* src, size_t bytes) {
  if (!bytes) return;
  transfer(g, dst, src, bytes, cudaMemcpyDeviceToHost);
  g.times.d2h_bytes += bytes;
}

void finish_und(Graph& g) {
  g.deg.ensure(g.n, &g.alloc);
  if (g.n)
    degree_kernel<<<blocks_for(g.n, 256), 256, 0, g.stream>>>(g.und_off.p, g.n, g.deg.p);
  KCG_LAUNCHED(g);
  g.has_und = true;
}

void install_rank_device(Graph& g) {
  // rank[] already on device: validate and build order[]
  uint32_t* seen = reinterpret_cast<uint32_t*>(g.scratch2.ensure(size_t(g.n) * 4 + 8, &g.alloc));
  g.counters.ensure(4, &g.alloc);
  KCG_CUDA(cudaMemsetAsync(seen, 0, size_t(g.n) * 4, g.stream));
  KCG_CUDA(cudaMemsetAsync(g.counters.p, 0, 8, g.stream));
  g.order.ensure(g.n, &g.alloc);
  if (g.n)
    bijection_kernel<<<blocks_for(g.n, 256), 256, 0, g.stream>>>(g.rank.p, g.n, seen,
                                                                   g.order.p, g.counters.p);
  KCG_LAUNCHED(g);
  unsigned long long bad = 0;
  KCG_CUDA(cudaMemcpyAsync(&bad, g.counters.p, 8, cudaMemcpyDeviceToHost, g.stream));
  g.sync();
  if (bad) fail(KCG_EINVAL, "ranking is not a bijection");
  g.has_rank = true;
  g.has_dag = g.has_rdag = false;
}

int count_range_impl(kcg_graph* h, int k, bool plan, uint32_t part, uint32_t nparts,
                     uint32_t r_lo, uint32_t r_hi, uint64_t* total, uint64_t* per_vertex) {
  return guarded([&] {
    Graph& g = *G(h);
    if (k < 2) fail(KCG_EINVAL, "k must be at least 2");
    if (plan && (nparts == 0 || part >= nparts)) fail(KCG_EINVAL, "part must be < nparts");
    if (!plan && r_lo > r_hi) fail(KCG_EINVAL, "source range must have r_lo <= r_hi");
    if (!g.has_rdag) {
      if (!g.has_rank) fail(KCG_EINVAL, "no DAG: call kcg_rank/kcg_direct first");
      build_dag(g, false);
    }
    if (plan) {
      std::vector<uint32_t> b(size_t(nparts) + 1);
      partition_plan(g, k, nparts, b.data());
      r_lo = b[part];
      r_hi = b[part + 1];
    }
    g.times.d2h_bytes = 0;
    uint64_t t = count_cliques(g, k, per_vertex != nullptr, r_lo, r_hi);
    if (per_vertex) {
      g.mark(4);
      download(g, per_vertex, g.pv.p, size_t(g.n) * 8);
      g.mark(5);
      g.sync();
      g.times.download_ms = g.elapsed(4, 5);
    }
    if (total) *total = t;
  });
}
}  // namespace
}  // namespace kcg

using namespace kcg;

extern "C" {

const char* kcg_last_error(void) { return g_last_error.c_str(); }
const char* kcg_version(void) { return "kcg 0.1 sm_100a"; }

int kcg_device_info(int* sm_count, int* smem_optin_bytes, int* l2_bytes, int* cc_major,
                    int* cc_minor) {
  return guarded([&] {
    const Device& d = device();
    if (sm_count) *sm_count = d.sms;
    if (smem_optin_bytes) *smem_optin_bytes = d.smem_optin;
    if (l2_bytes) *l2_bytes = d.l2;
    if (cc_major) *cc_major = d.major;
    if (cc_minor) *cc_minor = d.minor;
  });
}

int kcg_graph_create(uint32_t n, const uint64_t* offsets, const uint32_t* adj,
                     kcg_graph** out) {
  return guarded([&] {
    if (!out) fail(KCG_EINVAL, "out is null");
    *out = nullptr;
    if (!offsets) fail(KCG_EINVAL, "offsets is null");
    if (offsets[0] != 0) fail(KCG_EINVAL, "offsets[0] != 0");
    uint64_t two_m = offsets[n];
    if (two_m % 2) fail(KCG_EINVAL, "adjacency is not symmetric (odd length)");
    if (two_m && !adj) fail(KCG_EINVAL, "adj is null");
    auto* g = new Graph();
    try {
      g->n = n;
      g->m = two_m / 2;
      g->times = kcg_times{};
      g->mark(0);
      g->und_off.ensure(size_t(n) + 1, &g->alloc);
      g->und_adj.ensure(two_m, &g->alloc);
      upload(*g, g->und_off.p, offsets, (size_t(n) + 1) * 8);
      upload(*g, g->und_adj.p, adj, two_m * 4);
      finish_und(*g);
      g->mark(1);
      g->times.upload_ms = g->elapsed(0, 1);
    } catch (...) {
      delete g;
      throw;
    }
    *out = reinterpret_cast<kcg_graph*>(g);
  });
}

int kcg_graph_create_device(uint32_t n, uint64_t m, const uint64_t* d_offsets,
                            const uint32_t* d_adj, kcg_graph** out) {
  return guarded([&] {
    if (!out) fail(KCG_EINVAL, "out is null");
    *out = nullptr;
    auto* g = new Graph();
    try {
      g->n = n;
      g->m = m;
      g->und_off.ensure(size_t(n) + 1, &g->alloc);
      g->und_adj.ensure(2 * m, &g->alloc);
      KCG_CUDA(cudaMemcpyAsync(g->und_off.p, d_offsets, (size_t(n) + 1) * 8,
                               cudaMemcpyDeviceToDevice, g->stream));
      if (m)
        KCG_CUDA(cudaMemcpyAsync(g->und_adj.p, d_adj, 2 * m * 4, cudaMemcpyDeviceToDevice,
                                 g->stream));
      finish_und(*g);
      g->sync();
    } catch (...) {
      delete g;
      throw;
    }
    *out = reinterpret_cast<kcg_graph*>(g);
  });
}

int kcg_dag_create(uint32_t n, const uint64_t* out_offsets, const uint32_t* out_targets,
                   const uint32_t* rank, kcg_graph** out) {
  return guarded([&] {
    if (!out) fail(KCG_EINVAL, "out is null");
    *out = nullptr;
    if (!out_offsets) fail(KCG_EINVAL, "out_offsets is null");
    if (n && !rank) fail(KCG_EINVAL, "rank is null");
    uint64_t m = out_offsets[n];
    if (m && !out_targets) fail(KCG_EINVAL, "out_targets is null");
    auto* g = new Graph();
    try {
      g->n = n;
      g->m = m;
      g->times = kcg_times{};
      g->mark(0);
      g->dag_off.ensure(size_t(n) + 1, &g->alloc);
      g->dag_adj.ensure(m, &g->alloc);
      g->rank.ensure(n, &g->alloc);
      upload(*g, g->dag_off.p, out_offsets, (size_t(n) + 1) * 8);
      upload(*g, g->dag_adj.p, out_targets, m * 4);
      upload(*g, g->rank.p, rank, size_t(n) * 4);
      g->mark(1);
      g->times.upload_ms = g->elapsed(0, 1);
      install_rank_device(*g);
      g->has_dag = true;
      relabel_from_dag(*g);
    } catch (...) {
      delete g;
      throw;
    }
    *out = reinterpret_cast<kcg_graph*>(g);
  });
}

int kcg_graph_from_edges(uint32_t n, const uint32_t* us, const uint32_t* vs, uint64_t count,
                         kcg_graph** out) {
  return guarded([&] {
    if (!out) fail(KCG_EINVAL, "out is null");
    *out = nullptr;
    if (count && (!us || !vs)) fail(KCG_EINVAL, "edge arrays are null");
    auto* g = new Graph();
    try {
      g->times = kcg_times{};
      build_from_edges(*g, n, us, vs, count);
    } catch (...) {
      delete g;
      throw;
    }
    *out = reinterpret_cast<kcg_graph*>(g);
  });
}

int kcg_graph_rmat(int scale, uint64_t samples, double a, double b, double c, uint64_t seed,
                   int permute, kcg_graph** out) {
  return guarded([&] {
    if (!out) fail(KCG_EINVAL, "out is null");
    *out = nullptr;
    auto* g = new Graph();
    try {
      g->times = kcg_times{};
      build_rmat(*g, scale, samples, a, b, c, seed, permute != 0);
    } catch (...) {
      delete g;
      throw;
    }
    *out = reinterpret_cast<kcg_graph*>(g);
  });
}

int kcg_graph_csr(kcg_graph* h, uint64_t* offsets, uint32_t* adj) {
  return guarded([&] {
    Graph& g = *G(h);
    if (!g.has_und) fail(KCG_EINVAL, "handle holds no undirected graph");
    if (offsets) download(g, offsets, g.und_off.p, (size_t(g.n) + 1) * 8);
    if (adj) download(g, adj, g.und_adj.p, 2 * g.m * 4);
    g.sync();
  });
}

void kcg_graph_destroy(kcg_graph* h) {
  try {
    delete reinterpret_cast<Graph*>(h);
  } catch (...) {
  }
}

uint32_t kcg_num_vertices(const kcg_graph* h) {
  return h ? reinterpret_cast<const Graph*>(h)->n : 0;
}
uint64_t kcg_num_edges(const kcg_graph* h) {
  return h ? reinterpret_cast<const Graph*>(h)->m : 0;
}

int kcg_rank(kcg_graph* h, int strategy, double eps, uint64_t alpha_hat, uint32_t* rank_out,
             uint64_t* rounds_out, uint64_t* alpha_out) {
  return guarded([&] {
    Graph& g = *G(h);
    if (!g.has_und) fail(KCG_EINVAL, "handle holds no undirected graph");
    g.times.d2h_bytes = 0;
    uint64_t rounds = rank_graph(g, strategy, eps, alpha_hat, alpha_out);
    g.has_rank = true;
    g.has_dag = g.has_rdag = false;
    if (rank_out) {
      g.mark(4);
      download(g, rank_out, g.rank.p, size_t(g.n) * 4);
      g.mark(5);
      g.sync();
      g.times.download_ms = g.elapsed(4, 5);
    }
    if (rounds_out) *rounds_out = rounds;
  });
}

int kcg_estimate_arboricity(kcg_graph* h, double eps, uint64_t* out) {
  return guarded([&] {
    Graph& g = *G(h);
    if (!g.has_und) fail(KCG_EINVAL, "handle holds no undirected graph");
    uint64_t a = estimate_arboricity(g, eps);
    if (out) *out = a;
  });
}

int kcg_set_ranking(kcg_graph* h, const uint32_t* rank, uint32_t len) {
  return guarded([&] {
    Graph& g = *G(h);
    if (len != g.n) fail(KCG_EINVAL, "ranking size does not match graph");
    if (g.n && !rank) fail(KCG_EINVAL, "rank is null");
    g.rank.ensure(g.n, &g.alloc);
    upload(g, g.rank.p, rank, size_t(g.n) * 4);
    install_rank_device(g);
  });
}

int kcg_direct(kcg_graph* h, uint64_t* out_offsets, uint32_t* out_targets,
               uint64_t* max_out_degree) {
  return guarded([&] {
    Graph& g = *G(h);
    if (!g.has_rank) fail(KCG_EINVAL, "no ranking installed");
    if (!g.has_und && !g.has_dag) fail(KCG_EINVAL, "handle holds no graph");
    g.times.d2h_bytes = 0;
    bool want_id = out_offsets || out_targets;
    if (!g.has_rdag || (want_id && !g.has_dag)) build_dag(g, want_id);
    g.mark(4);
    if (out_offsets) download(g, out_offsets, g.dag_off.p, (size_t(g.n) + 1) * 8);
    if (out_targets) download(g, out_targets, g.dag_adj.p, g.m * 4);
    g.mark(5);
    g.sync();
    g.times.download_ms = g.elapsed(4, 5);
    if (max_out_degree) *max_out_degree = g.max_out;
  });
}

int kcg_count(kcg_graph* h, int k, uint64_t* total, uint64_t* per_vertex) {
  return guarded([&] {
    Graph& g = *G(h);
    if (k < 2) fail(KCG_EINVAL, "k must be at least 2");
    if (!g.has_rdag) {
      if (!g.has_rank) fail(KCG_EINVAL, "no DAG: call kcg_rank/kcg_direct first");
      build_dag(g, false);
    }
    g.times.d2h_bytes = 0;
    uint64_t t = count_cliques(g, k, per_vertex != nullptr);
    if (per_vertex) {
      g.mark(4);
      download(g, per_vertex, g.pv.p, size_t(g.n) * 8);
      g.mark(5);
      g.sync();
      g.times.download_ms = g.elapsed(4, 5);
    }
    if (total) *total = t;
  });
}

int kcg_partition_plan(kcg_graph* h, int k, uint32_t nparts, uint32_t* bounds) {
  return guarded([&] {
    Graph& g = *G(h);
    if (k < 2) fail(KCG_EINVAL, "k must be at least 2");
    if (!bounds) fail(KCG_EINVAL, "null bounds");
    if (!g.has_rdag) {
      if (!g.has_rank) fail(KCG_EINVAL, "no DAG: call kcg_rank/kcg_direct first");
      build_dag(g, false);
    }
    partition_plan(g, k, nparts, bounds);
  });
}

int kcg_dag_work(kcg_graph* h, uint64_t* sum_indeg_outdeg) {
  return guarded([&] {
    Graph& g = *G(h);
    if (!sum_indeg_outdeg) fail(KCG_EINVAL, "null out pointer");
    if (!g.has_rdag) {
      if (!g.has_rank) fail(KCG_EINVAL, "no DAG: call kcg_rank/kcg_direct first");
      build_dag(g, false);
    }
    *sum_indeg_outdeg = dag_work(g);
  });
}

int kcg_count_range(kcg_graph* h, int k, uint32_t r_lo, uint32_t r_hi, uint64_t* total,
                    uint64_t* per_vertex) {
  return count_range_impl(h, k, false, 0, 0, r_lo, r_hi, total, per_vertex);
}

int kcg_count_part(kcg_graph* h, int k, uint32_t part, uint32_t nparts, uint64_t* total,
                   uint64_t* per_vertex) {
  return count_range_impl(h, k, true, part, nparts, 0, 0, total, per_vertex);
}

void* kcg_stream(kcg_graph* h) {
  return h ? static_cast<void*>(reinterpret_cast<Graph*>(h)->stream) : nullptr;
}

int kcg_per_vertex_device(kcg_graph* h, const uint64_t** d_per_vertex) {
  return guarded([&] {
    Graph& g = *G(h);
    if (!d_per_vertex) fail(KCG_EINVAL, "null out pointer");
    *d_per_vertex = g.pv.p;
  });
}

int kcg_pipeline(kcg_graph* h, int strategy, double eps, uint64_t alpha_hat, int k,
                 uint64_t* total, uint64_t* per_vertex) {
  return guarded([&] {
    Graph& g = *G(h);
    if (k < 2) fail(KCG_EINVAL, "k must be at least 2");
    if (!g.has_und) fail(KCG_EINVAL, "handle holds no undirected graph");
    g.times.d2h_bytes = 0;
    rank_graph(g, strategy, eps, alpha_hat, nullptr);
    g.has_rank = true;
    g.has_dag = g.has_rdag = false;
    build_dag(g, false);
    uint64_t t = count_cliques(g, k, per_vertex != nullptr);
    if (per_vertex) {
      g.mark(4);
      download(g, per_vertex, g.pv.p, size_t(g.n) * 8);
      g.mark(5);
      g.sync();
      g.times.download_ms = g.elapsed(4, 5);
    }
    if (total) *total = t;
  });
}

int kcg_update_counts(kcg_graph* h, int k, uint64_t* counts, const uint32_t* batch,
                      uint64_t batch_len, const uint8_t* peeled, uint64_t* removed,
                      uint32_t* changed, uint64_t* changed_len) {
  return guarded([&] {
    Graph& g = *G(h);
    g.times.d2h_bytes = 0;
    UpdateOut r = update_counts(g, k, counts, batch, batch_len, peeled);
    if (removed) *removed = r.removed;
    if (changed && !r.changed.empty())
      std::memcpy(changed, r.changed.data(), r.changed.size() * 4);
    if (changed_len) *changed_len = r.changed.size();
  });
}

namespace {
void peel_result(const PeelOut& r, kcg_peel_result* out, uint32_t* dense) {
  if (out) {
    out->rounds = r.rounds;
    out->total_cliques = r.total;
    out->best_density = r.best_density;
    out->best_round = r.best_round;
    out->num_dense = r.dense.size();
  }
  if (dense && !r.dense.empty()) std::memcpy(dense, r.dense.data(), r.dense.size() * 4);
}
}  // namespace

int kcg_peel_exact(kcg_graph* h, int k, kcg_peel_result* out, uint64_t* core,
                   uint32_t* dense_vertices) {
  return guarded([&] {
    Graph& g = *G(h);
    g.times.d2h_bytes = 0;
    peel_result(peel(g, k, true, 0.0, core), out, dense_vertices);
  });
}

int kcg_peel_approx(kcg_graph* h, int k, double eps, kcg_peel_result* out,
                    uint32_t* dense_vertices) {
  return guarded([&] {
    Graph& g = *G(h);
    g.times.d2h_bytes = 0;
    peel_result(peel(g, k, false, eps, nullptr), out, dense_vertices);
  });
}

int kcg_colorful_sparsify(kcg_graph* h, uint64_t colors, uint64_t seed, kcg_graph** out) {
  return guarded([&] {
    if (!out) fail(KCG_EINVAL, "out is null");
    *out = nullptr;
    Graph& g = *G(h);
    if (colors < 1) fail(KCG_EINVAL, "colors must be at least 1");
    auto* d = new Graph();
    try {
      d->times = kcg_times{};
      colorful_sparsify(g, *d, colors, seed);
    } catch (...) {
      delete d;
      throw;
    }
    *out = reinterpret_cast<kcg_graph*>(d);
  });
}

int kcg_approx_count(kcg_graph* h, int k, uint64_t colors, uint64_t seed, int strategy,
                     double eps, uint64_t alpha_hat, kcg_sample_estimate* out) {
  return guarded([&] {
    Graph& g = *G(h);
    if (k < 2) fail(KCG_EINVAL, "k must be at least 2");
    if (colors < 1) fail(KCG_EINVAL, "colors must be at least 1");
    Graph sub;
    colorful_sparsify(g, sub, colors, seed);
    rank_graph(sub, strategy, eps, alpha_hat, nullptr);
    sub.has_rank = true;
    build_dag(sub, false);
    const uint64_t total = count_cliques(sub, k, false);
    g.times.count_ms = sub.times.count_ms;
    g.times.count_kernel_ms = sub.times.count_kernel_ms;
    g.times.launches += sub.times.launches;
    if (out) {
      out->k = k;
      out->colors = colors;
      out->p = 1.0 / double(colors);
      out->sub_count = total;
      out->estimate = double(total) * std::pow(double(colors), k - 1);
      out->seed = seed;
    }
  });
}

int kcg_list_cliques(kcg_graph* h, int k, uint64_t batch, kcg_clique_fn fn, void* user,
                     uint64_t* total) {
  return guarded([&] {
    Graph& g = *G(h);
    g.times.d2h_bytes = 0;
    const uint64_t t = list_cliques(g, k, batch, fn, user);
    if (total) *total = t;
  });
}

int kcg_timings(const kcg_graph* h, kcg_times* out) {
  return guarded([&] {
    if (!out) fail(KCG_EINVAL, "null out pointer");
    *out = G(h)->times;
  });
}

int kcg_last_count_stats(const kcg_graph* h, kcg_count_stats* out) {
  return guarded([&] {
    if (!out) fail(KCG_EINVAL, "null out pointer");
    *out = G(h)->stats;
  });
}

uint64_t kcg_device_bytes(const kcg_graph* h) {
  return h ? reinterpret_cast<const Graph*>(h)->alloc.bytes : 0;
}

int kcg_synchronize(kcg_graph* h) {
  return guarded([&] { G(h)->sync(); });
}

}  // extern "C"
