// Internal declarations shared by the kcg translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

#include "kcg.h"

namespace kcg {

// ---- errors ----------------------------------------------------------------
// Internal code throws; the extern "C" layer converts to status codes and
// kcg_last_error().  Matches the reference's exception split
// (std::invalid_argument -> KCG_EINVAL).
struct Error : std::runtime_error {
  int status;
  Error(int s, const std::string& m) : std::runtime_error(m), status(s) {}
};
[[noreturn]] void fail(int status, const std::string& msg);
void set_last_error(const std::string& msg);

#define KCG_CUDA(call)                                                       \
  do {                                                                       \
    cudaError_t e_ = (call);                                                 \
    if (e_ != cudaSuccess) {                                                 \
      (void)cudaGetLastError();                                              \
      ::kcg::fail(e_ == cudaErrorMemoryAllocation ? KCG_ENOMEM : KCG_ERUNTIME, \
                  std::string(#call) + ": " + cudaGetErrorString(e_));       \
    }                                                                        \
  } while (0)
#define KCG_LAUNCH_CHECK() KCG_CUDA(cudaGetLastError())
// after every kernel of this library: error check + launch accounting
#define KCG_LAUNCHED(g)   \
  do {                    \
    KCG_LAUNCH_CHECK();   \
    (g).times.launches++; \
  } while (0)

// ---- device buffers ----------------------------------------------------------
// from the library's own pool (device().pool), else the default pool
cudaError_t alloc_async(void** p, size_t bytes, cudaStream_t s);

// Stream-ordered allocations from the library's memory pool (release
// threshold raised at init), so creating and destroying handles -- the
// end-to-end path of every drop-in call -- reuses memory instead of paying
// cudaMalloc/cudaFree each time.
struct AllocCtx {
  size_t bytes = 0;             // device bytes the handle holds
  cudaStream_t stream = nullptr;
};

template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;           // elements allocated
  AllocCtx* ctx = nullptr;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  void release() {
    if (p) {
      cudaFreeAsync(p, ctx ? ctx->stream : nullptr);
      if (ctx) ctx->bytes -= n * sizeof(T);
    }
    p = nullptr;
    n = 0;
  }
  // grows (never shrinks) to at least `count` elements; contents are lost
  // when it grows
  T* ensure(size_t count, AllocCtx* c = nullptr) {
    if (c) ctx = c;
    if (count <= n && p) return p;
    release();
    const size_t e = count ? count : 1;
    KCG_CUDA(alloc_async(reinterpret_cast<void**>(&p), e * sizeof(T),
                         ctx ? ctx->stream : nullptr));
    n = e;
    if (ctx) ctx->bytes += n * sizeof(T);
    return p;
  }
};

struct PinnedBuf {
  void* p = nullptr;
  size_t bytes = 0;
  ~PinnedBuf() {
    if (p) cudaFreeHost(p);
  }
  void* ensure(size_t b) {
    if (b <= bytes && p) return p;
    if (p) cudaFreeHost(p);
    p = nullptr;
    KCG_CUDA(cudaMallocHost(&p, b ? b : 1));
    bytes = b;
    return p;
  }
};

struct Device {
  int id = 0;
  int sms = 148;
  int smem_optin = 227 * 1024;
  int l2 = 0;
  int major = 0, minor = 0;
  cudaMemPool_t pool = nullptr;  // library-owned, release threshold raised
};
const Device& device();

// ---- the graph handle --------------------------------------------------------
// Whole graph resident in HBM.  Layouts:
//   und_off/und_adj   undirected CSR (u64 offsets, u32 ids), ascending
//   deg               undirected degree (u32)
//   rank/order        rank[v], order[r] (u32)
//   dag_off/dag_adj   id-space DAG, slices ascending by id (== reference)
//   rdag_off/rdag_adj rank-relabelled DAG: vertex r = order[...], targets
//                     are ranks, slices ascending -> every induced
//                     subgraph is upper-triangular in local order
//   pv_rank/pv        per-vertex counts by rank / by id
struct Graph {
  uint32_t n = 0;
  uint64_t m = 0;
  bool has_und = false;
  bool has_rank = false;
  bool has_dag = false;     // id-space DAG valid for current ranking
  bool has_rdag = false;    // relabelled DAG valid for current ranking
  uint64_t max_out = 0;
  AllocCtx alloc;
  cudaStream_t stream = nullptr;

  DevBuf<uint64_t> und_off;
  DevBuf<uint32_t> und_adj;
  DevBuf<uint32_t> deg;
  DevBuf<uint32_t> rank, order;
  DevBuf<uint64_t> dag_off;
  DevBuf<uint32_t> dag_adj;
  DevBuf<uint64_t> rdag_off;
  DevBuf<uint32_t> rdag_adj;
  DevBuf<uint64_t> pv_rank, pv;
  DevBuf<unsigned char> scratch;   // CUB temp + misc
  DevBuf<unsigned char> scratch2;  // per-call work arrays
  DevBuf<unsigned char> scratch3;  // counting work items
  DevBuf<unsigned char> heavy;     // heavy-tier global bitmaps
  DevBuf<unsigned long long> counters;  // small device counters
  PinnedBuf pinned;
  // peeling (kcg_peel.cu): the DAG restricted to the live vertices, swapped
  // in for rdag_* while counting, and the per-round state
  DevBuf<uint64_t> live_off;
  DevBuf<uint32_t> live_adj;
  DevBuf<unsigned char> peel_ws;
  // counting restricted to sources r with src_mask[r] != 0 (rank space);
  // nullptr = every source
  const uint8_t* src_mask = nullptr;

  kcg_times times{};
  kcg_count_stats stats{};
  cudaEvent_t ev[8] = {};
  // auxiliary streams for concurrent counting launches (fork/join with
  // events against `stream`)
  static constexpr int kAux = 6;
  cudaStream_t aux[kAux] = {};
  cudaEvent_t fork_ev = nullptr;
  cudaEvent_t join_ev[kAux] = {};

  Graph();
  ~Graph();
  void release_all();
  void sync();
  // event-timed region on the handle's stream
  void mark(int i) { KCG_CUDA(cudaEventRecord(ev[i], stream)); }
  double elapsed(int a, int b);
};

// phases (kcg_rank.cu, kcg_direct.cu, kcg_count.cu)
uint64_t estimate_arboricity(Graph& g, double eps);
uint64_t rank_graph(Graph& g, int strategy, double eps, uint64_t alpha_hat,
                    uint64_t* alpha_out);  // returns rounds
void build_dag(Graph& g, bool want_id_dag);
void relabel_from_dag(Graph& g);  // rdag from an adopted id-space DAG
// cliques whose lowest-ranked vertex r lies in [r_lo, r_hi)
uint64_t count_cliques(Graph& g, int k, bool want_pv, uint32_t r_lo = 0,
                       uint32_t r_hi = 0xffffffffu);
// work-balanced contiguous source ranges (bounds[nparts + 1], rank space)
void partition_plan(Graph& g, int k, uint32_t nparts, uint32_t* bounds);
// sum_w indeg(w) * outdeg(w) of the DAG (the staging term of B_alg)
uint64_t dag_work(Graph& g);

// input construction on the device (kcg_build.cu)
void build_from_edges(Graph& g, uint32_t n, const uint32_t* us, const uint32_t* vs,
                      uint64_t cnt);
void build_rmat(Graph& g, int scale, uint64_t samples, double a, double b, double c,
                uint64_t seed, bool permute);

// clique listing (kcg_list.cu); returns the clique count
uint64_t list_cliques(Graph& g, int k, uint64_t batch, kcg_clique_fn fn, void* user);

// colour sparsification (kcg_sample.cu): dst receives the monochromatic
// subgraph of src
void colorful_sparsify(const Graph& src, Graph& dst, uint64_t colors, uint64_t seed);

// peeling consumers of the per-vertex counts (kcg_peel.cu)
struct UpdateOut {
  uint64_t removed = 0;
  std::vector<uint32_t> changed;
};
UpdateOut update_counts(Graph& g, int k, uint64_t* counts, const uint32_t* batch,
                        uint64_t batch_len, const uint8_t* peeled);
struct PeelOut {
  uint64_t rounds = 0, total = 0, best_round = 0;
  double best_density = 0.0;
  std::vector<uint32_t> dense;
};
PeelOut peel(Graph& g, int k, bool exact, double eps, uint64_t* core_out);

// small helpers
void* cub_temp(Graph& g, size_t bytes);
inline unsigned blocks_for(uint64_t work, unsigned threads, unsigned cap = 148u * 32u) {
  uint64_t b = (work + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > cap) b = cap;
  return unsigned(b);
}

}  // namespace kcg
