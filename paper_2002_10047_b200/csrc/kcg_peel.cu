// k-clique peeling on the device: the consumers of the per-vertex counts
// -- update_counts, peel_exact and peel_approx of
// proj/src/peeling.cpp:194-320.
//
// The reference destroys the cliques through each batch vertex with its
// recursion over the filtered neighbourhood of that vertex
// (run_update, peeling.cpp:114-191).  Here one batch update is a
// RESTRICTED RECOUNT with the counting kernels of kcg_count.cu.  With A the
// live vertex set and B the batch:
//
//   NB = live neighbours of B that are not in B,
//   S  = B ∪ N[NB]   (as a rank-space source mask for count_cliques).
//
// Every clique containing a vertex u has its lowest-ranked member in N[u],
// so counting on the DAG restricted to A\B with sources S yields the exact
// per-vertex counts of every u in NB; and every clique touching B is
// sourced in S (it either has a member in NB or lies inside B).  Hence
//
//   d_u     = pv_A[u] - pv_{A\B}[u]          (u in NB; 0 elsewhere)
//   removed = tot_A(S) - tot_{A\B}(S),
//
// which is exactly what the reference's decrements add up to, for any input
// counts (update_counts counts both sides).  The peeling loops keep the
// counts consistent (counts == pv_A, as the reference's loops do), so they
// count A\B only: d_u = counts[u] - pv_{A\B}[u] and
//
//   k * removed = sum_{b in B} counts[b] + sum_{u in NB} d_u.
//
// Round selection is the reference's: peel_exact extracts every live
// vertex holding the minimum count (BucketQueue::extract_min semantics,
// peeling.cpp:79-104), peel_approx every live vertex with
// double(count) <= k (1 + eps) remaining / alive evaluated in IEEE double
// exactly as peeling.cpp:285-291; densities are compared as exact
// fractions (peeling.cpp:196-211).
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include <algorithm>

#include "kcg_internal.cuh"

namespace kcg {
namespace {

typedef unsigned long long ull;
constexpr unsigned FULLW = 0xffffffffu;

__global__ void live_rank_kernel(const uint8_t* __restrict__ live,
                                 const uint32_t* __restrict__ order, uint32_t n,
                                 uint8_t* __restrict__ live_rank) {
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x)
    live_rank[r] = live[order[r]];
}

// One warp per rank r: out-degree of r in the DAG restricted to live
// vertices (0 for a dead r).  cnt has n + 1 entries, cnt[n] = 0.
__global__ void live_deg_kernel(const uint64_t* __restrict__ off, const uint32_t* __restrict__ adj,
                                const uint8_t* __restrict__ lr, uint32_t n,
                                ull* __restrict__ cnt) {
  const uint32_t lane = threadIdx.x & 31;
  for (uint64_t r = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; r <= n;
       r += (uint64_t(gridDim.x) * blockDim.x) >> 5) {
    uint32_t c = 0;
    if (r < n && lr[r]) {
      const uint64_t b = off[r], e = off[r + 1];
      for (uint64_t p0 = b; p0 < e; p0 += 32) {
        const uint64_t p = p0 + lane;
        c += __popc(__ballot_sync(FULLW, p < e && lr[adj[p]]));
      }
    }
    if (lane == 0) cnt[r] = c;
  }
}

// One warp per rank: ordered compaction of the live targets (slices stay
// ascending, so the restricted DAG keeps the topological-order invariant
// the counting kernels rely on).
__global__ void live_fill_kernel(const uint64_t* __restrict__ off, const uint32_t* __restrict__ adj,
                                 const uint8_t* __restrict__ lr, uint32_t n,
                                 const uint64_t* __restrict__ loff, uint32_t* __restrict__ ladj) {
  const uint32_t lane = threadIdx.x & 31;
  for (uint64_t r = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; r < n;
       r += (uint64_t(gridDim.x) * blockDim.x) >> 5) {
    if (!lr[r]) continue;
    const uint64_t b = off[r], e = off[r + 1];
    uint64_t w = loff[r];
    for (uint64_t p0 = b; p0 < e; p0 += 32) {
      const uint64_t p = p0 + lane;
      uint32_t t = 0;
      bool keep = false;
      if (p < e) {
        t = adj[p];
        keep = lr[t] != 0;
      }
      const unsigned bal = __ballot_sync(FULLW, keep);
      if (keep) ladj[w + __popc(bal & ((1u << lane) - 1u))] = t;
      w += __popc(bal);
    }
  }
}

// Flags the batch (in_b, and its ranks in the source mask); bad[0] counts
// members that are out of range or already peeled (peeling.cpp:133-136).
__global__ void batch_mark_kernel(const uint32_t* __restrict__ batch, uint64_t nb, uint32_t n,
                                  const uint8_t* __restrict__ live,
                                  const uint32_t* __restrict__ rank, uint8_t* __restrict__ in_b,
                                  uint8_t* __restrict__ smask, ull* __restrict__ bad) {
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nb;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t v = batch[i];
    if (v >= n || !live[v]) {
      atomicAdd(bad, 1ull);
      continue;
    }
    in_b[v] = 1;
    smask[rank[v]] = 1;
  }
}

// One warp per batch vertex: its live neighbours outside the batch are NB.
__global__ void batch_nbr_kernel(const uint32_t* __restrict__ batch, uint64_t nb,
                                 const uint64_t* __restrict__ off, const uint32_t* __restrict__ adj,
                                 const uint8_t* __restrict__ live, const uint8_t* __restrict__ in_b,
                                 uint8_t* __restrict__ nbr) {
  const uint32_t lane = threadIdx.x & 31;
  for (uint64_t i = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; i < nb;
       i += (uint64_t(gridDim.x) * blockDim.x) >> 5) {
    const uint32_t v = batch[i];
    const uint64_t b = off[v], e = off[v + 1];
    for (uint64_t p = b + lane; p < e; p += 32) {
      const uint32_t u = adj[p];
      if (live[u] && !in_b[u]) nbr[u] = 1;
    }
  }
}

// One warp per NB vertex u: N[u] joins the source mask.
__global__ void nbr_src_kernel(const uint32_t* __restrict__ nbl, const uint32_t* __restrict__ nnb,
                               const uint64_t* __restrict__ off, const uint32_t* __restrict__ adj,
                               const uint8_t* __restrict__ live, const uint32_t* __restrict__ rank,
                               uint8_t* __restrict__ smask) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t cnt = *nnb;
  for (uint64_t i = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; i < cnt;
       i += (uint64_t(gridDim.x) * blockDim.x) >> 5) {
    const uint32_t u = nbl[i];
    if (lane == 0) smask[rank[u]] = 1;
    const uint64_t b = off[u], e = off[u + 1];
    for (uint64_t p = b + lane; p < e; p += 32) {
      const uint32_t x = adj[p];
      if (live[x]) smask[rank[x]] = 1;
    }
  }
}

__global__ void batch_kill_kernel(const uint32_t* __restrict__ batch, uint64_t nb,
                                  uint8_t* __restrict__ live) {
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nb;
       i += uint64_t(gridDim.x) * blockDim.x)
    live[batch[i]] = 0;
}

// acc[0] += counts over the batch (before the update)
__global__ void batch_sum_kernel(const uint32_t* __restrict__ batch, uint64_t nb,
                                 const ull* __restrict__ counts, ull* __restrict__ acc) {
  ull s = 0;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nb;
       i += uint64_t(gridDim.x) * blockDim.x)
    s += counts[batch[i]];
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(FULLW, s, o);
  if ((threadIdx.x & 31) == 0 && s) atomicAdd(acc, s);
}

// Decrements the NB counts: d_u = pv_old[u] - pv_new[u] (pv_old null:
// counts[u] - pv_new[u]).  acc[1] += sum d_u, acc[2] counts underflows
// (a decrement below zero, peeling.cpp:159-161).
__global__ void apply_kernel(const uint32_t* __restrict__ nbl, const uint32_t* __restrict__ nnb,
                             const ull* __restrict__ pv_new, const ull* __restrict__ pv_old,
                             ull* __restrict__ counts, uint8_t* __restrict__ changed,
                             ull* __restrict__ acc) {
  ull s = 0;
  const uint64_t cnt = *nnb;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < cnt;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t u = nbl[i];
    const ull c = counts[u];
    const ull d = pv_old ? pv_old[u] - pv_new[u] : c - pv_new[u];
    if (d > c) atomicAdd(&acc[2], 1ull);
    counts[u] = c - d;
    if (changed) changed[u] = d != 0;
    s += d;
  }
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(FULLW, s, o);
  if ((threadIdx.x & 31) == 0 && s) atomicAdd(&acc[1], s);
}

__global__ void live_min_kernel(const uint8_t* __restrict__ live, const ull* __restrict__ cur,
                                uint32_t n, ull* __restrict__ out) {
  ull m = ~0ull;
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    if (live[v]) m = min(m, cur[v]);
  for (int o = 16; o; o >>= 1) m = min(m, __shfl_xor_sync(FULLW, m, o));
  if ((threadIdx.x & 31) == 0 && m != ~0ull) atomicMin(out, m);
}

// Round selection flags: exact -> live and cur == *minv; approx -> live and
// double(cur) <= cutoff (round-to-nearest conversion, as the host's).
__global__ void select_flags_kernel(const uint8_t* __restrict__ live, const ull* __restrict__ cur,
                                    uint32_t n, const ull* __restrict__ minv, double cutoff,
                                    uint8_t* __restrict__ flag) {
  const ull mv = minv ? *minv : 0;
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    bool f = false;
    if (live[v]) f = minv ? cur[v] == mv : __ull2double_rn(cur[v]) <= cutoff;
    flag[v] = f;
  }
}

__global__ void batch_retire_kernel(const uint32_t* __restrict__ batch, uint64_t nb,
                                    uint32_t round, ull level, uint32_t* __restrict__ peel_round,
                                    ull* __restrict__ core) {
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nb;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t v = batch[i];
    peel_round[v] = round;
    if (core) core[v] = level;
  }
}

__global__ void dense_flags_kernel(const uint32_t* __restrict__ peel_round, uint32_t n,
                                   uint64_t best_round, uint8_t* __restrict__ flag) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    flag[v] = uint64_t(peel_round[v]) > best_round;
}

__global__ void not_kernel(const uint8_t* __restrict__ in, uint32_t n, uint8_t* __restrict__ out) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    out[v] = in[v] ? 0 : 1;
}

// ---- workspace -------------------------------------------------------------
struct Ws {
  uint8_t *live, *live_rank, *in_b, *nbr, *smask, *flag;
  uint32_t *nbl, *batch, *sel, *peel_round;
  ull *cur, *pv_old, *cnt, *core, *acc;  // acc: [0] batch sum [1] d sum [2] underflow [3] bad [4] min
};

Ws workspace(Graph& g) {
  const size_t n = g.n;
  auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
  const size_t b8 = al(n + 1), b32 = al(4 * (n + 1)), b64 = al(8 * (n + 1));
  unsigned char* p = g.peel_ws.ensure(6 * b8 + 4 * b32 + 4 * b64 + 256, &g.alloc);
  Ws w;
  w.live = p;
  w.live_rank = p + b8;
  w.in_b = p + 2 * b8;
  w.nbr = p + 3 * b8;
  w.smask = p + 4 * b8;
  w.flag = p + 5 * b8;
  p += 6 * b8;
  w.nbl = reinterpret_cast<uint32_t*>(p);
  w.batch = reinterpret_cast<uint32_t*>(p + b32);
  w.sel = reinterpret_cast<uint32_t*>(p + 2 * b32);  // [0] selected count
  w.peel_round = reinterpret_cast<uint32_t*>(p + 3 * b32);
  p += 4 * b32;
  w.cur = reinterpret_cast<ull*>(p);
  w.pv_old = reinterpret_cast<ull*>(p + b64);
  w.cnt = reinterpret_cast<ull*>(p + 2 * b64);
  w.core = reinterpret_cast<ull*>(p + 3 * b64);
  w.acc = reinterpret_cast<ull*>(p + 4 * b64);
  return w;
}

// ids v in [0, n) with flag[v], ascending, into out; count into *cnt (device)
void select_ids(Graph& g, const uint8_t* flag, uint32_t* out, uint32_t* cnt) {
  thrust::counting_iterator<uint32_t> ids(0);
  size_t tb = 0;
  KCG_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, ids, flag, out, cnt, g.n, g.stream));
  KCG_CUDA(cub::DeviceSelect::Flagged(cub_temp(g, tb), tb, ids, flag, out, cnt, g.n, g.stream));
}

template <class T>
T fetch(Graph& g, const T* d) {
  T h;
  KCG_CUDA(cudaMemcpyAsync(&h, d, sizeof(T), cudaMemcpyDeviceToHost, g.stream));
  g.sync();
  return h;
}

// The DAG restricted to w.live, in g.live_off/live_adj.
void build_live_dag(Graph& g, const Ws& w) {
  const uint32_t n = g.n;
  live_rank_kernel<<<blocks_for(n, 256), 256, 0, g.stream>>>(w.live, g.order.p, n, w.live_rank);
  KCG_LAUNCHED(g);
  live_deg_kernel<<<blocks_for((uint64_t(n) + 1) * 32, 256), 256, 0, g.stream>>>(
      g.rdag_off.p, g.rdag_adj.p, w.live_rank, n, w.cnt);
  KCG_LAUNCHED(g);
  g.live_off.ensure(size_t(n) + 1, &g.alloc);
  size_t tb = 0;
  KCG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, w.cnt, g.live_off.p, n + 1, g.stream));
  KCG_CUDA(cub::DeviceScan::ExclusiveSum(cub_temp(g, tb), tb, w.cnt, g.live_off.p, n + 1,
                                         g.stream));
  g.live_adj.ensure(std::max<uint64_t>(g.m, 1), &g.alloc);
  live_fill_kernel<<<blocks_for(uint64_t(n) * 32, 256), 256, 0, g.stream>>>(
      g.rdag_off.p, g.rdag_adj.p, w.live_rank, n, g.live_off.p, g.live_adj.p);
  KCG_LAUNCHED(g);
}

// count_cliques on the live DAG with the batch-region source mask; the
// per-vertex counts land in g.pv (id order)
uint64_t count_live(Graph& g, const Ws& w, int k) {
  build_live_dag(g, w);
  std::swap(g.rdag_off.p, g.live_off.p);
  std::swap(g.rdag_off.n, g.live_off.n);
  std::swap(g.rdag_adj.p, g.live_adj.p);
  std::swap(g.rdag_adj.n, g.live_adj.n);
  g.src_mask = w.smask;
  struct Restore {
    Graph& g;
    ~Restore() {
      g.src_mask = nullptr;
      std::swap(g.rdag_off.p, g.live_off.p);
      std::swap(g.rdag_off.n, g.live_off.n);
      std::swap(g.rdag_adj.p, g.live_adj.p);
      std::swap(g.rdag_adj.n, g.live_adj.n);
    }
  } restore{g};
  return count_cliques(g, k, true);
}

struct RoundOut {
  uint64_t removed;
  bool underflow;
};

// One batch update (module comment).  w.batch holds nb distinct live ids;
// w.live is A on entry and A \ B on exit; w.cur is updated in place.
// exact_diff: count both sides (update_counts); else assume consistency.
RoundOut update_round(Graph& g, const Ws& w, int k, uint64_t nb, bool exact_diff,
                      bool want_changed) {
  const uint32_t n = g.n;
  KCG_CUDA(cudaMemsetAsync(w.in_b, 0, n, g.stream));
  KCG_CUDA(cudaMemsetAsync(w.nbr, 0, n, g.stream));
  KCG_CUDA(cudaMemsetAsync(w.smask, 0, n, g.stream));
  KCG_CUDA(cudaMemsetAsync(w.acc, 0, 8 * 8, g.stream));
  if (want_changed) KCG_CUDA(cudaMemsetAsync(w.flag, 0, n, g.stream));
  batch_mark_kernel<<<blocks_for(nb, 256), 256, 0, g.stream>>>(w.batch, nb, n, w.live, g.rank.p,
                                                               w.in_b, w.smask, w.acc + 3);
  KCG_LAUNCHED(g);
  if (fetch(g, w.acc + 3)) fail(KCG_EINVAL, "batch vertex already peeled");
  batch_nbr_kernel<<<blocks_for(nb * 32, 256), 256, 0, g.stream>>>(
      w.batch, nb, g.und_off.p, g.und_adj.p, w.live, w.in_b, w.nbr);
  KCG_LAUNCHED(g);
  select_ids(g, w.nbr, w.nbl, w.sel);
  nbr_src_kernel<<<blocks_for(uint64_t(n) * 32, 256), 256, 0, g.stream>>>(
      w.nbl, w.sel, g.und_off.p, g.und_adj.p, w.live, g.rank.p, w.smask);
  KCG_LAUNCHED(g);
  batch_sum_kernel<<<blocks_for(nb, 256), 256, 0, g.stream>>>(w.batch, nb, w.cur, w.acc);
  KCG_LAUNCHED(g);
  uint64_t tot_a = 0;
  if (exact_diff) {
    tot_a = count_live(g, w, k);
    KCG_CUDA(cudaMemcpyAsync(w.pv_old, g.pv.p, size_t(n) * 8, cudaMemcpyDeviceToDevice,
                             g.stream));
  }
  batch_kill_kernel<<<blocks_for(nb, 256), 256, 0, g.stream>>>(w.batch, nb, w.live);
  KCG_LAUNCHED(g);
  const uint64_t tot_ab = count_live(g, w, k);
  apply_kernel<<<blocks_for(n, 256), 256, 0, g.stream>>>(
      w.nbl, w.sel, reinterpret_cast<const ull*>(g.pv.p), exact_diff ? w.pv_old : nullptr, w.cur,
      want_changed ? w.flag : nullptr, w.acc);
  KCG_LAUNCHED(g);
  ull acc[3];
  KCG_CUDA(cudaMemcpyAsync(acc, w.acc, sizeof(acc), cudaMemcpyDeviceToHost, g.stream));
  g.sync();
  RoundOut r;
  r.underflow = acc[2] != 0;
  r.removed = exact_diff ? tot_a - tot_ab : (acc[0] + acc[1]) / uint64_t(k);
  return r;
}

void require_graphs(Graph& g) {
  if (!g.has_und) fail(KCG_EINVAL, "peeling needs the undirected graph on the handle");
  if (!g.has_rdag) {
    if (!g.has_rank) fail(KCG_EINVAL, "no DAG: call kcg_rank/kcg_direct first");
    build_dag(g, false);
  }
}

}  // namespace

UpdateOut update_counts(Graph& g, int k, uint64_t* counts, const uint32_t* batch,
                        uint64_t batch_len, const uint8_t* peeled) {
  if (k < 2) fail(KCG_EINVAL, "k must be at least 2");
  require_graphs(g);
  const uint32_t n = g.n;
  if (n && (!counts || !peeled)) fail(KCG_EINVAL, "counts and peeled must hold n entries");
  if (batch_len && !batch) fail(KCG_EINVAL, "batch is null");
  UpdateOut out;
  if (n == 0) {
    if (batch_len) fail(KCG_EINVAL, "batch vertex already peeled");
    return out;
  }
  if (batch_len > n) fail(KCG_EINVAL, "batch longer than the vertex set");
  const Ws w = workspace(g);
  KCG_CUDA(cudaMemcpyAsync(w.flag, peeled, n, cudaMemcpyHostToDevice, g.stream));
  not_kernel<<<blocks_for(n, 256), 256, 0, g.stream>>>(w.flag, n, w.live);
  KCG_LAUNCHED(g);
  KCG_CUDA(cudaMemcpyAsync(w.cur, counts, size_t(n) * 8, cudaMemcpyHostToDevice, g.stream));
  if (batch_len)
    KCG_CUDA(cudaMemcpyAsync(w.batch, batch, batch_len * 4, cudaMemcpyHostToDevice, g.stream));
  g.times.h2d_bytes += n + size_t(n) * 8 + batch_len * 4;
  if (batch_len == 0) return out;
  const RoundOut r = update_round(g, w, k, batch_len, true, true);
  select_ids(g, w.flag, w.nbl, w.sel);
  const uint32_t nch = fetch(g, w.sel);
  out.changed.resize(nch);
  if (nch)
    KCG_CUDA(cudaMemcpyAsync(out.changed.data(), w.nbl, size_t(nch) * 4, cudaMemcpyDeviceToHost,
                             g.stream));
  KCG_CUDA(cudaMemcpyAsync(counts, w.cur, size_t(n) * 8, cudaMemcpyDeviceToHost, g.stream));
  g.sync();
  g.times.d2h_bytes += size_t(nch) * 4 + size_t(n) * 8;
  if (r.underflow) fail(KCG_ELOGIC, "clique count went negative during update");
  out.removed = r.removed;
  return out;
}

PeelOut peel(Graph& g, int k, bool exact, double eps, uint64_t* core_out) {
  if (k < 2) fail(KCG_EINVAL, "k must be at least 2");
  if (!exact && !(eps > 0)) fail(KCG_EINVAL, "epsilon must be positive");
  require_graphs(g);
  const uint32_t n = g.n;
  PeelOut out;
  if (n == 0) return out;
  // per-vertex counts of the whole graph (peeling.cpp:206, 254)
  out.total = count_cliques(g, k, true);
  const Ws w = workspace(g);
  KCG_CUDA(cudaMemcpyAsync(w.cur, g.pv.p, size_t(n) * 8, cudaMemcpyDeviceToDevice, g.stream));
  KCG_CUDA(cudaMemsetAsync(w.live, 1, n, g.stream));
  KCG_CUDA(cudaMemsetAsync(w.peel_round, 0xff, size_t(n) * 4, g.stream));
  if (exact) KCG_CUDA(cudaMemsetAsync(w.core, 0, size_t(n) * 8, g.stream));
  // DensityTracker (peeling.cpp:196-211): exact fraction comparison
  uint64_t best_cliques = 0, best_alive = 1, best_round = 0;
  auto offer = [&](uint64_t cliques, uint64_t alive, uint64_t round) {
    if (alive == 0) return;
    typedef unsigned __int128 U;
    if (U(cliques) * best_alive > U(best_cliques) * alive) {
      best_cliques = cliques;
      best_alive = alive;
      best_round = round;
    }
  };
  offer(out.total, n, 0);
  uint64_t remaining = out.total, alive = n, round = 0, level = 0;
  while (alive > 0) {
    round++;
    if (exact) {
      KCG_CUDA(cudaMemsetAsync(w.acc + 4, 0xff, 8, g.stream));
      live_min_kernel<<<blocks_for(n, 256), 256, 0, g.stream>>>(w.live, w.cur, n, w.acc + 4);
      KCG_LAUNCHED(g);
      select_flags_kernel<<<blocks_for(n, 256), 256, 0, g.stream>>>(w.live, w.cur, n, w.acc + 4,
                                                                    0.0, w.flag);
    } else {
      const double cutoff =
          double(k) * (1.0 + eps) * (double(remaining) / double(alive));
      select_flags_kernel<<<blocks_for(n, 256), 256, 0, g.stream>>>(w.live, w.cur, n, nullptr,
                                                                    cutoff, w.flag);
    }
    KCG_LAUNCHED(g);
    select_ids(g, w.flag, w.batch, w.sel);
    uint64_t val = 0;
    uint32_t nb = 0;
    if (exact) {
      ull hv = 0;
      KCG_CUDA(cudaMemcpyAsync(&hv, w.acc + 4, 8, cudaMemcpyDeviceToHost, g.stream));
      nb = fetch(g, w.sel);
      val = hv;
      level = std::max(level, val);
    } else {
      nb = fetch(g, w.sel);
    }
    if (nb == 0) fail(KCG_ELOGIC, "approximate peeling made no progress");
    const RoundOut r = update_round(g, w, k, nb, false, false);
    if (r.underflow) fail(KCG_ELOGIC, "clique count went negative during update");
    batch_retire_kernel<<<blocks_for(nb, 256), 256, 0, g.stream>>>(
        w.batch, nb, uint32_t(round), level, w.peel_round, exact ? w.core : nullptr);
    KCG_LAUNCHED(g);
    remaining -= r.removed;
    alive -= nb;
    offer(remaining, alive, round);
  }
  out.rounds = round;
  out.best_round = best_round;
  out.best_density = best_alive ? double(best_cliques) / double(best_alive) : 0.0;
  dense_flags_kernel<<<blocks_for(n, 256), 256, 0, g.stream>>>(w.peel_round, n, best_round,
                                                               w.flag);
  KCG_LAUNCHED(g);
  select_ids(g, w.flag, w.nbl, w.sel);
  const uint32_t nd = fetch(g, w.sel);
  out.dense.resize(nd);
  if (nd)
    KCG_CUDA(cudaMemcpyAsync(out.dense.data(), w.nbl, size_t(nd) * 4, cudaMemcpyDeviceToHost,
                             g.stream));
  if (exact && core_out)
    KCG_CUDA(cudaMemcpyAsync(core_out, w.core, size_t(n) * 8, cudaMemcpyDeviceToHost, g.stream));
  g.sync();
  return out;
}

}  // namespace kcg
