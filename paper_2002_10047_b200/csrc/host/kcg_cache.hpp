// Device residency behind the drop-in API ("count_total(dg,
// k) reuses the device DAG when dg came from the device path (side table
// keyed by the DirectedGraph's data pointer)").
//
// The reference's call sequence is make_ranking(g) -> direct_by_ranking(g,
// r) -> count_*(dg) / peel_*(g, dg) (proj/tools/kclique_main.cpp:158-182,
// proj/src/sampling.cpp:47-48, proj/src/peeling.cpp:229-232).  Each call
// takes host objects, so a naive drop-in re-uploads the CSR for every call
// and the DAG for every count.  Here a process-wide registry keeps a small
// LRU of device handles ("residents"), each remembering which host objects
// its device buffers currently mirror:
//
//   graph : the Graph whose CSR was uploaded (its offsets/adjacency data
//           pointers, n, m and a sampled fingerprint)
//   rank  : the Ranking currently installed (returned by a rank_* call on
//           this resident or uploaded by direct_by_ranking)
//   dag   : the DirectedGraph last downloaded from this resident (its
//           out_targets data pointer, n, m, fingerprint)
//
// Graph, Ranking and DirectedGraph are immutable value types (graph.hpp:
// 29-31, 88-90), so pointer + size + fingerprint identifies their content
// while they live; a freed object whose storage is reused by another with
// the same sizes and the same sampled words would alias -- set
// KCG_DROPIN_CACHE=0 to upload on every call instead.
#pragma once

#include <cstdint>
#include <memory>
#include <mutex>
#include <vector>

#include "kcg.h"
#include "kclique/graph.hpp"

namespace kclique::b200 {

struct Key {
  const void* a = nullptr;
  const void* b = nullptr;
  uint64_t n = 0, m = 0, fp = 0;
  bool valid() const { return a != nullptr; }
  bool operator==(const Key& o) const {
    return a == o.a && b == o.b && n == o.n && m == o.m && fp == o.fp;
  }
};

Key key_of(const Graph& g);
Key key_of(const Ranking& r);
Key key_of(const DirectedGraph& dg);

struct Resident {
  std::mutex mu;  // held for every device call on h
  kcg_graph* h = nullptr;
  Key graph, rank, dag;
  uint64_t tick = 0;
  Resident() = default;
  Resident(const Resident&) = delete;
  Resident& operator=(const Resident&) = delete;
  ~Resident();
};
using ResidentPtr = std::shared_ptr<Resident>;

bool cache_enabled();

// The resident holding g's CSR (uploaded on a miss).
ResidentPtr resident_for_graph(const Graph& g);
// A resident whose device DAG mirrors dg (a graph resident after
// direct_by_ranking, else a DAG-only resident adopted from dg's arrays).
ResidentPtr resident_for_dag(const DirectedGraph& dg);
// With r.mu held: install dg's ranking on g's resident unless its device
// DAG already mirrors dg (peeling rebuilds the DAG from g and the ranking,
// direct_by_ranking being a function of the two, graph.cpp:94-114).
void ensure_oriented(Resident& r, const Graph& g, const DirectedGraph& dg);
// With r.mu held: install ranking `rk` unless it is the one on the device.
void ensure_ranking(Resident& r, const Ranking& rk);
// With r.mu held: record what the device now mirrors (a kcg_rank result,
// a downloaded DAG); invalid keys for "nothing known".
void set_keys(Resident& r, const Key& rank, const Key& dag);

// H2D bytes issued by the drop-in since the process started (for the API
// benchmark, tests/cpp/api_bench.cpp).
uint64_t dropin_h2d_bytes();
void note_h2d(uint64_t bytes);

}  // namespace kclique::b200
