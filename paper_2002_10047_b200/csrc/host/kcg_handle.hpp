// RAII wrapper over the kcg C ABI, shared by the drop-in translation units.
// Status codes map back onto the reference's exception types
// (SURVEY.md §8(b)): KCG_EINVAL -> std::invalid_argument,
// KCG_ENOMEM -> std::bad_alloc, KCG_ELOGIC -> std::logic_error, anything
// else -> std::runtime_error.
#pragma once

#include <sys/mman.h>

#include <cstdint>
#include <new>
#include <vector>
#include <stdexcept>
#include <string>

#include "kcg.h"
#include "kclique/graph.hpp"

namespace kclique::b200 {

// Sizes a large output vector with transparent huge pages requested for its
// storage before the value-initialisation touches it (2 MB pages: 512x
// fewer page faults when the vector is zero-filled and then pinned for the
// device copy).  Small vectors are just resized.
template <class T>
void resize_huge(std::vector<T>& v, size_t n) {
  const size_t bytes = n * sizeof(T);
  if (bytes >= (size_t(4) << 20) && v.capacity() < n) {
    v.reserve(n);
    const uintptr_t a = reinterpret_cast<uintptr_t>(v.data());
    const uintptr_t lo = (a + (uintptr_t(2) << 20) - 1) & ~((uintptr_t(2) << 20) - 1);
    const uintptr_t hi = (a + bytes) & ~((uintptr_t(2) << 20) - 1);
    if (hi > lo) madvise(reinterpret_cast<void*>(lo), hi - lo, MADV_HUGEPAGE);
  }
  v.resize(n);
}

inline void check(int rc) {
  if (rc == KCG_OK) return;
  std::string msg = kcg_last_error();
  if (rc == KCG_EINVAL) throw std::invalid_argument(msg);
  if (rc == KCG_ENOMEM) throw std::bad_alloc();
  if (rc == KCG_ELOGIC) throw std::logic_error(msg);
  throw std::runtime_error("kcg: " + msg);
}

// Adopts a device-built CSR (normalised on the GPU) as a host Graph.
struct GraphAccess {
  static Graph download(kcg_graph* h) {
    Graph g;
    g.n_ = kcg_num_vertices(h);
    g.m_ = kcg_num_edges(h);
    resize_huge(g.offsets_, size_t(g.n_) + 1);
    resize_huge(g.neighbors_, 2 * g.m_);
    check(kcg_graph_csr(h, g.offsets_.data(), g.neighbors_.data()));
    return g;
  }
};

class Handle {
 public:
  explicit Handle(kcg_graph* h) : h_(h) {}
  Handle(const Handle&) = delete;
  Handle& operator=(const Handle&) = delete;
  ~Handle() { kcg_graph_destroy(h_); }
  kcg_graph* get() const { return h_; }

  static Handle upload(const Graph& g) {
    kcg_graph* h = nullptr;
    check(kcg_graph_create(g.num_vertices(), g.offsets().data(), g.adjacency().data(), &h));
    return Handle(h);
  }
  static Handle adopt(const DirectedGraph& dg) {
    kcg_graph* h = nullptr;
    std::vector<uint64_t> off(size_t(dg.num_vertices()) + 1);
    for (VertexId v = 0; v < dg.num_vertices(); v++) off[v] = dg.out_offset(v);
    off[dg.num_vertices()] = dg.num_edges();
    check(kcg_dag_create(dg.num_vertices(), off.data(), dg.out_targets().data(),
                         dg.ranking().ranks().data(), &h));
    return Handle(h);
  }
  Handle(Handle&& o) noexcept : h_(o.h_) { o.h_ = nullptr; }

 private:
  kcg_graph* h_;
};

}  // namespace kclique::b200
