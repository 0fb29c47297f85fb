// Drop-in counting entry points (include/kclique/counting.hpp): the
// DirectedGraph is adopted by a device handle (kcg_dag_create, which
// relabels it by rank on the GPU) and counted by kcg_count.
#include <exception>

#include "kcg_handle.hpp"
#include "kclique/counting.hpp"

namespace kclique {

Parallelism default_parallelism(int k) { return k < 8 ? Parallelism::node : Parallelism::edge; }

namespace {

CliqueCounts run(const DirectedGraph& dg, int k, bool per_vertex) {
  if (k < 2) throw std::invalid_argument("k must be at least 2");
  CliqueCounts out;
  out.k = k;
  if (per_vertex) out.per_vertex.assign(dg.num_vertices(), 0);
  if (dg.num_vertices() == 0) return out;
  auto h = b200::Handle::adopt(dg);
  b200::check(kcg_count(h.get(), k, &out.total, per_vertex ? out.per_vertex.data() : nullptr));
  return out;
}

}  // namespace

CliqueCounts count_total(const DirectedGraph& dg, int k, const CountConfig&) {
  return run(dg, k, false);
}

CliqueCounts count_per_vertex(const DirectedGraph& dg, int k, const CountConfig&) {
  return run(dg, k, true);
}

CliqueCounts list_cliques(const DirectedGraph& dg, int k, const CountConfig&,
                          const CliqueCallback& emit) {
  if (k < 2) throw std::invalid_argument("k must be at least 2");
  CliqueCounts out;
  out.k = k;
  if (dg.num_vertices() == 0) return out;
  auto h = b200::Handle::adopt(dg);
  // cliques arrive in device batches; each is reported in ascending rank
  // (an exception from the callback aborts the listing and is rethrown)
  struct Ctx {
    const CliqueCallback* emit;
    std::exception_ptr err;
  } ctx{&emit, nullptr};
  auto fn = [](const uint32_t* c, uint64_t count, int kk, void* user) -> int {
    auto* cx = static_cast<Ctx*>(user);
    try {
      for (uint64_t i = 0; i < count; i++)
        (*cx->emit)(std::span<const VertexId>(c + i * uint64_t(kk), size_t(kk)));
    } catch (...) {
      cx->err = std::current_exception();
      return 1;
    }
    return 0;
  };
  const int rc = kcg_list_cliques(h.get(), k, 0, fn, &ctx, &out.total);
  if (ctx.err) std::rethrow_exception(ctx.err);
  b200::check(rc);
  return out;
}

}  // namespace kclique
