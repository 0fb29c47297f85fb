// Drop-in counting entry points (include/kclique/counting.hpp): a
// DirectedGraph from direct_by_ranking is counted on the handle that built
// it; any other is adopted once by a device handle (kcg_dag_create, which
// relabels it by rank on the GPU) and kept resident (kcg_cache.hpp).
#include <exception>

#include "kcg_cache.hpp"
#include "kcg_handle.hpp"
#include "kclique/counting.hpp"

namespace kclique {

Parallelism default_parallelism(int k) { return k < 8 ? Parallelism::node : Parallelism::edge; }

namespace {

CliqueCounts run(const DirectedGraph& dg, int k, bool per_vertex) {
  if (k < 2) throw std::invalid_argument("k must be at least 2");
  CliqueCounts out;
  out.k = k;
  if (per_vertex) b200::resize_huge(out.per_vertex, dg.num_vertices());
  if (dg.num_vertices() == 0) return out;
  // the resident whose device DAG mirrors dg (direct_by_ranking's), else
  // dg's arrays adopted once and kept for the next call
  auto res = b200::resident_for_dag(dg);
  std::lock_guard<std::mutex> lk(res->mu);
  b200::check(kcg_count(res->h, k, &out.total, per_vertex ? out.per_vertex.data() : nullptr));
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
  auto res = b200::resident_for_dag(dg);
  std::lock_guard<std::mutex> lk(res->mu);
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
  const int rc = kcg_list_cliques(res->h, k, 0, fn, &ctx, &out.total);
  if (ctx.err) std::rethrow_exception(ctx.err);
  b200::check(rc);
  return out;
}

}  // namespace kclique
