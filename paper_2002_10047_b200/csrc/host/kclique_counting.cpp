// Drop-in counting entry points (include/kclique/counting.hpp): the
// DirectedGraph is adopted by a device handle (kcg_dag_create, which
// relabels it by rank on the GPU) and counted by kcg_count.
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
  (void)dg;
  (void)emit;
  // Device-side emission is SURVEY.md §8(f) row 3 ("next"); refuse loudly
  // rather than enumerate on the CPU.
  throw std::runtime_error("list_cliques: clique emission is not implemented on the B200 path");
}

}  // namespace kclique
