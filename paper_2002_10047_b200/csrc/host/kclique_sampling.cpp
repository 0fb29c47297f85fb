// Drop-in sampling entry points (include/kclique/sampling.hpp): the
// sparsification and the exact count inside it run on the B200
// (kcg_colorful_sparsify, kcg_approx_count); analytic_variance is the
// closed form of proj/src/sampling.cpp:59-77 evaluated on the host.
#include <cmath>
#include <stdexcept>

#include "kcg_cache.hpp"
#include "kcg_handle.hpp"
#include "kclique/sampling.hpp"

namespace kclique {

namespace {

int strategy_code(OrientStrategy s) {
  switch (s) {
    case OrientStrategy::degree: return KCG_DEGREE;
    case OrientStrategy::original: return KCG_ORIGINAL;
    case OrientStrategy::kcore: return KCG_KCORE;
    case OrientStrategy::goodrich_pszona: return KCG_GOODRICH_PSZONA;
    case OrientStrategy::barenboim_elkin: return KCG_BARENBOIM_ELKIN;
  }
  throw std::invalid_argument("unknown orientation strategy");
}

}  // namespace

Graph colorful_sparsify(const Graph& g, uint64_t colors, uint64_t seed) {
  if (colors < 1) throw std::invalid_argument("colors must be at least 1");
  if (colors == 1) return g;
  auto res = b200::resident_for_graph(g);
  std::lock_guard<std::mutex> lk(res->mu);
  kcg_graph* out = nullptr;
  b200::check(kcg_colorful_sparsify(res->h, colors, seed, &out));
  b200::Handle sub(out);
  return b200::GraphAccess::download(sub.get());
}

SampleEstimate approx_count(const Graph& g, int k, uint64_t colors, uint64_t seed,
                            const OrientConfig& ocfg, const CountConfig&) {
  if (k < 2) throw std::invalid_argument("k must be at least 2");
  if (colors < 1) throw std::invalid_argument("colors must be at least 1");
  if (ocfg.alpha_hat && *ocfg.alpha_hat < 1)
    throw std::invalid_argument("alpha_hat must be >= 1");
  auto res = b200::resident_for_graph(g);
  std::lock_guard<std::mutex> lk(res->mu);
  kcg_sample_estimate e{};
  b200::check(kcg_approx_count(res->h, k, colors, seed, strategy_code(ocfg.strategy),
                               ocfg.epsilon, ocfg.alpha_hat ? *ocfg.alpha_hat : 0, &e));
  SampleEstimate est;
  est.k = e.k;
  est.colors = e.colors;
  est.p = e.p;
  est.sub_count = e.sub_count;
  est.estimate = e.estimate;
  est.seed = e.seed;
  return est;
}

double analytic_variance(uint64_t true_count, double p, int k,
                         std::span<const uint64_t> shared_pairs) {
  if (k < 2) throw std::invalid_argument("k must be at least 2");
  if (!(p > 0.0 && p <= 1.0)) throw std::invalid_argument("p must be in (0, 1]");
  // one clique survives with probability p^(k-1); two sharing z >= 2
  // vertices survive together with p^(2(k-1) - z + 1)
  const double e1 = k - 1;
  double var = double(true_count) * (std::pow(p, e1) - std::pow(p, 2 * e1));
  for (int z = 2; z <= k - 1 && size_t(z) < shared_pairs.size(); z++)
    var += 2.0 * double(shared_pairs[z]) * (std::pow(p, 2 * e1 - z + 1) - std::pow(p, 2 * e1));
  return var * std::pow(p, -2 * e1);
}

}  // namespace kclique
