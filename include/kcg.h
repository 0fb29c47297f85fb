/* kcg — B200-native arb-count (k-clique counting) C ABI.
 *
 * This is the drop-in boundary: a C-ABI shared library
 * (paper_2002_10047_b200/lib/libkcg.so, sm_100a) with plain pointers and
 * sizes.  The C++ library libkclique_b200.so implements the reference's own
 * entry points (the headers in include/kclique/, mirroring
 * /root/reference/proj/include/kclique/) on top of these calls; any other
 * host language binds them directly.
 *
 * Conventions
 *  - Every call returns a status: KCG_OK, KCG_EINVAL (the cases where the
 *    reference throws std::invalid_argument), KCG_ELOGIC (where it throws
 *    std::logic_error), KCG_ERUNTIME (CUDA/runtime failure), KCG_ENOMEM
 *    (device or host allocation failed).
 *    kcg_last_error() returns the calling thread's last message.
 *  - Host buffers are caller-allocated; device memory is owned by the
 *    kcg_graph handle and stays resident across calls.
 *  - A handle is not internally synchronised: use one handle per host
 *    thread (each handle owns its own CUDA stream), or serialise calls.
 *  - All counts are uint64 and wrap modulo 2^64 like the reference
 *    (SPEC.md:225).
 *  - There is no CPU fallback: without a usable sm_100 device every
 *    compute call fails with KCG_ERUNTIME.
 */
#ifndef KCG_H_
#define KCG_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KCG_OK 0
#define KCG_EINVAL 1
#define KCG_ERUNTIME 2
#define KCG_ENOMEM 3
#define KCG_ELOGIC 4  /* the reference's std::logic_error cases (peeling) */

/* OrientStrategy (proj/include/kclique/orientation.hpp:10-16), same order. */
#define KCG_DEGREE 0
#define KCG_ORIGINAL 1
#define KCG_KCORE 2
#define KCG_GOODRICH_PSZONA 3
#define KCG_BARENBOIM_ELKIN 4
/* Not in the reference: a bulk-synchronous degeneracy order (every vertex
 * at the current minimum level leaves in the same round, ranked by
 * (round, id)).  Same max out-degree as KCG_KCORE, which reproduces the
 * reference's sequential (degree, id) heap order exactly but pops one
 * vertex at a time. */
#define KCG_KCORE_PARALLEL 5

typedef struct kcg_graph kcg_graph;

/* Device-timed phase split of the most recent calls on a handle, in ms
 * (CUDA events on the handle's stream), plus transfer bytes. */
typedef struct kcg_times {
  double upload_ms;   /* H2D of the input CSR (kcg_graph_create) */
  double rank_ms;     /* last kcg_rank / kcg_estimate_arboricity */
  double direct_ms;   /* last kcg_direct (DAG + relabelled DAG build) */
  double count_ms;    /* last kcg_count, all counting kernels */
  double count_kernel_ms; /* the dominant counting kernel(s) only */
  double download_ms; /* D2H of the last call's host outputs */
  uint64_t h2d_bytes;
  uint64_t d2h_bytes;
  uint64_t launches;  /* kernels of this library launched on the handle, cumulative */
} kcg_times;

/* Static description of the counting work of the last kcg_count. */
typedef struct kcg_count_stats {
  uint64_t sources_warp;   /* sources with out-degree <= 32 */
  uint64_t sources_cta;    /* 32 < out-degree <= smem tier limit */
  uint64_t sources_heavy;  /* beyond the shared-memory limit */
  uint64_t max_out_degree;
  uint64_t staged_elems;   /* adjacency entries read while staging */
  uint64_t launches;       /* kernels launched by the last kcg_count */
} kcg_count_stats;

const char* kcg_last_error(void);
const char* kcg_version(void);

/* Device properties this library sizes itself from. */
int kcg_device_info(int* sm_count, int* smem_optin_bytes, int* l2_bytes,
                    int* cc_major, int* cc_minor);

/* Uploads an undirected simple CSR (kclique::Graph layout,
 * graph.hpp:59-62: u64 offsets[n+1], u32 adjacency[2m], ascending,
 * symmetric, loop-free).  Replaces the Graph the reference's entry points
 * take by const reference.  Host pointers. */
int kcg_graph_create(uint32_t n, const uint64_t* offsets, const uint32_t* adj,
                     kcg_graph** out);
/* Same from device-resident arrays (copied on the handle's stream). */
int kcg_graph_create_device(uint32_t n, uint64_t m, const uint64_t* d_offsets,
                            const uint32_t* d_adj, kcg_graph** out);
/* Adopts an already-oriented DAG (kclique::DirectedGraph layout,
 * graph.hpp:91-121: out_offsets[n+1], out-targets[m] ascending by id) and
 * its ranking, for count_total/count_per_vertex on a DirectedGraph that
 * did not come from this handle.  rank may be NULL only if n == 0. */
int kcg_dag_create(uint32_t n, const uint64_t* out_offsets,
                   const uint32_t* out_targets, const uint32_t* rank,
                   kcg_graph** out);
/* Graph::from_edges (graph.cpp:11-41) on the device: `count` edges
 * (host arrays us[i], vs[i]) are swapped to u < v, self-loops dropped,
 * sorted, deduplicated and symmetrised into the CSR the handle keeps.
 * KCG_EINVAL if an endpoint is >= n (the reference's invalid_argument). */
int kcg_graph_from_edges(uint32_t n, const uint32_t* us, const uint32_t* vs,
                         uint64_t count, kcg_graph** out);
/* The benchmark's R-MAT generator on the device (2^scale vertices,
 * `samples` draws, quadrant probabilities a, b, c, 1-a-b-c, optional seeded
 * id permutation), normalised like kcg_graph_from_edges.  Bit-identical to
 * the host generator (csrc/gen/kcgen.cpp kcgen_rmat). */
int kcg_graph_rmat(int scale, uint64_t samples, double a, double b, double c,
                   uint64_t seed, int permute, kcg_graph** out);
/* Downloads the handle's undirected CSR (offsets n+1, adjacency 2m);
 * either pointer may be NULL. */
int kcg_graph_csr(kcg_graph* g, uint64_t* offsets, uint32_t* adj);
void kcg_graph_destroy(kcg_graph* g);
uint32_t kcg_num_vertices(const kcg_graph* g);
uint64_t kcg_num_edges(const kcg_graph* g);

/* Ranking (orientation.cpp:10-174).  strategy is one of KCG_*; for
 * KCG_BARENBOIM_ELKIN an alpha_hat of 0 means "estimate it with
 * estimate_arboricity(g, eps)" exactly as make_ranking does
 * (orientation.cpp:167-170).  The ranking stays on the device for
 * kcg_direct.  rank_out (n entries), rounds_out and alpha_out may be NULL.
 * KCG_EINVAL for eps <= 0 (peeling strategies) or an unknown strategy. */
int kcg_rank(kcg_graph* g, int strategy, double eps, uint64_t alpha_hat,
             uint32_t* rank_out, uint64_t* rounds_out, uint64_t* alpha_out);
/* estimate_arboricity (orientation.cpp:124-155). */
int kcg_estimate_arboricity(kcg_graph* g, double eps, uint64_t* out);
/* Installs a host ranking; KCG_EINVAL unless it is a bijection onto [0,n)
 * (graph.cpp:48-55) of length n (graph.cpp:95-96). */
int kcg_set_ranking(kcg_graph* g, const uint32_t* rank, uint32_t len);

/* direct_by_ranking (graph.cpp:94-114) on the device with the handle's
 * current ranking.  Outputs are optional host buffers: out_offsets
 * (n+1), out_targets (m); max_out_degree may be NULL. */
int kcg_direct(kcg_graph* g, uint64_t* out_offsets, uint32_t* out_targets,
               uint64_t* max_out_degree);

/* count_total / count_per_vertex (counting.cpp:85-212) on the handle's
 * DAG (built by kcg_direct or adopted by kcg_dag_create).  per_vertex is
 * NULL for totals only, else n entries indexed by vertex id.
 * KCG_EINVAL for k < 2. */
int kcg_count(kcg_graph* g, int k, uint64_t* total, uint64_t* per_vertex);
/* Multi-GPU sharding (the reference's edge engine over
 * independent sources, proj/src/counting.cpp:138-198).  Every clique is
 * charged to its lowest-ranked vertex r (rank space), so source ranges
 * partition the cliques.
 * kcg_partition_plan: work-balanced contiguous ranges -- bounds[0..nparts],
 *   part p owns ranks [bounds[p], bounds[p+1]); the work of source r is
 *   1 + d + sum_{x in N+(r)} (1 + d+(x)) (+ d^2 for k >= 5), the staging
 *   term of the counting kernels (paper_2002_10047_b200/shard.py:plan is
 *   the host mirror).
 * kcg_count_range: the cliques whose lowest-ranked vertex lies in
 *   [r_lo, r_hi).
 * kcg_count_part: kcg_count_range over part `part` of kcg_partition_plan.
 * Summing the totals (and per-vertex arrays) of all parts gives kcg_count's
 * result; callers all-reduce them across GPUs.  per_vertex is NULL or n
 * entries.  KCG_EINVAL for k < 2, part >= nparts or r_lo > r_hi. */
int kcg_partition_plan(kcg_graph* g, int k, uint32_t nparts, uint32_t* bounds);
/* sum_w indeg(w) * outdeg(w) over the current DAG: the staging term of the
 * per-source scheme's algorithmic bytes (SURVEY.md §8(d) B_alg = 16n + 20m
 * + 4 * this), computed on the device (bench.py's roofline). */
int kcg_dag_work(kcg_graph* g, uint64_t* sum_indeg_outdeg);
int kcg_count_range(kcg_graph* g, int k, uint32_t r_lo, uint32_t r_hi,
                    uint64_t* total, uint64_t* per_vertex);
int kcg_count_part(kcg_graph* g, int k, uint32_t part, uint32_t nparts,
                   uint64_t* total, uint64_t* per_vertex);
/* Device pointer to the per-vertex counts of the last per-vertex count
 * (n u64, vertex-id order); valid until the next call on the handle. */
int kcg_per_vertex_device(kcg_graph* g, const uint64_t** d_per_vertex);

/* Fused rank -> direct -> count with no host round trip in between
 * (the benchmark's step).  per_vertex may be NULL. */
int kcg_pipeline(kcg_graph* g, int strategy, double eps, uint64_t alpha_hat,
                 int k, uint64_t* total, uint64_t* per_vertex);

/* list_cliques (counting.hpp:42-49, counting.cpp:214-217) on the device:
 * every k-clique exactly once, vertices in ascending rank, delivered to
 * `fn` in batches of at most `batch` cliques (0: 2^24) as count * k vertex
 * ids (row-major).  A non-zero return from fn aborts with KCG_ERUNTIME.
 * *total receives the clique count.  KCG_EINVAL for k < 2 or k > 33. */
typedef int (*kcg_clique_fn)(const uint32_t* cliques, uint64_t count, int k, void* user);
int kcg_list_cliques(kcg_graph* g, int k, uint64_t batch, kcg_clique_fn fn, void* user,
                     uint64_t* total);

/* ---- Peeling: consumers of the per-vertex counts (SURVEY.md §8(f) row 1,
 * proj/include/kclique/peeling.hpp:59-92).  The handle must hold the
 * undirected graph (kcg_graph_create) and a ranking (kcg_rank or
 * kcg_set_ranking); the DAG is built on demand.  Cliques are counted on the
 * device by restricted recounts (kcg_peel.cu). */

/* PeelOutcome (peeling.hpp:67-76) minus its arrays. */
typedef struct kcg_peel_result {
  uint64_t rounds;         /* extraction rounds */
  uint64_t total_cliques;  /* k-clique count of the input graph */
  double best_density;     /* max over rounds of remaining cliques / remaining vertices */
  uint64_t best_round;     /* first round attaining it (0 = before any removal) */
  uint64_t num_dense;      /* entries written to dense_vertices */
} kcg_peel_result;

/* update_counts (peeling.hpp:58-63, peeling.cpp:114-200): removes the
 * batch (batch_len distinct ids) from the graph minus the `peeled` flags
 * (n bytes), subtracts from counts (n u64, host, in/out) the k-cliques each
 * survivor loses, and reports the destroyed cliques and the survivors
 * whose count dropped (ascending ids; `changed` holds n entries).
 * KCG_EINVAL for k < 2 or a batch vertex that is out of range or peeled;
 * KCG_ELOGIC when a count would go negative (counts inconsistent). */
int kcg_update_counts(kcg_graph* g, int k, uint64_t* counts, const uint32_t* batch,
                      uint64_t batch_len, const uint8_t* peeled, uint64_t* removed,
                      uint32_t* changed, uint64_t* changed_len);
/* peel_exact (peeling.hpp:80, peeling.cpp:202-245).  core (n u64) and
 * dense_vertices (n u32) are optional host outputs. */
int kcg_peel_exact(kcg_graph* g, int k, kcg_peel_result* out, uint64_t* core,
                   uint32_t* dense_vertices);
/* peel_approx (peeling.hpp:87-92, peeling.cpp:247-320); KCG_EINVAL for
 * k < 2 or eps <= 0. */
int kcg_peel_approx(kcg_graph* g, int k, double eps, kcg_peel_result* out,
                    uint32_t* dense_vertices);

/* ---- Colour-sparsified approximate counting (SURVEY.md §8(f) row 3,
 * proj/include/kclique/sampling.hpp:12-43). */

/* SampleEstimate (sampling.hpp:12-19). */
typedef struct kcg_sample_estimate {
  int k;
  uint64_t colors;
  double p;            /* 1 / colors */
  uint64_t sub_count;  /* exact count inside the sparsified graph */
  double estimate;     /* sub_count * colors^(k-1) */
  uint64_t seed;
} kcg_sample_estimate;

/* colorful_sparsify (sampling.cpp:28-40): *out is a new handle holding
 * the subgraph of monochromatic edges.  KCG_EINVAL for colors < 1. */
int kcg_colorful_sparsify(kcg_graph* g, uint64_t colors, uint64_t seed, kcg_graph** out);
/* approx_count (sampling.cpp:42-57): sparsify, rank (strategy / eps /
 * alpha_hat as kcg_rank), orient and count on the device.  KCG_EINVAL for
 * k < 2 or colors < 1. */
int kcg_approx_count(kcg_graph* g, int k, uint64_t colors, uint64_t seed, int strategy,
                     double eps, uint64_t alpha_hat, kcg_sample_estimate* out);

int kcg_timings(const kcg_graph* g, kcg_times* out);
int kcg_last_count_stats(const kcg_graph* g, kcg_count_stats* out);
/* Bytes of device memory the handle currently holds. */
uint64_t kcg_device_bytes(const kcg_graph* g);
/* The CUDA stream (cudaStream_t) all of the handle's work is queued on,
 * for callers that time or order work around it with CUDA events. */
void* kcg_stream(kcg_graph* g);
/* Blocks until all work queued on the handle's stream is done. */
int kcg_synchronize(kcg_graph* g);

#ifdef __cplusplus
}
#endif
#endif /* KCG_H_ */
