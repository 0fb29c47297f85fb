/* Synthetic graph generators and CSR normalisation for the five benchmark
 * configurations.  Host-only C ABI (OpenMP inside).
 *
 * The reference ships no generators; these define the
 * canonical inputs shared by the GPU path, the CPU reference arm and the
 * golden fixtures.  Every random draw is a pure function of
 * (seed, stream, index) so output is identical for any thread count.
 *
 * Normalisation follows Graph::from_edges semantics
 * (proj/src/graph.cpp:11-41): endpoints swapped to u<v, self-loops dropped,
 * duplicates removed, symmetric CSR with ascending slices.
 */
#pragma once
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct kcgen_csr {
  uint64_t n;        /* vertices */
  uint64_t m;        /* undirected edges */
  uint64_t* offsets; /* n+1 */
  uint32_t* adj;     /* 2m */
} kcgen_csr;

/* Counter-based generator: the i-th output of splitmix64 seeded with
 * a key derived from (seed, stream). */
uint64_t kcgen_draw(uint64_t seed, uint64_t stream, uint64_t i);

/* Erdos-Renyi G(n, m): m distinct unordered pairs u != v, uniform, by
 * rejection.  Returns 0 on success. */
int kcgen_er(uint32_t n, uint64_t m, uint64_t seed, kcgen_csr* out);

/* R-MAT with 2^scale vertices and `samples` edge draws, quadrant
 * probabilities (a, b, c, 1-a-b-c), no noise.  permute != 0 relabels ids
 * by a seeded Fisher-Yates shuffle. */
int kcgen_rmat(int scale, uint64_t samples, double a, double b, double c,
               uint64_t seed, int permute, kcgen_csr* out);

/* Chung-Lu: w_i = clip(C * (i + i0)^(-1/(gamma-1)), wmin, wmax) with C
 * chosen so the clipped mean is `mean`; edge (i,j) kept with probability
 * min(1, w_i w_j / sum w), sampled with Miller-Hagberg skipping. */
int kcgen_chung_lu(uint32_t n, double gamma, double i0, double mean,
                   double wmin, double wmax, uint64_t seed, kcgen_csr* out);

/* Random geometric graph: n uniform points in [0,1)^2, edge iff
 * dx*dx + dy*dy < r*r with r = sqrt(mean_deg / (pi (n-1))). */
int kcgen_rgg(uint32_t n, double mean_deg, uint64_t seed, kcgen_csr* out);

/* Normalise an arbitrary edge list (from_edges semantics).  Returns 1 if
 * an endpoint is >= n. */
int kcgen_from_edges(uint32_t n, const uint32_t* us, const uint32_t* vs,
                     uint64_t count, kcgen_csr* out);

/* Order-independent 64-bit digests (sum of position-tagged mixes). */
uint64_t kcgen_digest_u32(const uint32_t* a, uint64_t len);
uint64_t kcgen_digest_u64(const uint64_t* a, uint64_t len);

int kcgen_save(const char* path, const kcgen_csr* g);
int kcgen_load(const char* path, kcgen_csr* out);
void kcgen_free(kcgen_csr* g);
int kcgen_threads(void);

#ifdef __cplusplus
}
#endif
