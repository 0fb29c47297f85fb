// Host-side synthetic graph generators (see kcgen.h).  Input construction
// is outside the timed hot path; it only has to be
// deterministic and fast enough to build the 537M-sample R-MAT in seconds.
#include "kcgen.h"

#include <omp.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <unordered_set>
#include <vector>

namespace {

inline uint64_t fmix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;

inline uint64_t stream_key(uint64_t seed, uint64_t stream) {
  return fmix(seed * 0xD6E8FEB86659FD93ull + fmix(stream + kGolden));
}
// i-th splitmix64 output for a stream whose state starts at `key`.
inline uint64_t draw(uint64_t key, uint64_t i) {
  return fmix(key + (i + 1) * kGolden);
}
inline double unit_open(uint64_t x) {  // (0, 1)
  return (double(x >> 11) + 0.5) * 0x1.0p-53;
}
inline double unit(uint64_t x) {  // [0, 1)
  return double(x >> 11) * 0x1.0p-53;
}

// Parallel LSD radix sort of u64 keys on the low `bits` bits.
void radix_sort(std::vector<uint64_t>& a, int bits) {
  const size_t n = a.size();
  if (n < 2) return;
  std::vector<uint64_t> tmp(n);
  const int nt = omp_get_max_threads();
  const int passes = (bits + 10) / 11;
  std::vector<size_t> hist(size_t(nt) * 2048);
  uint64_t* src = a.data();
  uint64_t* dst = tmp.data();
  for (int p = 0; p < passes; p++) {
    const int shift = 11 * p;
    std::fill(hist.begin(), hist.end(), 0);
#pragma omp parallel num_threads(nt)
    {
      const int t = omp_get_thread_num();
      const size_t lo = n * t / nt, hi = n * (t + 1) / nt;
      size_t* h = &hist[size_t(t) * 2048];
      for (size_t i = lo; i < hi; i++) h[(src[i] >> shift) & 2047]++;
#pragma omp barrier
#pragma omp single
      {
        size_t run = 0;
        for (int d = 0; d < 2048; d++)
          for (int u = 0; u < nt; u++) {
            size_t c = hist[size_t(u) * 2048 + d];
            hist[size_t(u) * 2048 + d] = run;
            run += c;
          }
      }
      for (size_t i = lo; i < hi; i++) dst[h[(src[i] >> shift) & 2047]++] = src[i];
    }
    std::swap(src, dst);
  }
  if (src != a.data()) std::memcpy(a.data(), src, n * sizeof(uint64_t));
}

int bits_for(uint64_t n) {
  int b = 0;
  while ((uint64_t(1) << b) < n) b++;
  return b;
}

// Keys are (u << 32 | v) with u < v; sorts, dedups and builds the CSR.
int csr_from_keys(uint32_t n, std::vector<uint64_t>& keys, kcgen_csr* out) {
  const int vb = std::max(1, bits_for(n));
  // pack to (u << vb | v) so the radix sort only touches 2*vb bits
  const size_t cnt = keys.size();
#pragma omp parallel for schedule(static)
  for (size_t i = 0; i < cnt; i++) {
    uint64_t k = keys[i];
    keys[i] = ((k >> 32) << vb) | (k & 0xffffffffull);
  }
  radix_sort(keys, 2 * vb);
  keys.erase(std::unique(keys.begin(), keys.end()), keys.end());
  const uint64_t m = keys.size();
  const uint64_t vmask = (uint64_t(1) << vb) - 1;

  std::vector<uint64_t> rev(m);
#pragma omp parallel for schedule(static)
  for (size_t i = 0; i < m; i++) {
    uint64_t u = keys[i] >> vb, v = keys[i] & vmask;
    rev[i] = (v << vb) | u;
  }
  radix_sort(rev, 2 * vb);

  std::vector<uint64_t> hi_start(size_t(n) + 1, 0), lo_start(size_t(n) + 1, 0);
  // run starts for the forward (higher-neighbour) and reversed
  // (lower-neighbour) sorted key arrays
  auto run_starts = [&](const std::vector<uint64_t>& arr, std::vector<uint64_t>& st) {
    std::vector<uint64_t> c(size_t(n) + 1, 0);
    for (size_t i = 0; i < arr.size(); i++) c[(arr[i] >> vb) + 1]++;
    for (size_t x = 0; x < n; x++) c[x + 1] += c[x];
    st.swap(c);
  };
  run_starts(keys, hi_start);
  run_starts(rev, lo_start);

  out->n = n;
  out->m = m;
  out->offsets = static_cast<uint64_t*>(std::malloc((size_t(n) + 1) * 8));
  out->adj = static_cast<uint32_t*>(std::malloc(std::max<size_t>(1, 2 * m) * 4));
  if (!out->offsets || !out->adj) return 3;
  out->offsets[0] = 0;
  for (size_t x = 0; x < n; x++)
    out->offsets[x + 1] = out->offsets[x] + (hi_start[x + 1] - hi_start[x]) +
                          (lo_start[x + 1] - lo_start[x]);
#pragma omp parallel for schedule(dynamic, 4096)
  for (size_t x = 0; x < n; x++) {
    uint64_t p = out->offsets[x];
    for (uint64_t i = lo_start[x]; i < lo_start[x + 1]; i++)
      out->adj[p++] = uint32_t(rev[i] & vmask);
    for (uint64_t i = hi_start[x]; i < hi_start[x + 1]; i++)
      out->adj[p++] = uint32_t(keys[i] & vmask);
  }
  return 0;
}

inline uint64_t key_of(uint32_t u, uint32_t v) {
  if (u > v) std::swap(u, v);
  return (uint64_t(u) << 32) | v;
}

// Drops the entries equal to `drop` while keeping order (parallel).
void compact(std::vector<uint64_t>& a, uint64_t drop) {
  const int nt = omp_get_max_threads();
  const size_t n = a.size();
  std::vector<size_t> cnt(size_t(nt) + 1, 0);
#pragma omp parallel num_threads(nt)
  {
    const int t = omp_get_thread_num();
    const size_t lo = n * t / nt, hi = n * (t + 1) / nt;
    size_t c = 0;
    for (size_t i = lo; i < hi; i++) c += a[i] != drop;
    cnt[t + 1] = c;
#pragma omp barrier
#pragma omp single
    for (int u = 0; u < nt; u++) cnt[u + 1] += cnt[u];
    // in-place is safe: every thread's destination range starts at or
    // before its source range, but threads could overlap each other, so
    // stage through a private buffer.
    std::vector<uint64_t> mine;
    mine.reserve(cnt[t + 1] - cnt[t]);
    for (size_t i = lo; i < hi; i++)
      if (a[i] != drop) mine.push_back(a[i]);
#pragma omp barrier
    std::memcpy(a.data() + cnt[t], mine.data(), mine.size() * 8);
  }
  a.resize(cnt[nt]);
}

}  // namespace

extern "C" {

uint64_t kcgen_draw(uint64_t seed, uint64_t stream, uint64_t i) {
  return draw(stream_key(seed, stream), i);
}

int kcgen_threads(void) { return omp_get_max_threads(); }

int kcgen_er(uint32_t n, uint64_t m, uint64_t seed, kcgen_csr* out) {
  if (n < 2 || m > uint64_t(n) * (n - 1) / 2) return 1;
  const uint64_t key = stream_key(seed, 1);
  std::unordered_set<uint64_t> seen;
  seen.reserve(m * 2);
  std::vector<uint64_t> keys;
  keys.reserve(m);
  for (uint64_t i = 0; keys.size() < m; i++) {
    uint64_t r = draw(key, i);
    uint32_t u = uint32_t(((r >> 32) * n) >> 32);
    uint32_t v = uint32_t(((r & 0xffffffffull) * n) >> 32);
    if (u == v) continue;
    uint64_t k = key_of(u, v);
    if (seen.insert(k).second) keys.push_back(k);
  }
  return csr_from_keys(n, keys, out);
}

int kcgen_rmat(int scale, uint64_t samples, double a, double b, double c,
               uint64_t seed, int permute, kcgen_csr* out) {
  if (scale < 1 || scale > 31) return 1;
  const uint32_t n = uint32_t(1) << scale;
  // integer thresholds on the 53-bit uniform so every platform agrees
  const double two53 = 0x1.0p53;
  const uint64_t t1 = uint64_t(a * two53);
  const uint64_t t2 = uint64_t((a + b) * two53);
  const uint64_t t3 = uint64_t((a + b + c) * two53);
  const uint64_t key = stream_key(seed, 1);
  const uint64_t loop = ~uint64_t(0);

  std::vector<uint32_t> perm;
  if (permute) {
    perm.resize(n);
    for (uint32_t i = 0; i < n; i++) perm[i] = i;
    const uint64_t pk = stream_key(seed, 2);
    for (uint32_t i = n - 1; i > 0; i--) {
      uint32_t j = uint32_t(draw(pk, i) % (uint64_t(i) + 1));
      std::swap(perm[i], perm[j]);
    }
  }
  std::vector<uint64_t> keys(samples);
#pragma omp parallel for schedule(static)
  for (uint64_t e = 0; e < samples; e++) {
    uint32_t u = 0, v = 0;
    const uint64_t base = e * uint64_t(scale);
    for (int l = 0; l < scale; l++) {
      uint64_t r = draw(key, base + l) >> 11;
      uint32_t bit = uint32_t(1) << (scale - 1 - l);
      if (r < t1) {
      } else if (r < t2) {
        v |= bit;
      } else if (r < t3) {
        u |= bit;
      } else {
        u |= bit;
        v |= bit;
      }
    }
    if (permute) {
      u = perm[u];
      v = perm[v];
    }
    keys[e] = (u == v) ? loop : key_of(u, v);
  }
  compact(keys, loop);
  return csr_from_keys(n, keys, out);
}

int kcgen_chung_lu(uint32_t n, double gamma, double i0, double mean,
                   double wmin, double wmax, uint64_t seed, kcgen_csr* out) {
  if (n < 2 || gamma <= 1 || mean <= 0) return 1;
  const double expo = -1.0 / (gamma - 1.0);
  std::vector<double> base(n), w(n);
#pragma omp parallel for schedule(static)
  for (uint32_t i = 0; i < n; i++) base[i] = std::pow(double(i) + i0, expo);
  // clipped mean as a function of the scale; fixed 64-way chunked sum so
  // the rounding does not depend on the thread count
  auto clipped_sum = [&](double cscale, bool store) {
    double part[64];
#pragma omp parallel for schedule(static)
    for (int ch = 0; ch < 64; ch++) {
      size_t lo = size_t(n) * ch / 64, hi = size_t(n) * (ch + 1) / 64;
      double s = 0;
      for (size_t i = lo; i < hi; i++) {
        double x = std::min(wmax, std::max(wmin, cscale * base[i]));
        if (store) w[i] = x;
        s += x;
      }
      part[ch] = s;
    }
    double s = 0;
    for (int ch = 0; ch < 64; ch++) s += part[ch];
    return s;
  };
  double lo = 0, hi = 1;
  while (clipped_sum(hi, false) / n < mean) hi *= 2;
  for (int it = 0; it < 200; it++) {
    double mid = 0.5 * (lo + hi);
    if (clipped_sum(mid, false) / n < mean)
      lo = mid;
    else
      hi = mid;
  }
  const double S = clipped_sum(hi, true);

  // Miller-Hagberg (2011) skipping sampler over non-increasing weights,
  // one counter-based random stream per source vertex.
  const int nt = omp_get_max_threads();
  std::vector<std::vector<uint64_t>> parts(nt);
#pragma omp parallel num_threads(nt)
  {
    auto& mine = parts[omp_get_thread_num()];
#pragma omp for schedule(dynamic, 256)
    for (uint32_t u = 0; u < n - 1; u++) {
      const uint64_t key = stream_key(seed, 3 + (uint64_t(u) << 8));
      uint64_t ctr = 0;
      uint64_t v = uint64_t(u) + 1;
      double p = std::min(w[u] * w[v] / S, 1.0);
      while (v < n && p > 0) {
        if (p != 1.0) {
          double r = unit_open(draw(key, ctr++));
          double skip = std::floor(std::log(r) / std::log(1.0 - p));
          if (skip >= double(n)) break;
          v += uint64_t(skip);
        }
        if (v < n) {
          double q = std::min(w[u] * w[v] / S, 1.0);
          double r = unit_open(draw(key, ctr++));
          if (r < q / p) mine.push_back((uint64_t(u) << 32) | uint32_t(v));
          p = q;
          v++;
        }
      }
    }
  }
  size_t total = 0;
  for (auto& p : parts) total += p.size();
  std::vector<uint64_t> keys;
  keys.reserve(total);
  for (auto& p : parts) {
    keys.insert(keys.end(), p.begin(), p.end());
    std::vector<uint64_t>().swap(p);
  }
  return csr_from_keys(n, keys, out);
}

int kcgen_rgg(uint32_t n, double mean_deg, uint64_t seed, kcgen_csr* out) {
  if (n < 2 || mean_deg <= 0) return 1;
  const double r = std::sqrt(mean_deg / (M_PI * double(n - 1)));
  const double r2 = r * r;
  const uint64_t key = stream_key(seed, 4);
  std::vector<double> x(n), y(n);
#pragma omp parallel for schedule(static)
  for (uint32_t i = 0; i < n; i++) {
    x[i] = unit(draw(key, 2 * uint64_t(i)));
    y[i] = unit(draw(key, 2 * uint64_t(i) + 1));
  }
  const uint32_t G = std::max<uint32_t>(1, uint32_t(1.0 / r));
  auto cell_of = [&](uint32_t i) {
    uint32_t cx = std::min<uint32_t>(G - 1, uint32_t(x[i] * G));
    uint32_t cy = std::min<uint32_t>(G - 1, uint32_t(y[i] * G));
    return uint64_t(cy) * G + cx;
  };
  const uint64_t cells = uint64_t(G) * G;
  std::vector<uint64_t> start(cells + 1, 0);
  std::vector<uint32_t> cell(n);
  for (uint32_t i = 0; i < n; i++) {
    cell[i] = uint32_t(cell_of(i));
    start[cell[i] + 1]++;
  }
  for (uint64_t c = 0; c < cells; c++) start[c + 1] += start[c];
  std::vector<uint32_t> pts(n);
  {
    std::vector<uint64_t> cur(start.begin(), start.end() - 1);
    for (uint32_t i = 0; i < n; i++) pts[cur[cell[i]]++] = i;
  }
  const int nt = omp_get_max_threads();
  std::vector<std::vector<uint64_t>> parts(nt);
#pragma omp parallel num_threads(nt)
  {
    auto& mine = parts[omp_get_thread_num()];
#pragma omp for schedule(dynamic, 1024)
    for (uint32_t i = 0; i < n; i++) {
      const int64_t cx = cell[i] % G, cy = cell[i] / G;
      for (int64_t dy = -1; dy <= 1; dy++)
        for (int64_t dx = -1; dx <= 1; dx++) {
          int64_t ax = cx + dx, ay = cy + dy;
          if (ax < 0 || ay < 0 || ax >= int64_t(G) || ay >= int64_t(G)) continue;
          uint64_t c = uint64_t(ay) * G + uint64_t(ax);
          for (uint64_t p = start[c]; p < start[c + 1]; p++) {
            uint32_t j = pts[p];
            if (j <= i) continue;
            double ddx = x[i] - x[j], ddy = y[i] - y[j];
            double d2 = ddx * ddx;
            d2 += ddy * ddy;
            if (d2 < r2) mine.push_back((uint64_t(i) << 32) | j);
          }
        }
    }
  }
  std::vector<uint64_t> keys;
  size_t total = 0;
  for (auto& p : parts) total += p.size();
  keys.reserve(total);
  for (auto& p : parts) keys.insert(keys.end(), p.begin(), p.end());
  return csr_from_keys(n, keys, out);
}

int kcgen_from_edges(uint32_t n, const uint32_t* us, const uint32_t* vs,
                     uint64_t count, kcgen_csr* out) {
  std::vector<uint64_t> keys;
  keys.reserve(count);
  for (uint64_t i = 0; i < count; i++) {
    if (us[i] >= n || vs[i] >= n) return 1;
    if (us[i] != vs[i]) keys.push_back(key_of(us[i], vs[i]));
  }
  if (n == 0) {
    out->n = 0;
    out->m = 0;
    out->offsets = static_cast<uint64_t*>(std::calloc(1, 8));
    out->adj = static_cast<uint32_t*>(std::malloc(4));
    return 0;
  }
  return csr_from_keys(n, keys, out);
}

uint64_t kcgen_digest_u32(const uint32_t* a, uint64_t len) {
  uint64_t s = 0;
#pragma omp parallel for reduction(+ : s) schedule(static)
  for (uint64_t i = 0; i < len; i++) s += fmix(i * kGolden + a[i] + 1);
  return s;
}

uint64_t kcgen_digest_u64(const uint64_t* a, uint64_t len) {
  uint64_t s = 0;
#pragma omp parallel for reduction(+ : s) schedule(static)
  for (uint64_t i = 0; i < len; i++) s += fmix(fmix(i * kGolden + 7) ^ a[i]);
  return s;
}

int kcgen_save(const char* path, const kcgen_csr* g) {
  FILE* f = std::fopen(path, "wb");
  if (!f) return 2;
  const char magic[8] = {'K', 'C', 'S', 'R', '0', '0', '0', '1'};
  bool ok = std::fwrite(magic, 1, 8, f) == 8 && std::fwrite(&g->n, 8, 1, f) == 1 &&
            std::fwrite(&g->m, 8, 1, f) == 1 &&
            std::fwrite(g->offsets, 8, g->n + 1, f) == g->n + 1 &&
            std::fwrite(g->adj, 4, 2 * g->m, f) == 2 * g->m;
  ok = (std::fclose(f) == 0) && ok;
  return ok ? 0 : 2;
}

int kcgen_load(const char* path, kcgen_csr* out) {
  FILE* f = std::fopen(path, "rb");
  if (!f) return 2;
  char magic[8];
  bool ok = std::fread(magic, 1, 8, f) == 8 && std::memcmp(magic, "KCSR0001", 8) == 0 &&
            std::fread(&out->n, 8, 1, f) == 1 && std::fread(&out->m, 8, 1, f) == 1;
  if (ok) {
    out->offsets = static_cast<uint64_t*>(std::malloc((out->n + 1) * 8));
    out->adj = static_cast<uint32_t*>(std::malloc(std::max<uint64_t>(1, 2 * out->m) * 4));
    ok = out->offsets && out->adj &&
         std::fread(out->offsets, 8, out->n + 1, f) == out->n + 1 &&
         std::fread(out->adj, 4, 2 * out->m, f) == 2 * out->m;
  }
  std::fclose(f);
  return ok ? 0 : 2;
}

void kcgen_free(kcgen_csr* g) {
  if (!g) return;
  std::free(g->offsets);
  std::free(g->adj);
  g->offsets = nullptr;
  g->adj = nullptr;
}

}  // extern "C"
