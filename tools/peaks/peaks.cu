// Microbenchmarks for the counting roofline (SURVEY.md §7.1 "Peaks to
// measure", §8(d) "Roof selection"): the denominators that MEASURED_PEAKS.json
// does not carry.
//
//   l2_read      LDG.128 sweeps over a working set that fits the 126 MB L2
//                (16 .. 96 MB, the DAG sizes of configs 1-2), all SMs
//   hbm_read     the same over 8 GB (compulsory-traffic roof, configs 3-5)
//   lop3/popc/iadd3/vote/lds/atoms_or
//                per-SM issue rates of the instructions the counting
//                recursion is made of (clique_rec.hpp:49-60 becomes
//                AND / POPC / BALLOT on bitmap words), 32 warps per SM,
//                8 independent chains per thread
//   sm clock     clock64() cycles of every CTA / event time = the SM clock
//                the rates were measured at
//
// Prints one JSON object.  Build: make -C tools/peaks (nvcc, sm_100a).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <algorithm>
#include <string>
#include <vector>

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e = (x);                                                             \
    if (e != cudaSuccess) {                                                          \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); \
      exit(1);                                                                       \
    }                                                                                \
  } while (0)

__device__ unsigned long long g_sink;
__device__ unsigned long long g_cycles[4096];

// ---- bandwidth -----------------------------------------------------------------
__global__ void __launch_bounds__(512) read_kernel(const uint4* __restrict__ p, size_t n4, int reps) {
  uint32_t acc = 0;
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  for (int r = 0; r < reps; r++) {
    size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    // 4 loads in flight per thread
    for (; i + 3 * stride < n4; i += 4 * stride) {
      uint4 a = __ldcg(p + i), b = __ldcg(p + i + stride), c = __ldcg(p + i + 2 * stride),
            d = __ldcg(p + i + 3 * stride);
      acc ^= a.x ^ a.y ^ a.z ^ a.w ^ b.x ^ b.y ^ b.z ^ b.w ^ c.x ^ c.y ^ c.z ^ c.w ^ d.x ^ d.y ^
             d.z ^ d.w;
    }
    for (; i < n4; i += stride) {
      uint4 a = __ldcg(p + i);
      acc ^= a.x ^ a.y ^ a.z ^ a.w;
    }
  }
  if (acc == 0x12345678u) g_sink = acc;
}

// ---- issue rates -----------------------------------------------------------------
// OP: 0 lop3 (and), 1 popc, 2 iadd3, 3 vote.ballot, 4 lds.32, 5 atoms.or (spread)
template <int OP>
__global__ void __launch_bounds__(256) issue_kernel(int iters, uint32_t seed) {
  __shared__ uint32_t sm[1024 * 2];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) sm[i] = i * seed;
  // the per-lane atomics target lane + 32 * warp: 8 warps per CTA
  __syncthreads();
  const long long t0 = clock64();
  uint32_t a0 = threadIdx.x ^ seed, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, a4 = a0 * 11,
           a5 = a0 * 13, a6 = a0 * 17, a7 = a0 * 19;
  const uint32_t k = seed | 1u;
#pragma unroll 1
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int u = 0; u < 16; u++) {
      if (OP == 0) {
        // 3-input XOR across the chains (LOP3.LUT 0x96), not foldable
        asm volatile(
            "lop3.b32 %0, %0, %1, %8, 0x96;\n\tlop3.b32 %1, %1, %2, %8, 0x96;\n\t"
            "lop3.b32 %2, %2, %3, %8, 0x96;\n\tlop3.b32 %3, %3, %4, %8, 0x96;\n\t"
            "lop3.b32 %4, %4, %5, %8, 0x96;\n\tlop3.b32 %5, %5, %6, %8, 0x96;\n\t"
            "lop3.b32 %6, %6, %7, %8, 0x96;\n\tlop3.b32 %7, %7, %0, %8, 0x96;"
            : "+r"(a0), "+r"(a1), "+r"(a2), "+r"(a3), "+r"(a4), "+r"(a5), "+r"(a6), "+r"(a7)
            : "r"(k));
      } else if (OP == 1) {
        asm volatile(
            "popc.b32 %0, %0;\n\tpopc.b32 %1, %1;\n\tpopc.b32 %2, %2;\n\t"
            "popc.b32 %3, %3;\n\tpopc.b32 %4, %4;\n\tpopc.b32 %5, %5;\n\t"
            "popc.b32 %6, %6;\n\tpopc.b32 %7, %7;"
            : "+r"(a0), "+r"(a1), "+r"(a2), "+r"(a3), "+r"(a4), "+r"(a5), "+r"(a6), "+r"(a7));
      } else if (OP == 2) {
        asm volatile(
            "add.u32 %0, %0, %8;\n\tadd.u32 %1, %1, %8;\n\tadd.u32 %2, %2, %8;\n\t"
            "add.u32 %3, %3, %8;\n\tadd.u32 %4, %4, %8;\n\tadd.u32 %5, %5, %8;\n\t"
            "add.u32 %6, %6, %8;\n\tadd.u32 %7, %7, %8;"
            : "+r"(a0), "+r"(a1), "+r"(a2), "+r"(a3), "+r"(a4), "+r"(a5), "+r"(a6), "+r"(a7)
            : "r"(k));
      } else if (OP == 3) {
        // a = ballot(a != 0): one ISETP + one VOTE per ballot (ptxas merges
        // ballots of the same predicate, so each needs its own)
        asm volatile(
            "{.reg .pred p;\n\t"
            "setp.ne.u32 p, %0, 0; vote.sync.ballot.b32 %0, p, 0xffffffff;\n\t"
            "setp.ne.u32 p, %1, 0; vote.sync.ballot.b32 %1, p, 0xffffffff;\n\t"
            "setp.ne.u32 p, %2, 0; vote.sync.ballot.b32 %2, p, 0xffffffff;\n\t"
            "setp.ne.u32 p, %3, 0; vote.sync.ballot.b32 %3, p, 0xffffffff;\n\t"
            "setp.ne.u32 p, %4, 0; vote.sync.ballot.b32 %4, p, 0xffffffff;\n\t"
            "setp.ne.u32 p, %5, 0; vote.sync.ballot.b32 %5, p, 0xffffffff;\n\t"
            "setp.ne.u32 p, %6, 0; vote.sync.ballot.b32 %6, p, 0xffffffff;\n\t"
            "setp.ne.u32 p, %7, 0; vote.sync.ballot.b32 %7, p, 0xffffffff;}"
            : "+r"(a0), "+r"(a1), "+r"(a2), "+r"(a3), "+r"(a4), "+r"(a5), "+r"(a6), "+r"(a7));
      } else if (OP == 4) {
        // conflict-free: the row (32 words) depends on the loaded value, the
        // word is the lane's own bank
        const uint32_t ln = threadIdx.x & 31;
        a0 = sm[((a0 & 31u) << 5) + ln];
        a1 = sm[((a1 & 31u) << 5) + ln + 1024];
        a2 = sm[((a2 & 31u) << 5) + ln];
        a3 = sm[((a3 & 31u) << 5) + ln + 1024];
        a4 = sm[((a4 & 31u) << 5) + ln];
        a5 = sm[((a5 & 31u) << 5) + ln + 1024];
        a6 = sm[((a6 & 31u) << 5) + ln];
        a7 = sm[((a7 & 31u) << 5) + ln + 1024];
      } else if (OP == 6) {
        // SHFL.IDX with a data-dependent source lane
        a0 = __shfl_sync(0xffffffffu, a0, a1);
        a1 = __shfl_sync(0xffffffffu, a1, a2);
        a2 = __shfl_sync(0xffffffffu, a2, a3);
        a3 = __shfl_sync(0xffffffffu, a3, a4);
        a4 = __shfl_sync(0xffffffffu, a4, a5);
        a5 = __shfl_sync(0xffffffffu, a5, a6);
        a6 = __shfl_sync(0xffffffffu, a6, a7);
        a7 = __shfl_sync(0xffffffffu, a7, a0);
      } else if (OP == 7) {
        // FLO (__ffs = BREV + FLO.SH; __clz = FLO)
        a0 = __clz(a0 ^ k); a1 = __clz(a1 ^ k); a2 = __clz(a2 ^ k); a3 = __clz(a3 ^ k);
        a4 = __clz(a4 ^ k); a5 = __clz(a5 ^ k); a6 = __clz(a6 ^ k); a7 = __clz(a7 ^ k);
      } else if (OP == 8) {
        // REDUX.OR (warp OR-reduction)
        a0 = __reduce_or_sync(0xffffffffu, a0 + k); a1 = __reduce_or_sync(0xffffffffu, a1 + k);
        a2 = __reduce_or_sync(0xffffffffu, a2 + k); a3 = __reduce_or_sync(0xffffffffu, a3 + k);
        a4 = __reduce_or_sync(0xffffffffu, a4 + k); a5 = __reduce_or_sync(0xffffffffu, a5 + k);
        a6 = __reduce_or_sync(0xffffffffu, a6 + k); a7 = __reduce_or_sync(0xffffffffu, a7 + k);
      } else if (OP == 9) {
        // random-bank LDS: the expected conflict degree of 32 random words
        const uint32_t m = 2047u;
        a0 = sm[(a0 * 0x9E3779B1u >> 21) & m];
        a1 = sm[(a1 * 0x9E3779B1u >> 21) & m];
        a2 = sm[(a2 * 0x9E3779B1u >> 21) & m];
        a3 = sm[(a3 * 0x9E3779B1u >> 21) & m];
        a4 = sm[(a4 * 0x9E3779B1u >> 21) & m];
        a5 = sm[(a5 * 0x9E3779B1u >> 21) & m];
        a6 = sm[(a6 * 0x9E3779B1u >> 21) & m];
        a7 = sm[(a7 * 0x9E3779B1u >> 21) & m];
      } else {
        // distinct banks, distinct words per lane
        const uint32_t base = (threadIdx.x & 31) + 32 * (threadIdx.x >> 5);
        atomicOr(&sm[base], a0);
        atomicOr(&sm[base], a1);
        atomicOr(&sm[base], a2);
        atomicOr(&sm[base], a3);
        atomicOr(&sm[base], a4);
        atomicOr(&sm[base], a5);
        atomicOr(&sm[base], a6);
        atomicOr(&sm[base], a7);
        a0 += k;
        a1 += k;
      }
    }
  }
  const long long t1 = clock64();
  const uint32_t r = a0 ^ a1 ^ a2 ^ a3 ^ a4 ^ a5 ^ a6 ^ a7 ^ sm[threadIdx.x];
  if (r == 0x9abcdef1u) g_sink = r;
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = (unsigned long long)(t1 - t0);
}

static float time_ms(void (*launch)(void*), void* arg, int reps) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  launch(arg);  // warm
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < reps; r++) {
    CK(cudaEventRecord(a));
    launch(arg);
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    best = std::min(best, ms);
  }
  CK(cudaEventDestroy(a));
  CK(cudaEventDestroy(b));
  return best;
}

struct ReadArg {
  const uint4* p;
  size_t n4;
  int reps, grid;
};
static void launch_read(void* v) {
  ReadArg* a = static_cast<ReadArg*>(v);
  read_kernel<<<a->grid, 512>>>(a->p, a->n4, a->reps);
}

struct IssueArg {
  int op, iters, grid;
};
template <int OP>
static void launch_issue_t(IssueArg* a) {
  issue_kernel<OP><<<a->grid, 256>>>(a->iters, 0x2545F491u);
}
static void launch_issue(void* v) {
  IssueArg* a = static_cast<IssueArg*>(v);
  switch (a->op) {
    case 6: launch_issue_t<6>(a); break;
    case 7: launch_issue_t<7>(a); break;
    case 8: launch_issue_t<8>(a); break;
    case 9: launch_issue_t<9>(a); break;
    case 0: launch_issue_t<0>(a); break;
    case 1: launch_issue_t<1>(a); break;
    case 2: launch_issue_t<2>(a); break;
    case 3: launch_issue_t<3>(a); break;
    case 4: launch_issue_t<4>(a); break;
    default: launch_issue_t<5>(a); break;
  }
}

int main() {
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  const int sms = prop.multiProcessorCount;
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"l2_bytes\": %d, \"smem_optin\": %zu", prop.name, sms,
         prop.l2CacheSize, prop.sharedMemPerBlockOptin);
  // ---- L2 read bandwidth over DAG-sized working sets
  const size_t big = size_t(8) << 30;
  uint4* buf;
  CK(cudaMalloc(&buf, big));
  CK(cudaMemset(buf, 1, big));
  printf(", \"l2_read\": [");
  double l2_best = 0;
  const int mbs[] = {16, 32, 48, 64, 72, 96};
  for (int i = 0; i < 6; i++) {
    const size_t bytes = size_t(mbs[i]) << 20;
    ReadArg a{buf, bytes / 16, 20, sms * 4};
    float ms = time_ms(launch_read, &a, 5);
    const double gbs = double(bytes) * a.reps / (ms * 1e-3) / 1e9;
    l2_best = std::max(l2_best, gbs);
    printf("%s{\"mb\": %d, \"gbs\": %.1f}", i ? ", " : "", mbs[i], gbs);
  }
  printf("], \"l2_read_gbs\": %.1f", l2_best);
  {
    ReadArg a{buf, big / 16, 1, sms * 4};
    float ms = time_ms(launch_read, &a, 3);
    printf(", \"hbm_read_gbs\": %.1f", double(big) / (ms * 1e-3) / 1e9);
  }
  CK(cudaFree(buf));
  // ---- issue rates: warp instructions per SM per cycle, and the clock
  const char* names[] = {"lop3", "popc", "iadd", "vote_ballot_with_isetp", "lds32_conflict_free", "atoms_or_distinct_banks", "shfl_idx", "flo_clz", "redux_or", "lds32_random_banks"};
  printf(", \"issue\": {");
  for (int op = 0; op < 10; op++) {
    // 8 CTAs x 256 threads = 64 warps per SM, all co-resident
    IssueArg a{op, (op == 4 || op == 5 || op == 9) ? 256 : 1024, sms * 8};
    float ms = time_ms(launch_issue, &a, 3);
    std::vector<unsigned long long> cyc(a.grid);
    CK(cudaMemcpyFromSymbol(cyc.data(), g_cycles, sizeof(unsigned long long) * a.grid));
    const double cmax = double(*std::max_element(cyc.begin(), cyc.end()));
    const double mhz = cmax / (ms * 1e-3) / 1e6;
    const double warp_inst = double(a.grid) * (256 / 32) * a.iters * 16 * 8;  // per op kind
    const double per_sm_cycle = warp_inst / sms / (double(ms) * 1e-3 * mhz * 1e6);
    const double lane_ops = warp_inst * 32.0 / (ms * 1e-3);
    printf("%s\"%s\": {\"warp_inst_per_sm_cycle\": %.3f, \"lane_ops_per_s\": %.4g, \"sm_mhz\": %.0f, "
           "\"ms\": %.3f}",
           op ? ", " : "", names[op], per_sm_cycle, lane_ops, mhz, ms);
  }
  printf("}}\n");
  return 0;
}
