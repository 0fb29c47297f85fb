#!/usr/bin/env python3
"""arb-count benchmark on B200 (contract: DESIGN.md §Measurement).

Default workload = BASELINE.json configs[1]: R-MAT scale 20 (16,777,216
samples, seed 2, permuted ids), Barenboim-Elkin ranking (eps = 0.5, alpha
estimated), k = 4.  One step = one pass of the hot path over the graph
resident in HBM: rank -> orient (DAG) -> count.  k = 5 on the same DAG is
reported as a secondary measurement.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl kcg|reference]
                    [--config C] [--k K] [--no-cpu-baseline]

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import subprocess
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_2002_10047_b200 import gen  # noqa: E402

STRAT_NAMES = {0: "degree", 1: "original", 2: "kcore", 3: "goodrich_pszona",
               4: "barenboim_elkin", 5: "kcore_parallel"}
FALLBACK_HBM_GBS = 6650.0


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["kcg", "reference"], default="kcg")
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--k", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sweep", action="store_true",
                    help="skip the per-config sweep reported under `configs`")
    ap.add_argument("--no-config5", action="store_true",
                    help="skip the instrumented config-5 block")
    ap.add_argument("--cpu-budget-s", type=float, default=240.0,
                    help="wall budget for the reference arm's timed steps")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def workload(cfg_id, k):
    spec = gen.CONFIGS[cfg_id]
    k = k or spec["ks"][0]
    return spec, k


def config_obj(cfg_id, spec, k, g, extra=None):
    c = {"workload": f"config{cfg_id}: {spec['desc']}", "k": k,
         "strategy": STRAT_NAMES[gen.gpu_strategy(spec)], "eps": spec["eps"], "n": g.n, "m": g.m,
         "step": "rank + orient (DAG) + count_total",
         "l2": "flushed between timed steps (512 MiB memset on the library stream)"}
    if extra:
        c.update(extra)
    return c


# ---------------------------------------------------------------------------
# clocks sampled during the timed region
# ---------------------------------------------------------------------------
class ClockSampler:
    """Samples SM clocks and clock-event reasons every ~5 ms through NVML on
    a background thread while the timed region runs (nvidia-smi's -lms loop
    needs ~0.3 s to start, longer than a short timed region)."""

    REASONS = [("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"),
               ("hw_power_brake_slowdown", "nvmlClocksEventReasonHwPowerBrakeSlowdown")]

    def __init__(self, index=0, period_s=0.005):
        self.index = index
        self.period = period_s
        self.rows = []
        self.max_mhz = None
        self._stop = threading.Event()
        self.thread = None

    def start(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = int(vis.split(",")[self.index]) if vis and vis.split(",")[0].isdigit() \
                else self.index
            self.h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self.nv = pynvml
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:  # noqa: BLE001 - no NVML: report unsampled
            self.nv = None
            return
        self.thread = threading.Thread(target=self._run, daemon=True)
        self.thread.start()

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.rows.append((sm, rs))
            except Exception:  # noqa: BLE001
                pass
            self._stop.wait(self.period)

    def stop(self):
        self._stop.set()
        if self.thread:
            self.thread.join(timeout=2)
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"]}
        reasons = sorted({name for _, rs in self.rows for name, attr in self.REASONS
                          if rs & getattr(self.nv, attr, 0)})
        return {"sm_mhz": statistics.median(sm for sm, _ in self.rows),
                "sm_max_mhz": self.max_mhz, "reasons": reasons, "samples": len(self.rows),
                "source": "NVML, every %.0f ms during the timed steps" % (1e3 * self.period)}


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        d = json.load(open(path))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def counting_peaks():
    """The §8(d) roof denominators: HBM from MEASURED_PEAKS.json (driver-
    measured copy), L2 read bandwidth and the POPC issue rate from our own
    microbenchmark on the B200 (tools/peaks/peaks.cu -> profiles/r02_peaks.json:
    LDG.128 sweeps over 16-96 MB working sets; POPC at 16 lanes per SM per
    clock, one eighth of LOP3/IADD3)."""
    hbm, hbm_src = measured_peaks()
    p = {"hbm_gbs": hbm, "hbm_source": hbm_src}
    path = os.path.join(ROOT, "profiles", "r02_peaks.json")
    if os.path.exists(path):
        d = json.load(open(path))
        iss = d["issue"]
        p.update({"l2_gbs": float(d["l2_read_gbs"]),
                  "popc_lane_ops_per_s": float(iss["popc"]["lane_ops_per_s"]),
                  "popc_warp_inst_per_sm_cycle": float(iss["popc"]["warp_inst_per_sm_cycle"]),
                  "peaks_source": "measured (profiles/r02_peaks.json, tools/peaks/peaks.cu)"})
    return p


def ops_table():
    """OPS(k) of SURVEY.md §8(d) (one AND + one POPC per bitmap word of every
    intersection the reference's edge engine performs): tools/kc_ops.c, an
    instrumented restatement of clique_rec.hpp:24-62, totals cross-checked
    against the goldens (profiles/r01_ops_k.jsonl)."""
    out = {}
    path = os.path.join(ROOT, "profiles", "r01_ops_k.jsonl")
    if os.path.exists(path):
        for line in open(path):
            d = json.loads(line)
            out[(d["config"], d["k"])] = int(d["ops"])
    return out


def roofline_entry(cid, k, n, m, sum_io, count_ms, peaks, ops, l2_bytes, per_vertex=False,
                   t3=None):
    """SURVEY.md §8(d) roof selection for one (config, k) count:
    T_roof = max(B_alg / BW, (OPS / 2) / P_popc), BW = measured L2 when the
    DAG (8(n+1) + 4m bytes) fits in L2, else measured HBM; OPS counts an AND
    and a POPC per word, and POPC (16 lanes/SM/clk) is the binding integer
    pipe.  frac = T_roof / T_measured."""
    b_alg = 16.0 * n + 20.0 * m + 4.0 * sum_io
    if per_vertex and t3 is not None:
        b_alg += 16.0 * (t3 + 2.0 * m)  # u64 per-vertex atomics (§8(d))
    dag_bytes = 8.0 * (n + 1) + 4.0 * m
    fits = bool(l2_bytes) and dag_bytes <= l2_bytes and "l2_gbs" in peaks
    bw = peaks["l2_gbs"] if fits else peaks["hbm_gbs"]
    t_bytes = b_alg / (bw * 1e9)
    op = None if per_vertex else ops.get((cid, k))
    t_ops = (op / 2.0) / peaks["popc_lane_ops_per_s"] \
        if op and "popc_lane_ops_per_s" in peaks else None
    t = count_ms / 1e3
    e = {"alg_bytes": b_alg, "dag_bytes": dag_bytes, "bw_roof": "l2" if fits else "hbm",
         "bw_peak_gbs": bw, "t_bytes_ms": t_bytes * 1e3,
         "ops": op, "t_issue_ms": t_ops * 1e3 if t_ops else None,
         "count_ms": count_ms}
    if t_ops and t_ops > t_bytes:
        e.update({"bound": "int_issue_popc", "achieved": (op / 2.0) / t / 1e12,
                  "peak": peaks["popc_lane_ops_per_s"] / 1e12, "unit": "Tpopc/s"})
    else:
        e.update({"bound": e["bw_roof"], "achieved": b_alg / t / 1e9, "peak": bw,
                  "unit": "GB/s"})
    e["frac"] = max(t_bytes, t_ops or 0.0) / t
    e["hbm_frac"] = b_alg / t / 1e9 / peaks["hbm_gbs"]
    return e


def phase_rooflines(strat, n, m, rank_ms, direct_ms, peaks):
    """SURVEY.md §8(d) byte formulas for the streaming phases against measured
    HBM: degree ranking 8(n+1) + 4n; DAG build 16(n+1) + 8m + 8m + 4n + 4m
    (offsets, adjacency, rank gathers, writes).  The round-based rankings read
    at least 5n + 8(n+1) + 8m (first round's scan + every adjacency entry once):
    quoted as a lower bound on their bytes."""
    hbm = peaks["hbm_gbs"]
    out = {}
    if strat == 0:
        rb, note = 8.0 * (n + 1) + 4.0 * n, "degree: 8(n+1) + 4n"
    else:
        rb, note = 5.0 * n + 8.0 * (n + 1) + 8.0 * m, "lower bound: 5n + 8(n+1) + 8m"
    if rank_ms:
        out["rank"] = {"alg_bytes": rb, "formula": note, "ms": rank_ms, "bound": "hbm",
                       "achieved": rb / (rank_ms / 1e3) / 1e9, "peak": hbm, "unit": "GB/s",
                       "frac": rb / (rank_ms / 1e3) / 1e9 / hbm}
    db = 16.0 * (n + 1) + 20.0 * m + 4.0 * n
    if direct_ms:
        out["direct"] = {"alg_bytes": db, "formula": "16(n+1) + 8m + 8m + 4n + 4m", "ms": direct_ms,
                         "bound": "hbm", "achieved": db / (direct_ms / 1e3) / 1e9, "peak": hbm,
                         "unit": "GB/s", "frac": db / (direct_ms / 1e3) / 1e9 / hbm}
    return out


def cpp_api_e2e(cfg_id, steps, pv=False):
    """The reference's own call sequence through the drop-in C++ API with host
    objects in and out (tests/cpp/api_bench.cpp over libkclique_b200.so):
    make_ranking -> direct_by_ranking -> count_*; cold = a fresh Graph per
    step (CSR uploaded inside the timed region), warm = the same Graph found
    resident on the device.  Separate process: it owns its own handles."""
    exe = os.path.join(ROOT, "tests", "cpp", "bin", "api_bench")
    if not os.path.exists(exe):
        return {"unavailable": "tests/cpp/bin/api_bench not built"}
    try:
        out = subprocess.run([exe, str(cfg_id), str(steps), "1" if pv else "0"],
                             capture_output=True, text=True, timeout=900, check=True).stdout
        return json.loads(out.strip().splitlines()[-1])
    except (subprocess.SubprocessError, ValueError, IndexError) as e:
        return {"unavailable": f"api_bench failed: {e}"[:200]}


def ncu_entry(cfg_id, k, pv=False):
    """The committed ncu counters of one counting call (profiles/ncu_summary.json,
    written by tools/ncu_counts.py on the B200)."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if not os.path.exists(path):
        return None
    try:
        return json.load(open(path)).get(f"config{cfg_id}_k{k}" + ("_pv" if pv else ""))
    except ValueError:
        return None


def attach_ncu(roofline, ncu):
    """ncu's own view of what binds the counting kernels, next to the algorithmic
    roof: DRAM and L2 bytes of one count, and the two busiest units, time-weighted
    over the count's launches -- the LSU data pipe (shared-memory and global
    wavefronts: the staging probes and the bitmap rows) and the issue slots."""
    if not ncu:
        roofline.setdefault("traffic", None)
        return
    roofline["traffic"] = ncu.get("dram_bytes_per_launch")
    roofline["l2_traffic"] = ncu.get("l2_bytes_per_launch")
    if "lsu_wavefront_pct_time_weighted" in ncu:
        roofline["limiter"] = {
            "lsu_wavefront_pct_of_peak": ncu["lsu_wavefront_pct_time_weighted"],
            "issue_active_pct_of_peak": ncu["issue_active_pct_time_weighted"],
            "l2_pct_of_peak": ncu.get("l2_pct_time_weighted"),
            "dram_pct_of_peak": ncu.get("dram_pct_time_weighted"),
            "threads_per_inst": ncu.get("threads_per_inst_time_weighted"),
            "ncu_kernel_ms": ncu["ncu_duration_ns_sum"] / 1e6,
            "source": "profiles/ncu_summary.json (tools/ncu_counts.py: ncu --metrics, "
                      "time-weighted over the count's launches)"}


# ---------------------------------------------------------------------------
# CPU reference (oracle/_ref = the unmodified reference library)
# ---------------------------------------------------------------------------
def reference_step(R, rg, g, spec, k):
    t0 = time.perf_counter()
    rank, rounds, _ = R.rank(rg, g.n, spec["strategy"], spec["eps"], 0)
    dg, _ = R.direct(rg, rank)
    total, _, _ = R.count(dg, g.n, k, parallelism=2)
    dt = time.perf_counter() - t0
    R.dg_destroy(dg)
    return total, dt


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    from tests import reforacle
    spec, k = workload(args.config, args.k)
    g = gen.load_config_graph(args.config, cache=False)
    try:
        R = reforacle.Ref()
        kind = "reference"
    except FileNotFoundError:
        print(json.dumps({"impl": "reference",
                          "unavailable": "oracle/_ref/libkclique_ref.so not built"}))
        return 0
    cores = os.cpu_count() or 1
    R.set_threads(cores)
    rg = R.graph(g)
    # first step doubles as warm-up and sizes the run to the budget
    total, t_first = reference_step(R, rg, g, spec, k)
    # the same number of warm-up steps as the B200 arm (>= 3); the first
    # step counts as one
    warm = max(args.warmup, 3) - 1
    for _ in range(warm):
        reference_step(R, rg, g, spec, k)
    steps = max(1, min(args.steps, int(args.cpu_budget_s // max(t_first, 1e-3))))
    times = []
    for _ in range(steps):
        t, dt = reference_step(R, rg, g, spec, k)
        assert t == total
        times.append(dt)
    sec = sum(times) / len(times)
    value = total / sec
    sample = (f"{steps} full step(s) of config {args.config} k={k} "
              f"(rank+direct+count, OpenMP {cores} threads)")
    print(json.dumps({
        "impl": "reference", "metric": f"k-cliques/s (k={k})", "value": value,
        "unit": "cliques/s", "n_gpus": world, "steps": steps, "warmup": 1 + warm,
        "requested_steps": args.steps, "ms_per_step": sec * 1e3, "higher_is_better": True,
        "scaling": "strong", "warmup_steps_run": 1 + warm, "vs_baseline": None, "dtype": "u32 ids / u64 counts",
        "data": "synthetic (in-repo deterministic generator)",
        "config": config_obj(args.config, spec, k, g),
        "cpu_baseline": {"value": value, "unit": "cliques/s", "cores": cores, "kind": kind,
                         "sample": sample},
        "e2e": {"value": value, "unit": "cliques/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "total": str(total)}))
    return 0


def cpu_baseline(g, spec, k):
    from tests import reforacle
    try:
        R = reforacle.Ref()
        kind = "reference"
    except FileNotFoundError:
        return None
    cores = os.cpu_count() or 1
    R.set_threads(cores)
    rg = R.graph(g)
    total, dt = reference_step(R, rg, g, spec, k)
    R.graph_destroy(rg)
    return {"value": total / dt, "unit": "cliques/s", "cores": cores, "kind": kind,
            "sample": f"one full step (rank+direct+count k={k}) on the same graph, "
                      f"{dt:.2f} s", "total": str(total)}


# ---------------------------------------------------------------------------
# B200 arm
# ---------------------------------------------------------------------------
def config_sweep(kcg, peaks, ops, l2_bytes):
    """One line per (config, k[, per-vertex]) with the reference goldens'
    verdict (tests/golden/config*.json) and the §8(d) roofline of the count.
    Config 5 is left to config5_block (its own e2e and roofline)."""
    out = []
    for cid in (1, 2, 3, 4):
        spec = gen.CONFIGS[cid]
        strat = gen.gpu_strategy(spec)
        gpath = os.path.join(ROOT, "tests", "golden", f"config{cid}.json")
        golden = json.load(open(gpath)) if os.path.exists(gpath) else {}
        t0 = time.perf_counter()
        h = kcg.DeviceGraph.from_graph(gen.load_config_graph(cid, cache=False))
        build_s = time.perf_counter() - t0
        for _ in range(2):  # second pass: buffers allocated, timings warm
            h.rank(strat, spec["eps"], download=False)
            rank_ms = h.timings()["rank_ms"]
            h.direct(download=False)
            direct_ms = h.timings()["direct_ms"]
        m = h.m
        sum_io = h.dag_work()
        phases = phase_rooflines(strat, h.n, m, rank_ms, direct_ms, peaks)
        t3 = None
        for k in spec["ks"]:
            for pv in ([False, True] if k in spec["pv_ks"] else [False]):
                if pv and t3 is None:
                    t3, _ = h.count(3)
                h.count(k, per_vertex=pv)  # warm
                total, _ = h.count(k, per_vertex=pv)
                tm = h.timings()
                cms = tm["count_ms"]
                step = rank_ms + direct_ms + cms
                gold = (golden.get("per_vertex" if pv else "counts", {}).get(str(k), {})
                        .get("total"))
                out.append({"config": cid, "k": k, "per_vertex": pv, "total": str(total),
                            "matches_reference": (str(total) == gold) if gold else None,
                            "strategy": STRAT_NAMES[strat], "n": h.n, "m": m,
                            "rank_ms": rank_ms, "direct_ms": direct_ms, "count_ms": cms,
                            "cliques_per_s": total / (cms / 1e3) if cms else None,
                            "oriented_edges_per_s": m / (step / 1e3),
                            "roofline": roofline_entry(cid, k, h.n, m, sum_io,
                                                       tm["count_kernel_ms"], peaks, ops,
                                                       l2_bytes, pv, t3),
                            "phase_rooflines": phases,
                            "build_s": build_s})
                attach_ncu(out[-1]["roofline"], ncu_entry(cid, k, pv))
        h.close()
    return out


def config5_block(kcg, peaks, ops, l2_bytes, steps=2):
    """Config 5 (R-MAT s24, EF32, degree order; k=4 totals and per-vertex
    counts) measured like the headline: device-timed phases with the graph
    resident in HBM, and e2e through the C ABI from a pinned HOST CSR
    (kcg_graph_create H2D + kcg_pipeline + per-vertex D2H inside the timed
    region), the §8(d) roofline (HBM: the 2 GB DAG exceeds L2) and the
    reference's time from the committed offline golden run."""
    import torch

    spec = gen.CONFIGS[5]
    p = spec["rmat"]
    gpath = os.path.join(ROOT, "tests", "golden", "config5.json")
    golden = json.load(open(gpath)) if os.path.exists(gpath) else {}
    t0 = time.perf_counter()
    hd = kcg.DeviceGraph.rmat(p["scale"], p["samples"], seed=p["seed"], permute=p["permute"])
    build_s = time.perf_counter() - t0
    off, adj = hd.csr()
    hd.close()
    off_p = torch.from_numpy(off.view(np.int64)).pin_memory()
    adj_p = torch.from_numpy(adj.view(np.int32)).pin_memory()
    del off, adj
    n = off_p.numel() - 1
    strat = gen.gpu_strategy(spec)
    blk = {"workload": "config5: " + spec["desc"], "k": 4, "n": n,
           "m": adj_p.numel() // 2, "strategy": STRAT_NAMES[strat],
           "device_build_s": build_s}
    # device-resident phases (graph uploaded once)
    h = kcg.DeviceGraph.from_csr_ptr(n, off_p.data_ptr(), adj_p.data_ptr())
    for _ in range(2):  # second pass: buffers allocated, timings warm
        h.rank(strat, spec["eps"], download=False)
        rank_ms = h.timings()["rank_ms"]
        h.direct(download=False)
        direct_ms = h.timings()["direct_ms"]
    m = h.m
    sum_io = h.dag_work()
    blk["phase_rooflines"] = phase_rooflines(strat, n, m, rank_ms, direct_ms, peaks)
    t3, _ = h.count(3)
    for pv in (False, True):
        key = "per_vertex" if pv else "totals"
        cms, kms = [], []
        total = None
        for _ in range(steps):
            total, _ = h.count(4, per_vertex=pv)
            tm = h.timings()
            cms.append(tm["count_ms"])
            kms.append(tm["count_kernel_ms"])
        cm, km = sum(cms) / len(cms), sum(kms) / len(kms)
        gold = golden.get("per_vertex" if pv else "counts", {}).get("4", {})
        blk[key] = {"total": str(total),
                    "matches_reference": (str(total) == gold.get("total")) if gold else None,
                    "rank_ms": rank_ms, "direct_ms": direct_ms, "count_ms": cm,
                    "step_ms": rank_ms + direct_ms + cm,
                    "cliques_per_s": total / (cm / 1e3),
                    "oriented_edges_per_s": m / ((rank_ms + direct_ms + cm) / 1e3),
                    "roofline": roofline_entry(5, 4, n, m, sum_io, km, peaks, ops, l2_bytes,
                                               pv, t3)}
        attach_ncu(blk[key]["roofline"], ncu_entry(5, 4, pv))
        if gold.get("t_count_s"):
            ref_s = gold["t_count_s"] + golden.get("t_rank_s", 0) + golden.get("t_direct_s", 0)
            blk[key]["cpu_baseline"] = {
                "value": int(gold["total"]) / gold["t_count_s"], "unit": "cliques/s",
                "cores": golden.get("threads"), "kind": "reference",
                "sample": "OFFLINE: the unmodified reference's make_ranking + "
                          "direct_by_ranking + count_%s on this config in the build "
                          "container (tests/golden/config5.json, %.0f s count, %.0f s "
                          "step); too long to rerun in the bench" % (key, gold["t_count_s"],
                                                                    ref_s)}
    h.close()
    # e2e through the C ABI with host buffers, every step: H2D of the CSR,
    # rank + orient + count on the device, D2H of the result
    for pv in (False, True):
        key = "per_vertex" if pv else "totals"
        times = []
        total = None
        for i in range(steps + 1):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            he = kcg.DeviceGraph.from_csr_ptr(n, off_p.data_ptr(), adj_p.data_ptr())
            total, _ = he.pipeline(strat, spec["eps"], 4, per_vertex=pv)
            he.close()
            dt = time.perf_counter() - t0
            if i:
                times.append(dt)
        esec = sum(times) / len(times)
        blk[key]["e2e"] = {"value": total / esec, "unit": "cliques/s", "ms_per_step": esec * 1e3,
                           "h2d_bytes_per_step": int(off_p.numel() * 8 + adj_p.numel() * 4),
                           "d2h_bytes_per_step": 8 + (8 * n if pv else 0),
                           "path": "kcg_graph_create(pinned host CSR) + kcg_pipeline%s + "
                                   "destroy" % (" (per-vertex, D2H)" if pv else "")}
    return blk


def run_kcg(args):
    import torch
    import torch.distributed as dist

    from paper_2002_10047_b200 import kcg

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    spec, k = workload(args.config, args.k)
    strat, eps = gen.gpu_strategy(spec), spec["eps"]
    g = gen.load_config_graph(args.config, cache=False)
    h = kcg.DeviceGraph.from_graph(g)
    stream = torch.cuda.ExternalStream(h.stream_ptr())
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    red = torch.zeros(1, dtype=torch.int64, device="cuda")

    def step():
        if world == 1:
            return h.pipeline(strat, eps, k)[0]
        # one GPU's share: replicated rank + DAG, its work-balanced source
        # range, then the all-reduce of the u64 total (on the library
        # stream, so the step's events cover it)
        h.rank(strat, eps, download=False)
        h.direct(download=False)
        b = h.partition_plan(k, world)
        t, _ = h.count_range(k, int(b[rank]), int(b[rank + 1]))
        with torch.cuda.stream(stream):
            red.fill_(int(np.uint64(t).view(np.int64)))
            dist.all_reduce(red)
        return None

    for _ in range(max(args.warmup, 3)):
        step()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    launches0 = h.timings()["launches"]
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    phase = {"rank_ms": 0.0, "direct_ms": 0.0, "count_ms": 0.0, "count_kernel_ms": 0.0}
    total = None
    for i in range(args.steps):
        with torch.cuda.stream(stream):
            flush.zero_()
        ev[i][0].record(stream)
        total = step()
        ev[i][1].record(stream)
        t = h.timings()
        for key in phase:
            phase[key] += t[key]
    torch.cuda.synchronize()
    launches = h.timings()["launches"] - launches0
    clk = clocks.stop()
    ms = sum(a.elapsed_time(b) for a, b in ev)
    if world > 1:
        total = int(np.int64(red.item()).view(np.uint64))
        tt = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
        dist.barrier()
    ms_per_step = ms / args.steps
    value = total / (ms_per_step / 1e3)
    for key in phase:
        phase[key] /= args.steps
    stats = h.count_stats()

    # roofline of the dominant (counting) kernels, SURVEY.md §8(d)
    peaks = counting_peaks()
    ops = ops_table()
    l2_bytes = kcg.device_info().get("l2_bytes", 0)
    sum_io = h.dag_work()
    roofline = roofline_entry(args.config, k, g.n, g.m, sum_io, phase["count_kernel_ms"],
                              peaks, ops, l2_bytes)
    ncu = ncu_entry(args.config, k)
    attach_ncu(roofline, ncu)
    roofline.update({
        "kernel_ms": phase["count_kernel_ms"], "peaks": peaks,
        "note": "achieved = B_alg (16n+20m+4*sum indeg*outdeg) / device time of the counting "
                "kernels (CUDA events on the library stream); BW = measured L2 read bandwidth "
                "because the DAG fits the 126 MB L2 (SURVEY.md §8(d)); hbm_frac = the same "
                "bytes against measured HBM; traffic = ncu dram bytes of one count"})
    if ncu and "smem_wavefront_floor_ms" in ncu:
        roofline["smem"] = {k2: ncu[k2] for k2 in ("smem_wavefronts", "smem_wavefront_floor_ms",
                                                    "sm_throughput_pct_time_weighted")
                            if k2 in ncu}

    # secondary: the config's other k values on the same DAG (counting only)
    secondary = {}
    if world == 1:
        for k2 in spec["ks"]:
            if k2 == k:
                continue
            h.rank(strat, eps, download=False)
            h.direct(download=False)
            reps = 3
            tot2 = 0
            cms = kms = 0.0
            for _ in range(reps):
                tot2, _ = h.count(k2)
                cms += h.timings()["count_ms"]
                kms += h.timings()["count_kernel_ms"]
            cms /= reps
            kms /= reps
            secondary[f"k{k2}"] = {"total": str(tot2), "count_ms": cms,
                                   "cliques_per_s": tot2 / (cms / 1e3),
                                   "oriented_edges_per_s": g.m / (cms / 1e3),
                                   "roofline": roofline_entry(args.config, k2, g.n, g.m, sum_io,
                                                              kms, peaks, ops, l2_bytes)}

    # downstream consumer of the per-vertex counts:
    # approximate k-clique densest-subgraph peeling on the same handle
    if world == 1:
        h.rank(strat, eps, download=False)
        h.direct(download=False)
        h.peel_approx(k, 0.5)  # warm
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        po = h.peel_approx(k, 0.5)
        pms = (time.perf_counter() - t0) * 1e3
        ent = {"ms": pms, "eps": 0.5, "rounds": po["rounds"], "best_round": po["best_round"],
               "best_density": po["best_density"], "dense_vertices": len(po["dense_vertices"]),
               "note": "per-vertex count + restricted recount per round, host-timed"}
        pg = os.path.join(ROOT, "tests", "golden", "peel_configs.json")
        if os.path.exists(pg):
            ref = json.load(open(pg)).get(f"config{args.config}_k{k}_approx")
            if ref:
                ent["matches_reference"] = (
                    ref["rounds"] == po["rounds"] and ref["best_round"] == po["best_round"]
                    and ref["best_density"] == float(po["best_density"]).hex())
                ent["reference_s"] = ref["ref_seconds"]
                ent["reference_threads"] = ref["threads"]
        secondary[f"peel_approx_k{k}"] = ent

    # every other BASELINE config at every k (SURVEY.md §8(d) units) with its
    # roofline; config 5 gets its own fully instrumented block
    sweep = c5 = None
    if world == 1 and not args.no_sweep:
        sweep = config_sweep(kcg, peaks, ops, l2_bytes)
    if world == 1 and not args.no_config5:
        c5 = config5_block(kcg, peaks, ops, l2_bytes)

    # the same sequence through the reference's C++ headers (drop-in library)
    api = None
    if world == 1 and not args.no_sweep:
        api = {"config2": cpp_api_e2e(2, 5)}
        if not args.no_config5:
            api["config5"] = cpp_api_e2e(5, 2)
            api["config5_per_vertex"] = cpp_api_e2e(5, 1, True)

    # e2e: the reference-facing C ABI with host buffers (pinned), H2D + D2H
    # inside the timed region
    e2e = None
    if world == 1:
        off_p = torch.from_numpy(g.offsets.view(np.int64)).pin_memory()
        adj_p = torch.from_numpy(g.adj.view(np.int32)).pin_memory()
        e_steps = max(1, min(args.steps, 5))
        e_times = []
        split = np.zeros(3)
        for i in range(max(args.warmup, 3) + e_steps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            he = kcg.DeviceGraph.from_csr_ptr(g.n, off_p.data_ptr(), adj_p.data_ptr())
            t1 = time.perf_counter()
            te, _ = he.pipeline(strat, eps, k)
            t2 = time.perf_counter()
            he.close()
            t3 = time.perf_counter()
            if i >= max(args.warmup, 3):
                e_times.append(t3 - t0)
                split += (t1 - t0, t2 - t1, t3 - t2)
            assert te == total
        esec = sum(e_times) / len(e_times)
        split *= 1e3 / len(e_times)
        e2e = {"value": total / esec, "unit": "cliques/s",
               "h2d_bytes_per_step": int(off_p.numel() * 8 + adj_p.numel() * 4),
               "d2h_bytes_per_step": 8, "ms_per_step": esec * 1e3,
               "split_ms": {"create_h2d": split[0], "pipeline": split[1], "destroy": split[2]},
               "path": "kcg_graph_create(pinned host CSR) + kcg_pipeline + destroy"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(g, spec, k)
        if cpu and cpu.pop("total") != str(total):
            raise AssertionError("GPU total differs from the reference")

    if rank == 0:
        line = {
            "metric": f"k-cliques/s (k={k})", "value": value, "unit": "cliques/s",
            "n_gpus": world, "steps": args.steps, "warmup": max(args.warmup, 3),
            "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None, "dtype": "u32 ids / u64 counts",
            "data": "synthetic (in-repo deterministic generator, seeded)",
            "config": config_obj(args.config, spec, k, g,
                                 {"parallelism": "work-balanced contiguous source ranges "
                                                 "(kcg_partition_plan) + NCCL all-reduce, "
                                                 f"{world} GPUs" if world > 1
                                  else "single GPU",
                                  "reference_arm": "the driver's --impl reference arm runs "
                                                   "this same config (config 2) on the host "
                                                   "cores; config 5's reference time is the "
                                                   "committed offline run (config5 block)"}),
            "total": str(total),
            "oriented_edges_per_s": g.m / (ms_per_step / 1e3),
            "phases_ms": phase,
            "phase_rooflines": phase_rooflines(gen.gpu_strategy(spec), g.n, g.m,
                                               phase.get("rank_ms"), phase.get("direct_ms"),
                                               peaks),
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "e2e_cpp_api": api,
            "gpu_launches": launches,
            "clocks": clk,
            "count_stats": stats,
            "config5": c5,
            "secondary": secondary,
            "configs": sweep,
        }
        print(json.dumps(line))
    h.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    args = parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_kcg(args)


if __name__ == "__main__":
    sys.exit(main())
