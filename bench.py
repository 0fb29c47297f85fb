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


def alg_bytes(n, out_off, out_adj):
    """B_alg = 16n + 20m + 4 * sum_w indeg(w) * outdeg(w)."""
    outdeg = np.diff(out_off).astype(np.float64)
    indeg = np.bincount(out_adj, minlength=n).astype(np.float64)
    m = len(out_adj)
    return 16.0 * n + 20.0 * m + 4.0 * float(np.dot(indeg, outdeg))


def ncu_entry(cfg_id, k):
    """The committed ncu capture of one counting call (profiles/)."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if not os.path.exists(path):
        return None
    try:
        return json.load(open(path)).get(f"config{cfg_id}_k{k}")
    except ValueError:
        return None


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
    warm = max(0, min(args.warmup, 1) - 1)
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
        "scaling": "strong", "vs_baseline": None, "dtype": "u32 ids / u64 counts",
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
def config_sweep(kcg, skip_cfg):
    """One line per (config, k[, per-vertex]) with the reference goldens'
    verdict (tests/golden/config*.json)."""
    out = []
    for cid in (1, 2, 3, 4, 5):
        spec = gen.CONFIGS[cid]
        strat = gen.gpu_strategy(spec)
        gpath = os.path.join(ROOT, "tests", "golden", f"config{cid}.json")
        golden = json.load(open(gpath)) if os.path.exists(gpath) else {}
        t0 = time.perf_counter()
        if cid == 5:
            p = spec["rmat"]
            h = kcg.DeviceGraph.rmat(p["scale"], p["samples"], seed=p["seed"],
                                     permute=p["permute"])
        else:
            h = kcg.DeviceGraph.from_graph(gen.load_config_graph(cid, cache=False))
        build_s = time.perf_counter() - t0
        h.rank(strat, spec["eps"], download=False)
        rank_ms = h.timings()["rank_ms"]
        h.direct(download=False)
        direct_ms = h.timings()["direct_ms"]
        m = h.m
        for k in spec["ks"]:
            for pv in ([False, True] if k in spec["pv_ks"] else [False]):
                if cid != 5:
                    h.count(k, per_vertex=pv)  # warm
                total, _ = h.count(k, per_vertex=pv)
                cms = h.timings()["count_ms"]
                step = rank_ms + direct_ms + cms
                gold = golden.get("counts", {}).get(str(k), {}).get("total")
                out.append({"config": cid, "k": k, "per_vertex": pv, "total": str(total),
                            "matches_reference": (str(total) == gold) if gold else None,
                            "strategy": STRAT_NAMES[strat], "n": h.n, "m": m,
                            "rank_ms": rank_ms, "direct_ms": direct_ms, "count_ms": cms,
                            "cliques_per_s": total / (cms / 1e3) if cms else None,
                            "oriented_edges_per_s": m / (step / 1e3),
                            "build_s": build_s})
        h.close()
    return out


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

    def step():
        if world == 1:
            return h.pipeline(strat, eps, k)[0]
        h.rank(strat, eps, download=False)
        h.direct(download=False)
        return h.count_part(k, rank, world)[0]

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
    part_total = 0
    for i in range(args.steps):
        with torch.cuda.stream(stream):
            flush.zero_()
        ev[i][0].record(stream)
        part_total = step()
        ev[i][1].record(stream)
        t = h.timings()
        for key in phase:
            phase[key] += t[key]
    torch.cuda.synchronize()
    launches = h.timings()["launches"] - launches0
    clk = clocks.stop()
    ms = sum(a.elapsed_time(b) for a, b in ev)
    total = part_total
    if world > 1:
        tt = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
        from paper_2002_10047_b200 import shard
        total, _ = shard.allreduce_counts(part_total, None, device="cuda")
        dist.barrier()
    ms_per_step = ms / args.steps
    value = total / (ms_per_step / 1e3)
    for key in phase:
        phase[key] /= args.steps
    stats = h.count_stats()

    # roofline of the dominant (counting) kernels
    off, adj, max_out = h.direct()
    b_alg = alg_bytes(g.n, off, adj)
    peak, peak_src = measured_peaks()
    achieved = b_alg / (phase["count_kernel_ms"] / 1e3) / 1e9
    dag_bytes = 8 * (g.n + 1) + 4 * g.m
    ncu = ncu_entry(args.config, k)
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak,
                "traffic": ncu.get("dram_bytes_per_launch") if ncu else None,
                "alg_bytes_per_launch": b_alg, "kernel_ms": phase["count_kernel_ms"],
                "peak_source": peak_src,
                "note": "achieved = B_alg (SURVEY.md §8(d): 16n+20m+4*sum indeg*outdeg) / "
                        "device time of the counting kernels; the DAG (%.0f MB) %s L2"
                        % (dag_bytes / 1e6, "fits in" if dag_bytes < 126e6 else "exceeds")}
    if ncu and "sm_throughput_pct_time_weighted" in ncu:
        # the limiting roof of the L2-resident counting kernels is integer
        # issue: ncu's SM throughput = achieved fraction of
        # peak issue, time-weighted over the launches of one count
        roofline["issue"] = {
            "frac": ncu["sm_throughput_pct_time_weighted"] / 100.0,
            "ipc": ncu["ipc_time_weighted"], "peak_ipc": ncu["issue_slot_peak_ipc"],
            "threads_per_inst": ncu["threads_per_inst_time_weighted"],
            "source": "profiles/ncu_summary.json: " + ncu["source"]}

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
            cms = 0.0
            for _ in range(reps):
                tot2, _ = h.count(k2)
                cms += h.timings()["count_ms"]
            cms /= reps
            secondary[f"k{k2}"] = {"total": str(tot2), "count_ms": cms,
                                   "cliques_per_s": tot2 / (cms / 1e3),
                                   "oriented_edges_per_s": g.m / (cms / 1e3)}

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

    # every BASELINE config at every k (SURVEY.md §8(d) units): device-timed
    # phases, cliques/s of the count and oriented edges/s of the step; the
    # graphs are the canonical generators' (config 5 built on the device)
    sweep = None
    if world == 1 and not args.no_sweep:
        sweep = config_sweep(kcg, args.config)

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
                                 {"parallelism": f"sources r % {world}" if world > 1
                                  else "single GPU"}),
            "total": str(total),
            "oriented_edges_per_s": g.m / (ms_per_step / 1e3),
            "phases_ms": phase,
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk,
            "count_stats": stats,
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
