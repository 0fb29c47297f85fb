"""ctypes bindings for the kcg C ABI (include/kcg.h, lib/libkcg.so).

The product path: every call goes to the sm_100a kernels.  There is no CPU
fallback — if the library or a B200 is missing, calls raise KcgError.

Besides the handle class, the module mirrors the reference's entry points
(proj/include/kclique/{orientation,graph,counting}.hpp) so tests read like
the reference's own: ``rank_by_degree(g)``, ``make_ranking(g, cfg)``,
``direct_by_ranking(g, rank)``, ``count_total(dg, k)``,
``count_per_vertex(dg, k)``.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from typing import Optional

import numpy as np

from ._paths import LIB_DIR

KCG_OK, KCG_EINVAL, KCG_ERUNTIME, KCG_ENOMEM, KCG_ELOGIC = 0, 1, 2, 3, 4
DEGREE, ORIGINAL, KCORE, GOODRICH_PSZONA, BARENBOIM_ELKIN = 0, 1, 2, 3, 4
KCORE_PARALLEL = 5  # bulk-synchronous degeneracy order (not in the reference)
STRATEGY_NAMES = {"degree": DEGREE, "original": ORIGINAL, "kcore": KCORE,
                  "goodrich_pszona": GOODRICH_PSZONA, "barenboim_elkin": BARENBOIM_ELKIN,
                  "kcore_parallel": KCORE_PARALLEL}

EXPORTED = [
    "kcg_last_error", "kcg_version", "kcg_device_info", "kcg_graph_create",
    "kcg_graph_create_device", "kcg_dag_create", "kcg_graph_destroy", "kcg_num_vertices",
    "kcg_num_edges", "kcg_rank", "kcg_estimate_arboricity", "kcg_set_ranking", "kcg_direct",
    "kcg_count", "kcg_per_vertex_device", "kcg_pipeline", "kcg_timings",
    "kcg_last_count_stats", "kcg_device_bytes", "kcg_synchronize", "kcg_count_part",
    "kcg_count_range", "kcg_partition_plan", "kcg_dag_work",
    "kcg_stream", "kcg_update_counts", "kcg_peel_exact", "kcg_peel_approx",
    "kcg_graph_from_edges", "kcg_graph_rmat", "kcg_graph_csr", "kcg_colorful_sparsify",
    "kcg_approx_count", "kcg_list_cliques",
]


class KcgError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"[kcg status {status}] {msg}")
        self.status = status


class KcgOutOfMemory(KcgError, MemoryError):
    pass


class KcgLogicError(KcgError):
    """The reference's std::logic_error cases (peeling)."""


CLIQUE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.POINTER(ctypes.c_uint32), ctypes.c_uint64,
                             ctypes.c_int, ctypes.c_void_p)


class SampleEstimate(ctypes.Structure):
    _fields_ = [("k", ctypes.c_int), ("colors", ctypes.c_uint64), ("p", ctypes.c_double),
                ("sub_count", ctypes.c_uint64), ("estimate", ctypes.c_double),
                ("seed", ctypes.c_uint64)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class PeelResult(ctypes.Structure):
    _fields_ = [("rounds", ctypes.c_uint64), ("total_cliques", ctypes.c_uint64),
                ("best_density", ctypes.c_double), ("best_round", ctypes.c_uint64),
                ("num_dense", ctypes.c_uint64)]


class Times(ctypes.Structure):
    _fields_ = [("upload_ms", ctypes.c_double), ("rank_ms", ctypes.c_double),
                ("direct_ms", ctypes.c_double), ("count_ms", ctypes.c_double),
                ("count_kernel_ms", ctypes.c_double), ("download_ms", ctypes.c_double),
                ("h2d_bytes", ctypes.c_uint64), ("d2h_bytes", ctypes.c_uint64),
                ("launches", ctypes.c_uint64)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class CountStats(ctypes.Structure):
    _fields_ = [("sources_warp", ctypes.c_uint64), ("sources_cta", ctypes.c_uint64),
                ("sources_heavy", ctypes.c_uint64), ("max_out_degree", ctypes.c_uint64),
                ("staged_elems", ctypes.c_uint64), ("launches", ctypes.c_uint64)]

    def as_dict(self):
        return {f: int(getattr(self, f)) for f, _ in self._fields_}


_lib = None


def lib_path() -> str:
    # KCG_LIB: a variant build of the same library (tools/ab_build.sh A/B runs)
    return os.environ.get("KCG_LIB") or os.path.join(LIB_DIR, "libkcg.so")


def lib():
    """Loads libkcg.so; raises if it is absent (no fallback)."""
    global _lib
    if _lib is None:
        path = lib_path()
        if not os.path.exists(path):
            raise KcgError(KCG_ERUNTIME, f"{path} missing: run __graft_entry__.build()")
        L = ctypes.CDLL(path)
        vp, u32, u64 = ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64
        P = ctypes.POINTER
        L.kcg_last_error.restype = ctypes.c_char_p
        L.kcg_version.restype = ctypes.c_char_p
        L.kcg_device_info.argtypes = [P(ctypes.c_int)] * 5
        L.kcg_graph_create.argtypes = [u32, vp, vp, P(vp)]
        L.kcg_graph_create_device.argtypes = [u32, u64, vp, vp, P(vp)]
        L.kcg_dag_create.argtypes = [u32, vp, vp, vp, P(vp)]
        L.kcg_graph_destroy.argtypes = [vp]
        L.kcg_graph_destroy.restype = None
        L.kcg_num_vertices.argtypes = [vp]
        L.kcg_num_vertices.restype = u32
        L.kcg_num_edges.argtypes = [vp]
        L.kcg_num_edges.restype = u64
        L.kcg_rank.argtypes = [vp, ctypes.c_int, ctypes.c_double, u64, vp, P(u64), P(u64)]
        L.kcg_estimate_arboricity.argtypes = [vp, ctypes.c_double, P(u64)]
        L.kcg_set_ranking.argtypes = [vp, vp, u32]
        L.kcg_direct.argtypes = [vp, vp, vp, P(u64)]
        L.kcg_count.argtypes = [vp, ctypes.c_int, P(u64), vp]
        L.kcg_per_vertex_device.argtypes = [vp, P(vp)]
        L.kcg_count_part.argtypes = [vp, ctypes.c_int, u32, u32, P(u64), vp]
        L.kcg_count_range.argtypes = [vp, ctypes.c_int, u32, u32, P(u64), vp]
        L.kcg_partition_plan.argtypes = [vp, ctypes.c_int, u32, vp]
        L.kcg_dag_work.argtypes = [vp, P(u64)]
        L.kcg_stream.argtypes = [vp]
        L.kcg_stream.restype = vp
        L.kcg_pipeline.argtypes = [vp, ctypes.c_int, ctypes.c_double, u64, ctypes.c_int,
                                   P(u64), vp]
        L.kcg_timings.argtypes = [vp, P(Times)]
        L.kcg_last_count_stats.argtypes = [vp, P(CountStats)]
        L.kcg_device_bytes.argtypes = [vp]
        L.kcg_device_bytes.restype = u64
        L.kcg_synchronize.argtypes = [vp]
        L.kcg_graph_from_edges.argtypes = [u32, vp, vp, u64, P(vp)]
        L.kcg_graph_rmat.argtypes = [ctypes.c_int, u64, ctypes.c_double, ctypes.c_double,
                                     ctypes.c_double, u64, ctypes.c_int, P(vp)]
        L.kcg_graph_csr.argtypes = [vp, vp, vp]
        L.kcg_list_cliques.argtypes = [vp, ctypes.c_int, u64, CLIQUE_FN, vp, P(u64)]
        L.kcg_colorful_sparsify.argtypes = [vp, u64, u64, P(vp)]
        L.kcg_approx_count.argtypes = [vp, ctypes.c_int, u64, u64, ctypes.c_int, ctypes.c_double,
                                       u64, P(SampleEstimate)]
        L.kcg_update_counts.argtypes = [vp, ctypes.c_int, vp, vp, u64, vp, P(u64), vp, P(u64)]
        L.kcg_peel_exact.argtypes = [vp, ctypes.c_int, P(PeelResult), vp, vp]
        L.kcg_peel_approx.argtypes = [vp, ctypes.c_int, ctypes.c_double, P(PeelResult), vp]
        _lib = L
    return _lib


def _check(rc: int):
    if rc == KCG_OK:
        return
    msg = lib().kcg_last_error().decode(errors="replace")
    if rc == KCG_EINVAL:
        raise ValueError(msg)  # std::invalid_argument in the reference
    if rc == KCG_ENOMEM:
        raise KcgOutOfMemory(rc, msg)
    if rc == KCG_ELOGIC:
        raise KcgLogicError(rc, msg)
    raise KcgError(rc, msg)


def device_info() -> dict:
    vals = [ctypes.c_int(0) for _ in range(5)]
    _check(lib().kcg_device_info(*[ctypes.byref(v) for v in vals]))
    return dict(zip(["sm_count", "smem_optin", "l2_bytes", "cc_major", "cc_minor"],
                    [v.value for v in vals]))


def _u32(a):
    return np.ascontiguousarray(a, dtype=np.uint32)


def _u64(a):
    return np.ascontiguousarray(a, dtype=np.uint64)


class DeviceGraph:
    """A kcg_graph handle: the whole graph resident in HBM."""

    def __init__(self, handle: ctypes.c_void_p):
        self._h = handle

    @classmethod
    def from_csr(cls, offsets, adj) -> "DeviceGraph":
        off, a = _u64(offsets), _u32(adj)
        h = ctypes.c_void_p()
        _check(lib().kcg_graph_create(len(off) - 1, off.ctypes.data, a.ctypes.data,
                                      ctypes.byref(h)))
        return cls(h)

    @classmethod
    def from_csr_ptr(cls, n: int, offsets_ptr: int, adj_ptr: int) -> "DeviceGraph":
        """Host pointers (e.g. pinned buffers) to offsets[n+1] u64, adj[2m] u32."""
        h = ctypes.c_void_p()
        _check(lib().kcg_graph_create(n, ctypes.c_void_p(offsets_ptr), ctypes.c_void_p(adj_ptr),
                                      ctypes.byref(h)))
        return cls(h)

    @classmethod
    def from_edges(cls, n: int, edges) -> "DeviceGraph":
        """Graph::from_edges normalisation on the device (kcg_build.cu)."""
        e = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
        if len(e) and (e.min() < 0 or e.max() >= 1 << 32):
            raise ValueError("edge endpoint out of range")
        us, vs = _u32(e[:, 0]), _u32(e[:, 1])
        h = ctypes.c_void_p()
        _check(lib().kcg_graph_from_edges(int(n), us.ctypes.data, vs.ctypes.data, len(e),
                                          ctypes.byref(h)))
        return cls(h)

    @classmethod
    def rmat(cls, scale, samples, a=0.57, b=0.19, c=0.19, seed=0, permute=False):
        """The R-MAT generator on the device (same graph as gen.rmat)."""
        h = ctypes.c_void_p()
        _check(lib().kcg_graph_rmat(int(scale), int(samples), float(a), float(b), float(c),
                                    int(seed), int(bool(permute)), ctypes.byref(h)))
        return cls(h)

    def csr(self):
        """(offsets u64[n+1], adjacency u32[2m]) of the undirected graph."""
        off = np.zeros(self.n + 1, np.uint64)
        adj = np.zeros(max(2 * self.m, 1), np.uint32)
        _check(lib().kcg_graph_csr(self._h, off.ctypes.data, adj.ctypes.data))
        return off, adj[:2 * self.m]

    @classmethod
    def from_graph(cls, g) -> "DeviceGraph":
        return cls.from_csr(g.offsets, g.adj)

    @classmethod
    def from_dag(cls, out_offsets, out_targets, rank) -> "DeviceGraph":
        off, t, r = _u64(out_offsets), _u32(out_targets), _u32(rank)
        h = ctypes.c_void_p()
        _check(lib().kcg_dag_create(len(off) - 1, off.ctypes.data, t.ctypes.data,
                                    r.ctypes.data, ctypes.byref(h)))
        return cls(h)

    def close(self):
        if self._h:
            lib().kcg_graph_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    @property
    def n(self) -> int:
        return int(lib().kcg_num_vertices(self._h))

    @property
    def m(self) -> int:
        return int(lib().kcg_num_edges(self._h))

    def rank(self, strategy=DEGREE, eps=1.0, alpha_hat=0, download=True):
        """Returns (rank[n] or None, rounds, alpha_hat used)."""
        if isinstance(strategy, str):
            strategy = STRATEGY_NAMES[strategy]
        out = np.zeros(self.n, np.uint32) if download else None
        rounds, alpha = ctypes.c_uint64(0), ctypes.c_uint64(0)
        _check(lib().kcg_rank(self._h, strategy, float(eps), int(alpha_hat),
                              out.ctypes.data if download else None, ctypes.byref(rounds),
                              ctypes.byref(alpha)))
        return out, int(rounds.value), int(alpha.value)

    def estimate_arboricity(self, eps: float) -> int:
        out = ctypes.c_uint64(0)
        _check(lib().kcg_estimate_arboricity(self._h, float(eps), ctypes.byref(out)))
        return int(out.value)

    def set_ranking(self, rank):
        r = _u32(rank)
        _check(lib().kcg_set_ranking(self._h, r.ctypes.data, len(r)))

    def direct(self, download=True):
        """Returns (out_offsets, out_targets, max_out_degree)."""
        off = np.zeros(self.n + 1, np.uint64) if download else None
        tgt = np.zeros(self.m, np.uint32) if download else None
        mx = ctypes.c_uint64(0)
        _check(lib().kcg_direct(self._h, off.ctypes.data if download else None,
                                tgt.ctypes.data if download else None, ctypes.byref(mx)))
        return off, tgt, int(mx.value)

    def count(self, k: int, per_vertex=False):
        total = ctypes.c_uint64(0)
        pv = np.zeros(max(self.n, 1), np.uint64) if per_vertex else None
        _check(lib().kcg_count(self._h, int(k), ctypes.byref(total),
                               pv.ctypes.data if per_vertex else None))
        return int(total.value), (pv[:self.n] if per_vertex else None)

    def count_part(self, k: int, part: int, nparts: int, per_vertex=False):
        """Cliques whose lowest-ranked vertex lies in part `part` of
        partition_plan(k, nparts)."""
        total = ctypes.c_uint64(0)
        pv = np.zeros(max(self.n, 1), np.uint64) if per_vertex else None
        _check(lib().kcg_count_part(self._h, int(k), int(part), int(nparts), ctypes.byref(total),
                                    pv.ctypes.data if per_vertex else None))
        return int(total.value), (pv[:self.n] if per_vertex else None)

    def count_range(self, k: int, r_lo: int, r_hi: int, per_vertex=False):
        """Cliques whose lowest-ranked vertex r has r_lo <= r < r_hi."""
        total = ctypes.c_uint64(0)
        pv = np.zeros(max(self.n, 1), np.uint64) if per_vertex else None
        _check(lib().kcg_count_range(self._h, int(k), int(r_lo), int(r_hi), ctypes.byref(total),
                                     pv.ctypes.data if per_vertex else None))
        return int(total.value), (pv[:self.n] if per_vertex else None)

    def dag_work(self) -> int:
        """sum_w indeg(w) * outdeg(w) of the current DAG (device)."""
        v = ctypes.c_uint64(0)
        _check(lib().kcg_dag_work(self._h, ctypes.byref(v)))
        return int(v.value)

    def partition_plan(self, k: int, nparts: int) -> np.ndarray:
        """Work-balanced contiguous source ranges: nparts + 1 rank bounds."""
        b = np.zeros(int(nparts) + 1, np.uint32)
        _check(lib().kcg_partition_plan(self._h, int(k), int(nparts), b.ctypes.data))
        return b

    def stream_ptr(self) -> int:
        return int(lib().kcg_stream(self._h) or 0)

    def pipeline(self, strategy, eps, k, alpha_hat=0, per_vertex=False):
        if isinstance(strategy, str):
            strategy = STRATEGY_NAMES[strategy]
        total = ctypes.c_uint64(0)
        pv = np.zeros(max(self.n, 1), np.uint64) if per_vertex else None
        _check(lib().kcg_pipeline(self._h, strategy, float(eps), int(alpha_hat), int(k),
                                  ctypes.byref(total), pv.ctypes.data if per_vertex else None))
        return int(total.value), (pv[:self.n] if per_vertex else None)

    def per_vertex_device_ptr(self) -> int:
        p = ctypes.c_void_p()
        _check(lib().kcg_per_vertex_device(self._h, ctypes.byref(p)))
        return int(p.value or 0)

    def timings(self) -> dict:
        t = Times()
        _check(lib().kcg_timings(self._h, ctypes.byref(t)))
        return t.as_dict()

    def count_stats(self) -> dict:
        s = CountStats()
        _check(lib().kcg_last_count_stats(self._h, ctypes.byref(s)))
        return s.as_dict()

    def device_bytes(self) -> int:
        return int(lib().kcg_device_bytes(self._h))

    def synchronize(self):
        _check(lib().kcg_synchronize(self._h))

    def list_cliques(self, k, batch=0):
        """list_cliques: (total, array[total, k] of vertex ids, each row in
        ascending rank)."""
        parts = []

        def cb(ptr, count, kk, _user):
            parts.append(np.ctypeslib.as_array(ptr, shape=(int(count) * kk,)).copy()
                         .reshape(-1, kk))
            return 0

        fn = CLIQUE_FN(cb)
        total = ctypes.c_uint64(0)
        _check(lib().kcg_list_cliques(self._h, int(k), int(batch), fn, None,
                                      ctypes.byref(total)))
        arr = np.concatenate(parts) if parts else np.zeros((0, k), np.uint32)
        return int(total.value), arr

    # ---- colour sparsification (kcg_sample.cu; sampling.hpp:21-36) ----
    def colorful_sparsify(self, colors, seed) -> "DeviceGraph":
        h = ctypes.c_void_p()
        _check(lib().kcg_colorful_sparsify(self._h, int(colors), int(seed), ctypes.byref(h)))
        return DeviceGraph(h)

    def approx_count(self, k, colors, seed, strategy=0, eps=1.0, alpha_hat=0) -> dict:
        est = SampleEstimate()
        _check(lib().kcg_approx_count(self._h, int(k), int(colors), int(seed), int(strategy),
                                      float(eps), int(alpha_hat), ctypes.byref(est)))
        return est.as_dict()

    # ---- peeling (kcg_peel.cu; peeling.hpp:58-92) ----
    def update_counts(self, k, counts, batch, peeled):
        """update_counts: returns (removed, changed ids); `counts` (u64
        numpy array, n entries) is updated in place."""
        n = self.n
        if counts.dtype != np.uint64 or not counts.flags.c_contiguous or len(counts) < n:
            raise TypeError("counts must be a contiguous uint64 array of n entries")
        b = _u32(batch)
        pe = np.ascontiguousarray(peeled, dtype=np.uint8)
        removed = ctypes.c_uint64(0)
        nch = ctypes.c_uint64(0)
        changed = np.zeros(max(n, 1), np.uint32)
        _check(lib().kcg_update_counts(self._h, int(k), counts.ctypes.data, b.ctypes.data,
                                       len(b), pe.ctypes.data, ctypes.byref(removed),
                                       changed.ctypes.data, ctypes.byref(nch)))
        return int(removed.value), changed[:nch.value].copy()

    def peel_exact(self, k):
        """peel_exact: dict(rounds, total_cliques, best_density, best_round,
        core, dense_vertices)."""
        n = self.n
        r = PeelResult()
        core = np.zeros(max(n, 1), np.uint64)
        dense = np.zeros(max(n, 1), np.uint32)
        _check(lib().kcg_peel_exact(self._h, int(k), ctypes.byref(r), core.ctypes.data,
                                    dense.ctypes.data))
        return {"rounds": r.rounds, "total_cliques": r.total_cliques,
                "best_density": r.best_density, "best_round": r.best_round,
                "core": core[:n].copy(), "dense_vertices": dense[:r.num_dense].copy()}

    def peel_approx(self, k, eps):
        n = self.n
        r = PeelResult()
        dense = np.zeros(max(n, 1), np.uint32)
        _check(lib().kcg_peel_approx(self._h, int(k), float(eps), ctypes.byref(r),
                                     dense.ctypes.data))
        return {"rounds": r.rounds, "total_cliques": r.total_cliques,
                "best_density": r.best_density, "best_round": r.best_round,
                "dense_vertices": dense[:r.num_dense].copy()}


# ---- reference-shaped entry points ------------------------------------------

@dataclass
class OrientConfig:
    """orientation.hpp:18-22"""
    strategy: int = DEGREE
    epsilon: float = 1.0
    alpha_hat: Optional[int] = None


@dataclass
class DirectedGraph:
    """graph.hpp:91-121: out_offsets, out_targets (ascending by id), ranking."""
    out_offsets: np.ndarray
    out_targets: np.ndarray
    rank: np.ndarray

    @property
    def n(self):
        return len(self.out_offsets) - 1

    @property
    def m(self):
        return len(self.out_targets)

    def out_degree(self, v):
        return int(self.out_offsets[v + 1] - self.out_offsets[v])

    def out_neighbors(self, v):
        return self.out_targets[self.out_offsets[v]:self.out_offsets[v + 1]]

    def max_out_degree(self):
        return int(np.diff(self.out_offsets).max()) if self.n else 0


def _with_graph(g, fn):
    with DeviceGraph.from_graph(g) as dgh:
        return fn(dgh)


def rank_by_degree(g):
    return _with_graph(g, lambda h: h.rank(DEGREE)[0])


def rank_original(g):
    return _with_graph(g, lambda h: h.rank(ORIGINAL)[0])


def rank_by_kcore(g):
    return _with_graph(g, lambda h: h.rank(KCORE)[0])


def rank_goodrich_pszona(g, epsilon, with_rounds=False):
    r, rounds, _ = _with_graph(g, lambda h: h.rank(GOODRICH_PSZONA, epsilon))
    return (r, rounds) if with_rounds else r


def rank_barenboim_elkin(g, epsilon, alpha_hat, with_rounds=False):
    if alpha_hat < 1:
        raise ValueError("alpha_hat must be >= 1")
    r, rounds, _ = _with_graph(g, lambda h: h.rank(BARENBOIM_ELKIN, epsilon, alpha_hat))
    return (r, rounds) if with_rounds else r


def estimate_arboricity(g, epsilon):
    return _with_graph(g, lambda h: h.estimate_arboricity(epsilon))


def make_ranking(g, cfg: OrientConfig = OrientConfig()):
    a = cfg.alpha_hat or 0
    return _with_graph(g, lambda h: h.rank(cfg.strategy, cfg.epsilon, a)[0])


def direct_by_ranking(g, rank) -> DirectedGraph:
    rank = _u32(rank)
    if len(rank) != g.n:
        raise ValueError("ranking size does not match graph")

    def run(h):
        h.set_ranking(rank)
        off, tgt, _ = h.direct()
        return DirectedGraph(off, tgt, rank.copy())
    return _with_graph(g, run)


def count_total(dg: DirectedGraph, k: int) -> int:
    if k < 2:
        raise ValueError("k must be at least 2")
    with DeviceGraph.from_dag(dg.out_offsets, dg.out_targets, dg.rank) as h:
        return h.count(k)[0]


def count_per_vertex(dg: DirectedGraph, k: int):
    if k < 2:
        raise ValueError("k must be at least 2")
    with DeviceGraph.from_dag(dg.out_offsets, dg.out_targets, dg.rank) as h:
        return h.count(k, per_vertex=True)
