"""Synthetic inputs for the five BASELINE.json configs.

Thin ctypes layer over ``lib/libkcgen.so`` (host C++, OpenMP).  Input
construction is not part of the timed hot path; it only has to be
deterministic, so every config is a pure function of its parameters and
the resulting CSR is cached under ``data/`` keyed by that tuple.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

import numpy as np

from ._paths import LIB_DIR, REPO_ROOT

_lib = None


class _Csr(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_uint64),
        ("m", ctypes.c_uint64),
        ("offsets", ctypes.POINTER(ctypes.c_uint64)),
        ("adj", ctypes.POINTER(ctypes.c_uint32)),
    ]


def lib():
    global _lib
    if _lib is None:
        path = os.path.join(LIB_DIR, "libkcgen.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run __graft_entry__.build()")
        L = ctypes.CDLL(path)
        P = ctypes.POINTER
        L.kcgen_er.argtypes = [ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint64, P(_Csr)]
        L.kcgen_rmat.argtypes = [ctypes.c_int, ctypes.c_uint64, ctypes.c_double,
                                 ctypes.c_double, ctypes.c_double, ctypes.c_uint64,
                                 ctypes.c_int, P(_Csr)]
        L.kcgen_chung_lu.argtypes = [ctypes.c_uint32, ctypes.c_double, ctypes.c_double,
                                     ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                     ctypes.c_uint64, P(_Csr)]
        L.kcgen_rgg.argtypes = [ctypes.c_uint32, ctypes.c_double, ctypes.c_uint64, P(_Csr)]
        L.kcgen_from_edges.argtypes = [ctypes.c_uint32, ctypes.c_void_p, ctypes.c_void_p,
                                       ctypes.c_uint64, P(_Csr)]
        L.kcgen_digest_u32.argtypes = [ctypes.c_void_p, ctypes.c_uint64]
        L.kcgen_digest_u32.restype = ctypes.c_uint64
        L.kcgen_digest_u64.argtypes = [ctypes.c_void_p, ctypes.c_uint64]
        L.kcgen_digest_u64.restype = ctypes.c_uint64
        L.kcgen_draw.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64]
        L.kcgen_draw.restype = ctypes.c_uint64
        L.kcgen_save.argtypes = [ctypes.c_char_p, P(_Csr)]
        L.kcgen_load.argtypes = [ctypes.c_char_p, P(_Csr)]
        L.kcgen_free.argtypes = [P(_Csr)]
        L.kcgen_threads.restype = ctypes.c_int
        _lib = L
    return _lib


@dataclass
class CSR:
    """Undirected simple graph: u64 offsets[n+1], u32 adjacency[2m]
    (the layout of kclique::Graph, proj/include/kclique/graph.hpp:59-62)."""

    offsets: np.ndarray
    adj: np.ndarray
    name: str = ""
    meta: dict = field(default_factory=dict)

    @property
    def n(self) -> int:
        return len(self.offsets) - 1

    @property
    def m(self) -> int:
        return len(self.adj) // 2

    def degrees(self) -> np.ndarray:
        return np.diff(self.offsets)

    def digest(self) -> str:
        return f"{digest_u64(self.offsets):016x}:{digest_u32(self.adj):016x}"


def _take(c: _Csr, name="", meta=None) -> CSR:
    n, m = int(c.n), int(c.m)
    off = np.ctypeslib.as_array(c.offsets, shape=(n + 1,)).copy()
    adj = (np.ctypeslib.as_array(c.adj, shape=(2 * m,)).copy() if m
           else np.zeros(0, np.uint32))
    lib().kcgen_free(ctypes.byref(c))
    return CSR(off, adj, name, meta or {})


def _check(rc: int, what: str):
    if rc == 1:
        raise ValueError(f"{what}: invalid argument")
    if rc != 0:
        raise RuntimeError(f"{what}: failed with status {rc}")


def digest_u32(a: np.ndarray) -> int:
    a = np.ascontiguousarray(a, dtype=np.uint32)
    return int(lib().kcgen_digest_u32(a.ctypes.data, a.size))


def digest_u64(a: np.ndarray) -> int:
    a = np.ascontiguousarray(a, dtype=np.uint64)
    return int(lib().kcgen_digest_u64(a.ctypes.data, a.size))


def er(n: int, m: int, seed: int) -> CSR:
    c = _Csr()
    _check(lib().kcgen_er(n, m, seed, ctypes.byref(c)), "er")
    return _take(c, f"er_n{n}_m{m}_s{seed}")


def rmat(scale: int, samples: int, a=0.57, b=0.19, c_=0.19, seed=0, permute=False) -> CSR:
    c = _Csr()
    _check(lib().kcgen_rmat(scale, samples, a, b, c_, seed, int(permute), ctypes.byref(c)), "rmat")
    return _take(c, f"rmat_s{scale}_e{samples}_s{seed}_p{int(permute)}")


def chung_lu(n: int, gamma=2.1, i0=1000.0, mean=30.0, wmin=2.0, wmax=20000.0, seed=3) -> CSR:
    c = _Csr()
    _check(lib().kcgen_chung_lu(n, gamma, i0, mean, wmin, wmax, seed, ctypes.byref(c)), "chung_lu")
    return _take(c, f"cl_n{n}_g{gamma}_i{i0}_mu{mean}_s{seed}")


def rgg(n: int, mean_deg=48.0, seed=4) -> CSR:
    c = _Csr()
    _check(lib().kcgen_rgg(n, mean_deg, seed, ctypes.byref(c)), "rgg")
    return _take(c, f"rgg_n{n}_d{mean_deg}_s{seed}")


def from_edges(n: int, edges) -> CSR:
    """Graph::from_edges semantics (proj/src/graph.cpp:11-41)."""
    e = np.asarray(list(edges) if not isinstance(edges, np.ndarray) else edges,
                   dtype=np.int64).reshape(-1, 2)
    if e.size and (e.min() < 0 or e.max() >= n):
        raise ValueError("edge endpoint out of range")
    us = np.ascontiguousarray(e[:, 0], dtype=np.uint32)
    vs = np.ascontiguousarray(e[:, 1], dtype=np.uint32)
    c = _Csr()
    _check(lib().kcgen_from_edges(n, us.ctypes.data, vs.ctypes.data, len(us), ctypes.byref(c)),
           "from_edges")
    return _take(c)


def gnp(n: int, p: float, seed: int) -> CSR:
    """testutil::gnp (proj/tests/testutil.hpp:39-46): mt19937_64 raw bits,
    uniform = (x >> 11) * 2^-53, edge (u,v) for u<v iff uniform < p.
    numpy's MT19937 is the 32-bit engine, so the 64-bit engine is restated
    here (std::mersenne_twister_engine parameters for mt19937_64)."""
    mt = _MT64(seed)
    edges = []
    for u in range(n):
        for v in range(u + 1, n):
            if (mt.next() >> 11) * 2.0 ** -53 < p:
                edges.append((u, v))
    return from_edges(n, np.array(edges, dtype=np.int64).reshape(-1, 2))


class _MT64:
    """std::mt19937_64 (the C++ standard's published parameters)."""

    N, M = 312, 156
    MATRIX_A = 0xB5026F5AA96619E9
    UM, LM = 0xFFFFFFFF80000000, 0x7FFFFFFF
    MASK = (1 << 64) - 1

    def __init__(self, seed: int):
        self.mt = [0] * self.N
        self.mt[0] = seed & self.MASK
        for i in range(1, self.N):
            prev = self.mt[i - 1]
            self.mt[i] = (6364136223846793005 * (prev ^ (prev >> 62)) + i) & self.MASK
        self.idx = self.N

    def _twist(self):
        mt = self.mt
        for i in range(self.N):
            x = (mt[i] & self.UM) | (mt[(i + 1) % self.N] & self.LM)
            xa = x >> 1
            if x & 1:
                xa ^= self.MATRIX_A
            mt[i] = mt[(i + self.M) % self.N] ^ xa
        self.idx = 0

    def next(self) -> int:
        if self.idx >= self.N:
            self._twist()
        y = self.mt[self.idx]
        self.idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & self.MASK


# ---- the five BASELINE.json configs --------------------------------------

# strategy codes shared with include/kcg.h
DEGREE, ORIGINAL, KCORE, GOODRICH_PSZONA, BARENBOIM_ELKIN = 0, 1, 2, 3, 4
KCORE_PARALLEL = 5

CONFIGS = {
    1: dict(name="er_n20000_m200000", build=lambda: er(20000, 200000, 1),
            strategy=DEGREE, eps=1.0, ks=[3, 4], pv_ks=[3, 4],
            desc="Erdos-Renyi G(n=20000, m=200000), seed 1, degree order"),
    2: dict(name="rmat_s20_e16", build=lambda: rmat(20, 1 << 24, seed=2, permute=True),
            rmat=dict(scale=20, samples=1 << 24, seed=2, permute=True),
            strategy=BARENBOIM_ELKIN, eps=0.5, ks=[4, 5], pv_ks=[],
            desc="R-MAT scale 20, 16,777,216 samples, (0.57,0.19,0.19,0.05), seed 2, "
                 "permuted; Barenboim-Elkin eps=0.5"),
    3: dict(name="chunglu_n4m_i1000", build=lambda: chung_lu(4_000_000, 2.1, 1000.0, 30.0,
                                                            2.0, 20000.0, 3),
            strategy=DEGREE, eps=1.0, ks=[4, 5, 6, 7, 8], pv_ks=[],
            desc="Chung-Lu n=4M, gamma=2.1, i0=1000, mean 30, clip [2,20000], seed 3; "
                 "degree order"),
    4: dict(name="rgg_n2m_d48", build=lambda: rgg(2_000_000, 48.0, 4),
            strategy=KCORE, gpu_strategy=KCORE_PARALLEL, eps=1.0, ks=[6, 8], pv_ks=[6],
            desc="Random geometric graph n=2M, mean degree 48, seed 4; degeneracy order"),
    5: dict(name="rmat_s24_e32", build=lambda: rmat(24, 1 << 29, seed=5, permute=False),
            rmat=dict(scale=24, samples=1 << 29, seed=5, permute=False),
            strategy=DEGREE, eps=1.0, ks=[4], pv_ks=[4],
            desc="R-MAT scale 24, edge factor 32 (536,870,912 samples), seed 5; "
                 "degree order; full pipeline"),
}

def gpu_strategy(spec) -> int:
    """The ranking the GPU runs use for a config: config 4's "degeneracy-
    style peeling" is the bulk-synchronous degeneracy order (same max
    out-degree, hence the same DAG work, as the reference's sequential
    rank_by_kcore, which KCORE reproduces exactly and the parity tests use)."""
    return spec.get("gpu_strategy", spec["strategy"])


DATA_DIR = os.environ.get("KCG_DATA_DIR", os.path.join(REPO_ROOT, "data"))


def load_config_graph(cfg_id: int, cache: bool = True) -> CSR:
    """Builds (or loads the cached CSR of) config `cfg_id`."""
    spec = CONFIGS[cfg_id]
    path = os.path.join(DATA_DIR, spec["name"] + ".kcsr")
    if cache and os.path.exists(path):
        c = _Csr()
        _check(lib().kcgen_load(path.encode(), ctypes.byref(c)), "load")
        return _take(c, spec["name"])
    g = spec["build"]()
    g.name = spec["name"]
    if cache:
        os.makedirs(DATA_DIR, exist_ok=True)
        c = _Csr(g.n, g.m, g.offsets.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)),
                 g.adj.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)))
        tmp = path + ".tmp"
        _check(lib().kcgen_save(tmp.encode(), ctypes.byref(c)), "save")
        os.replace(tmp, path)
    return g
