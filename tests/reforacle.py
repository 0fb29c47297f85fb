"""TEST INFRASTRUCTURE ONLY: ctypes bindings for the two oracles.

* ``Ref``  — the UNMODIFIED reference library compiled from /root/reference
  (oracle/_ref/libkclique_ref.so via oracle/Makefile + oracle/ref_capi.cpp).
* ``Port`` — the plain-C restatement oracle/kc_oracle.c
  (oracle/_ref/libkcoracle.so).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg import
this module, and only as the checker.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(os.path.dirname(_HERE), "oracle", "_ref")
P = ctypes.POINTER
c_u64p = ctypes.c_void_p


def _arr(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


class OracleError(Exception):
    pass


class OracleLogicError(OracleError):
    pass


def _check(rc, what):
    if rc == 1:
        raise ValueError(f"{what}: invalid argument")
    if rc == 4:
        raise OracleLogicError(f"{what}: logic error")
    if rc != 0:
        raise OracleError(f"{what}: status {rc}")


class Ref:
    """The compiled reference library."""

    def __init__(self, path=None):
        path = path or os.path.join(REF_DIR, "libkclique_ref.so")
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = ctypes.CDLL(path)
        vp = ctypes.c_void_p
        L.ref_graph_create.argtypes = [ctypes.c_uint32, vp, vp, P(vp)]
        L.ref_graph_from_edge_list.argtypes = [ctypes.c_uint32, vp, vp, ctypes.c_uint64, P(vp)]
        L.ref_graph_destroy.argtypes = [vp]
        L.ref_graph_m.argtypes = [vp]
        L.ref_graph_m.restype = ctypes.c_uint64
        L.ref_graph_csr.argtypes = [vp, vp, vp]
        L.ref_rank.argtypes = [vp, ctypes.c_int, ctypes.c_double, ctypes.c_uint64, vp,
                               P(ctypes.c_uint64), P(ctypes.c_double)]
        L.ref_estimate_arboricity.argtypes = [vp, ctypes.c_double, P(ctypes.c_uint64)]
        L.ref_direct.argtypes = [vp, vp, P(vp), P(ctypes.c_double)]
        L.ref_direct_sized.argtypes = [vp, vp, ctypes.c_uint32, P(vp)]
        L.ref_dg_destroy.argtypes = [vp]
        L.ref_dg_csr.argtypes = [vp, vp, vp]
        L.ref_dg_max_out_degree.argtypes = [vp]
        L.ref_dg_max_out_degree.restype = ctypes.c_uint64
        L.ref_count.argtypes = [vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                P(ctypes.c_uint64), vp, P(ctypes.c_double)]
        L.ref_brute_force.argtypes = [vp, ctypes.c_int, P(ctypes.c_uint64), vp]
        L.ref_exact_arboricity.argtypes = [vp, P(ctypes.c_uint64)]
        L.ref_set_threads.argtypes = [ctypes.c_int]
        L.ref_update_counts.argtypes = [vp, vp, ctypes.c_int, vp, vp, ctypes.c_uint64, vp,
                                        P(ctypes.c_uint64), vp, P(ctypes.c_uint64)]
        L.ref_colorful_sparsify.argtypes = [vp, ctypes.c_uint64, ctypes.c_uint64, P(vp)]
        L.ref_approx_count.argtypes = [vp, ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64,
                                       ctypes.c_int, ctypes.c_double, P(ctypes.c_uint64),
                                       P(ctypes.c_double), P(ctypes.c_double)]
        L.ref_analytic_variance.argtypes = [ctypes.c_uint64, ctypes.c_double, ctypes.c_int, vp,
                                            ctypes.c_uint64]
        L.ref_analytic_variance.restype = ctypes.c_double
        L.ref_peel.argtypes = [vp, vp, ctypes.c_int, ctypes.c_int, ctypes.c_double, vp,
                               P(ctypes.c_double), vp, vp, P(ctypes.c_double)]
        self.L = L

    def set_threads(self, t):
        self.L.ref_set_threads(int(t))

    def max_threads(self):
        return int(self.L.ref_max_threads())

    def graph(self, g):
        h = ctypes.c_void_p()
        off, adj = _arr(g.offsets, np.uint64), _arr(g.adj, np.uint32)
        _check(self.L.ref_graph_create(g.n, off.ctypes.data, adj.ctypes.data, ctypes.byref(h)),
               "graph")
        return h

    def graph_from_edges(self, n, edges):
        e = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
        us, vs = _arr(e[:, 0], np.uint32), _arr(e[:, 1], np.uint32)
        h = ctypes.c_void_p()
        _check(self.L.ref_graph_from_edge_list(n, us.ctypes.data, vs.ctypes.data, len(us),
                                               ctypes.byref(h)), "from_edges")
        return h

    def graph_csr(self, h, n):
        m = int(self.L.ref_graph_m(h))
        off = np.zeros(n + 1, np.uint64)
        adj = np.zeros(2 * m, np.uint32)
        self.L.ref_graph_csr(h, off.ctypes.data, adj.ctypes.data)
        return off, adj

    def graph_digest(self, h, n):
        from paper_2002_10047_b200 import gen
        off, adj = self.graph_csr(h, n)
        return f"{gen.digest_u64(off):016x}:{gen.digest_u32(adj):016x}"

    def graph_destroy(self, h):
        self.L.ref_graph_destroy(h)

    def rank(self, h, n, strategy, eps=1.0, alpha_hat=0):
        rank = np.zeros(n, np.uint32)
        rounds = ctypes.c_uint64(0)
        secs = ctypes.c_double(0)
        _check(self.L.ref_rank(h, strategy, eps, alpha_hat, rank.ctypes.data,
                               ctypes.byref(rounds), ctypes.byref(secs)), "rank")
        return rank, int(rounds.value), float(secs.value)

    def estimate_arboricity(self, h, eps):
        out = ctypes.c_uint64(0)
        _check(self.L.ref_estimate_arboricity(h, eps, ctypes.byref(out)), "estimate")
        return int(out.value)

    def direct(self, h, rank):
        rank = _arr(rank, np.uint32)
        dg = ctypes.c_void_p()
        secs = ctypes.c_double(0)
        _check(self.L.ref_direct(h, rank.ctypes.data, ctypes.byref(dg), ctypes.byref(secs)),
               "direct")
        return dg, float(secs.value)

    def direct_sized(self, h, rank):
        rank = _arr(rank, np.uint32)
        dg = ctypes.c_void_p()
        _check(self.L.ref_direct_sized(h, rank.ctypes.data, len(rank), ctypes.byref(dg)),
               "direct")
        return dg

    def dg_csr(self, dg, n, m):
        off = np.zeros(n + 1, np.uint64)
        adj = np.zeros(m, np.uint32)
        self.L.ref_dg_csr(dg, off.ctypes.data, adj.ctypes.data)
        return off, adj

    def dg_destroy(self, dg):
        self.L.ref_dg_destroy(dg)

    def count(self, dg, n, k, parallelism=2, build_induced=True, want_pv=False):
        total = ctypes.c_uint64(0)
        secs = ctypes.c_double(0)
        pv = np.zeros(n if want_pv else 1, np.uint64)
        _check(self.L.ref_count(dg, k, parallelism, int(build_induced), int(want_pv),
                                ctypes.byref(total), pv.ctypes.data, ctypes.byref(secs)),
               "count")
        return int(total.value), (pv if want_pv else None), float(secs.value)

    def brute_force(self, h, n, k):
        total = ctypes.c_uint64(0)
        pv = np.zeros(max(n, 1), np.uint64)
        _check(self.L.ref_brute_force(h, k, ctypes.byref(total), pv.ctypes.data), "brute")
        return int(total.value), pv[:n]

    def update_counts(self, h, dg, n, k, counts, batch, peeled):
        """Reference update_counts; counts (u64, n) updated in place."""
        b = _arr(batch, np.uint32)
        pe = _arr(peeled, np.uint8)
        removed = ctypes.c_uint64(0)
        nch = ctypes.c_uint64(0)
        changed = np.zeros(max(n, 1), np.uint32)
        _check(self.L.ref_update_counts(h, dg, k, counts.ctypes.data, b.ctypes.data, len(b),
                                        pe.ctypes.data, ctypes.byref(removed),
                                        changed.ctypes.data, ctypes.byref(nch)),
               "update_counts")
        return int(removed.value), changed[:nch.value].copy()

    def colorful_sparsify(self, h, n, colors, seed):
        """Returns the sparsified reference Graph as (offsets, adjacency)."""
        out = ctypes.c_void_p()
        _check(self.L.ref_colorful_sparsify(h, colors, seed, ctypes.byref(out)), "sparsify")
        csr = self.graph_csr(out, n)
        self.graph_destroy(out)
        return csr

    def approx_count(self, h, k, colors, seed, strategy=0, eps=1.0):
        sc = ctypes.c_uint64(0)
        p = ctypes.c_double(0)
        e = ctypes.c_double(0)
        _check(self.L.ref_approx_count(h, k, colors, seed, strategy, eps, ctypes.byref(sc),
                                       ctypes.byref(p), ctypes.byref(e)), "approx_count")
        return {"sub_count": int(sc.value), "p": p.value, "estimate": e.value}

    def analytic_variance(self, true_count, p, k, pairs):
        a = _arr(pairs, np.uint64)
        return self.L.ref_analytic_variance(true_count, p, k, a.ctypes.data, len(a))

    def peel(self, h, dg, n, k, exact, eps=0.5):
        res = np.zeros(4, np.uint64)
        dens = ctypes.c_double(0)
        secs = ctypes.c_double(0)
        core = np.zeros(max(n, 1), np.uint64)
        dense = np.zeros(max(n, 1), np.uint32)
        _check(self.L.ref_peel(h, dg, k, int(exact), float(eps), res.ctypes.data,
                               ctypes.byref(dens), core.ctypes.data, dense.ctypes.data,
                               ctypes.byref(secs)), "peel")
        out = {"rounds": int(res[0]), "total_cliques": int(res[1]),
               "best_round": int(res[2]), "best_density": float(dens.value),
               "dense_vertices": dense[:int(res[3])].copy(), "seconds": float(secs.value)}
        if exact:
            out["core"] = core[:n].copy()
        return out

    def exact_arboricity(self, h):
        out = ctypes.c_uint64(0)
        _check(self.L.ref_exact_arboricity(h, ctypes.byref(out)), "arboricity")
        return int(out.value)


class Port:
    """The C restatement oracle/kc_oracle.c."""

    def __init__(self, path=None):
        path = path or os.path.join(REF_DIR, "libkcoracle.so")
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = ctypes.CDLL(path)
        vp = ctypes.c_void_p
        L.kco_rank_degree.argtypes = [ctypes.c_uint32, vp, vp]
        L.kco_estimate_arboricity.argtypes = [ctypes.c_uint32, ctypes.c_uint64, vp, vp,
                                              ctypes.c_double, P(ctypes.c_uint64)]
        L.kco_rank_be.argtypes = [ctypes.c_uint32, vp, vp, ctypes.c_double, ctypes.c_uint64,
                                  vp, P(ctypes.c_uint64)]
        L.kco_rank_kcore.argtypes = [ctypes.c_uint32, vp, vp, vp]
        L.kco_direct.argtypes = [ctypes.c_uint32, vp, vp, vp, vp, vp]
        L.kco_count.argtypes = [ctypes.c_uint32, vp, vp, ctypes.c_int, P(ctypes.c_uint64), vp]
        L.kco_alg_bytes.argtypes = [ctypes.c_uint32, vp, vp]
        L.kco_alg_bytes.restype = ctypes.c_uint64
        L.kco_update_counts.argtypes = [ctypes.c_uint32, vp, vp, ctypes.c_int, vp, vp,
                                        ctypes.c_uint64, vp, P(ctypes.c_uint64), vp,
                                        P(ctypes.c_uint64)]
        L.kco_sparsify.argtypes = [ctypes.c_uint32, vp, vp, ctypes.c_uint64, ctypes.c_uint64,
                                   vp, vp]
        L.kco_peel.argtypes = [ctypes.c_uint32, vp, vp, ctypes.c_int, ctypes.c_int,
                               ctypes.c_double, vp, P(ctypes.c_double), vp, vp]
        self.L = L

    def rank_degree(self, g):
        r = np.zeros(g.n, np.uint32)
        _check(self.L.kco_rank_degree(g.n, _arr(g.offsets, np.uint64).ctypes.data,
                                      r.ctypes.data), "rank_degree")
        return r

    def estimate_arboricity(self, g, eps):
        out = ctypes.c_uint64(0)
        _check(self.L.kco_estimate_arboricity(g.n, g.m, g.offsets.ctypes.data, g.adj.ctypes.data,
                                              eps, ctypes.byref(out)), "estimate")
        return int(out.value)

    def rank_be(self, g, eps, alpha):
        r = np.zeros(g.n, np.uint32)
        rounds = ctypes.c_uint64(0)
        _check(self.L.kco_rank_be(g.n, g.offsets.ctypes.data, g.adj.ctypes.data, eps, alpha,
                                  r.ctypes.data, ctypes.byref(rounds)), "rank_be")
        return r, int(rounds.value)

    def rank_kcore(self, g):
        r = np.zeros(g.n, np.uint32)
        _check(self.L.kco_rank_kcore(g.n, g.offsets.ctypes.data, g.adj.ctypes.data,
                                     r.ctypes.data), "rank_kcore")
        return r

    def direct(self, g, rank):
        rank = _arr(rank, np.uint32)
        off = np.zeros(g.n + 1, np.uint64)
        adj = np.zeros(g.m, np.uint32)
        self.L.kco_direct(g.n, g.offsets.ctypes.data, g.adj.ctypes.data, rank.ctypes.data,
                          off.ctypes.data, adj.ctypes.data)
        return off, adj

    def count(self, n, off, adj, k, want_pv=False):
        off, adj = _arr(off, np.uint64), _arr(adj, np.uint32)
        total = ctypes.c_uint64(0)
        pv = np.zeros(max(n, 1), np.uint64) if want_pv else None
        _check(self.L.kco_count(n, off.ctypes.data, adj.ctypes.data, k, ctypes.byref(total),
                                pv.ctypes.data if want_pv else None), "count")
        return int(total.value), (pv[:n] if want_pv else None)

    def alg_bytes(self, n, off, adj):
        off, adj = _arr(off, np.uint64), _arr(adj, np.uint32)
        return int(self.L.kco_alg_bytes(n, off.ctypes.data, adj.ctypes.data))

    def update_counts(self, g, k, counts, batch, peeled):
        """Recount-differencing restatement of update_counts; counts (u64,
        n) updated in place.  Returns (removed, changed)."""
        b = _arr(batch, np.uint32)
        pe = _arr(peeled, np.uint8)
        removed = ctypes.c_uint64(0)
        nch = ctypes.c_uint64(0)
        changed = np.zeros(max(g.n, 1), np.uint32)
        _check(self.L.kco_update_counts(g.n, g.offsets.ctypes.data, g.adj.ctypes.data, k,
                                        counts.ctypes.data, b.ctypes.data, len(b),
                                        pe.ctypes.data, ctypes.byref(removed),
                                        changed.ctypes.data, ctypes.byref(nch)),
               "update_counts")
        return int(removed.value), changed[:nch.value].copy()

    def peel(self, g, k, exact, eps=0.5):
        res = np.zeros(4, np.uint64)
        dens = ctypes.c_double(0)
        core = np.zeros(max(g.n, 1), np.uint64)
        dense = np.zeros(max(g.n, 1), np.uint32)
        _check(self.L.kco_peel(g.n, g.offsets.ctypes.data, g.adj.ctypes.data, k, int(exact),
                               float(eps), res.ctypes.data, ctypes.byref(dens),
                               core.ctypes.data, dense.ctypes.data), "peel")
        out = {"rounds": int(res[0]), "total_cliques": int(res[1]),
               "best_round": int(res[2]), "best_density": float(dens.value),
               "dense_vertices": dense[:int(res[3])].copy()}
        if exact:
            out["core"] = core[:g.n].copy()
        return out

    def sparsify(self, g, colors, seed):
        """colorful_sparsify restatement -> (offsets, adjacency)."""
        off = np.zeros(g.n + 1, np.uint64)
        adj = np.zeros(max(2 * g.m, 1), np.uint32)
        _check(self.L.kco_sparsify(g.n, g.offsets.ctypes.data, g.adj.ctypes.data, colors, seed,
                                   off.ctypes.data, adj.ctypes.data), "sparsify")
        return off, adj[:int(off[-1])]
