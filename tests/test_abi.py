"""The C-ABI boundary: libraries load and export every declared symbol;
without a GPU every compute call fails loudly (no CPU fallback)."""
import os
import re
import subprocess

import pytest

from paper_2002_10047_b200 import kcg
from paper_2002_10047_b200._paths import LIB_DIR, REPO_ROOT


def _declared(header):
    text = open(os.path.join(REPO_ROOT, "include", header)).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(kcg_[a-z_]+)\s*\(", text)))


def _exported(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", os.path.join(LIB_DIR, lib)],
                         capture_output=True, text=True, check=True).stdout
    return {line.split()[-1] for line in out.splitlines() if " T " in line}


def test_libkcg_exports_every_declared_symbol():
    declared = _declared("kcg.h")
    assert len(declared) >= 18
    exported = _exported("libkcg.so")
    missing = [s for s in declared if s not in exported]
    assert not missing, missing
    assert sorted(declared) == sorted(kcg.EXPORTED)


def test_libkcg_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", os.path.join(LIB_DIR, "libkcg.so")],
                         capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_dropin_library_exports_reference_api():
    out = subprocess.run(["nm", "-DC", "--defined-only",
                          os.path.join(LIB_DIR, "libkclique_b200.so")],
                         capture_output=True, text=True, check=True).stdout
    for sym in ["kclique::rank_by_degree(kclique::Graph const&)",
                "kclique::rank_original(kclique::Graph const&)",
                "kclique::rank_by_kcore(kclique::Graph const&)",
                "kclique::rank_goodrich_pszona(kclique::Graph const&, double, unsigned long*)",
                "kclique::rank_barenboim_elkin(kclique::Graph const&, double, unsigned long, "
                "unsigned long*)",
                "kclique::estimate_arboricity(kclique::Graph const&, double)",
                "kclique::make_ranking(kclique::Graph const&, kclique::OrientConfig const&)",
                "kclique::direct_by_ranking(kclique::Graph const&, kclique::Ranking const&)",
                "kclique::count_total(kclique::DirectedGraph const&, int, "
                "kclique::CountConfig const&)",
                "kclique::count_per_vertex(kclique::DirectedGraph const&, int, "
                "kclique::CountConfig const&)",
                "kclique::default_parallelism(int)",
                "kclique::Graph::from_edges(unsigned int, std::vector<std::pair<unsigned int, "
                "unsigned int>, std::allocator<std::pair<unsigned int, unsigned int> > >)"]:
        assert sym in out, sym
    # the drop-in links the CUDA library, not a CPU engine
    deps = subprocess.run(["ldd", os.path.join(LIB_DIR, "libkclique_b200.so")],
                          capture_output=True, text=True).stdout
    assert "libkcg.so" in deps


def _has_gpu():
    try:
        kcg.device_info()
        return True
    except kcg.KcgError:
        return False


def test_no_cpu_fallback_without_gpu():
    if _has_gpu():
        pytest.skip("a GPU is present")
    with pytest.raises(kcg.KcgError):
        kcg.DeviceGraph.from_csr([0, 1, 2], [1, 0])
    with pytest.raises(kcg.KcgError):
        kcg.device_info()
