"""B200-native k-clique counting (arb-count) behind the reference C++ API.

The product is the CUDA C-ABI library ``lib/libkcg.so`` (include/kcg.h) and
the drop-in C++ library ``lib/libkclique_b200.so`` (include/kclique/*.hpp).
This Python package is host plumbing: ctypes bindings, generators, builds.
"""
