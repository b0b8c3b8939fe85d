"""C-ABI library checks that need no GPU (-m "not gpu").

* libeh.so loads and exports every function include/eh.h declares;
* argument errors are reported before any device work (EH_EINVAL);
* without a usable CUDA device every compute entry point fails loudly -- there
  is no CPU fallback;
* the product package never imports the oracle.
"""
from __future__ import annotations

import ast
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

import paper_1503_02368_b200 as eh
from paper_1503_02368_b200 import build as ehbuild

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_functions():
    src = open(os.path.join(ROOT, "include", "eh.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(eh_[a-z0-9_]+)\s*\(", src)))


def test_library_builds_and_loads():
    path = ehbuild.build()
    assert os.path.exists(path)
    assert eh.lib() is not None


def test_every_declared_symbol_is_exported():
    declared = _header_functions()
    assert "eh_load_edges" in declared and "eh_count_triangles" in declared
    assert "eh_count_4cliques" in declared and "eh_intersect" in declared
    out = subprocess.run(["nm", "-D", "--defined-only", eh.eh.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (eh_[a-z0-9_]+)", out))
    missing = [f for f in declared if f not in exported]
    assert not missing, missing
    L = eh.lib()
    for f in declared:
        assert hasattr(L, f)
    assert set(eh.EXPORTED_SYMBOLS) == set(declared)


def test_header_compiles_as_c():
    # the boundary is plain C: no C++ types in the signatures
    code = '#include "eh.h"\nint main(void){ eh_config c = {0}; eh_stats s; (void)c; (void)s; return 0; }\n'
    r = subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), "-x", "c",
                        "-", "-o", "/dev/null"], input=code, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_argument_errors_without_device_work():
    L = eh.lib()
    assert L.eh_count_triangles(None) == eh.EH_COUNT_ERROR and L.eh_last_status() == eh.EH_EINVAL
    assert L.eh_count_4cliques(None) == eh.EH_COUNT_ERROR and L.eh_last_status() == eh.EH_EINVAL
    assert L.eh_load_edges(None, None, 5) is None and L.eh_last_status() == eh.EH_EINVAL
    assert L.eh_intersect(None, 3, None, 0, None) == eh.EH_EINVAL
    assert L.eh_graph_stats(None, None) == eh.EH_EINVAL
    L.eh_free(None)  # NULL-safe
    cfg = eh.eh.EHConfig()
    cfg.flags = 0x80
    assert L.eh_load_edges_ex(None, None, 0, ctypes.byref(cfg)) is None and L.eh_last_status() == eh.EH_EINVAL
    assert b"flags" in L.eh_last_error()
    # eh_count_batch: argument checks precede any device work
    cnt = (ctypes.c_uint64 * 1)()
    assert L.eh_count_batch(None, None, None, 1, 0, None, cnt) == eh.EH_EINVAL
    arr = (ctypes.c_void_p * 1)()
    ns = (ctypes.c_uint64 * 1)(0)
    assert L.eh_count_batch(arr, arr, ns, 1, 7, None, cnt) == eh.EH_EINVAL and b"query" in L.eh_last_error()
    cfg.flags = eh.EH_INPUT_ON_DEVICE
    assert L.eh_count_batch(arr, arr, ns, 1, 0, ctypes.byref(cfg), cnt) == eh.EH_EINVAL
    assert L.eh_count_triangles_range(None, 0, 1) == eh.EH_COUNT_ERROR and L.eh_last_status() == eh.EH_EINVAL
    assert L.eh_count_4cliques_range(None, 0, 1) == eh.EH_COUNT_ERROR and L.eh_last_status() == eh.EH_EINVAL
    assert L.eh_alg_bytes_k4(None) == eh.EH_COUNT_ERROR and L.eh_last_status() == eh.EH_EINVAL
    L.eh_release_cached_memory()  # safe with nothing cached (and without a device)
    # int-returning calls report the status of the failure itself
    out2 = (ctypes.c_uint64 * 2)()
    assert L.eh_count_lollipop(None, out2) == eh.EH_EINVAL and L.eh_count_barbell(None, out2) == eh.EH_EINVAL
    assert L.eh_triangles_per_vertex(None, None) == eh.EH_EINVAL
    assert L.eh_symmetric_stats(None, None) == eh.EH_EINVAL
    assert L.eh_graph_export(None, None, None, None, None) == eh.EH_EINVAL


def _has_cuda():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_has_cuda(), reason="checks the no-device behaviour")
def test_no_cpu_fallback_without_device():
    with pytest.raises(eh.EHError) as ei:
        eh.Graph(np.array([0, 1], np.uint32), np.array([1, 2], np.uint32))
    assert ei.value.status == eh.EH_ECUDA
    with pytest.raises(eh.EHError):
        eh.intersect(np.array([1, 2], np.uint32), np.array([2, 3], np.uint32))


def test_product_package_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_1503_02368_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            p = os.path.join(dirpath, f)
            if f.endswith(".py"):
                tree = ast.parse(open(p).read())
                for node in ast.walk(tree):
                    if isinstance(node, ast.Import):
                        assert all(not a.name.startswith("oracle") for a in node.names), p
                    if isinstance(node, ast.ImportFrom):
                        assert not (node.module or "").startswith("oracle"), p
            if f.endswith((".cu", ".cuh", ".h", ".c")):
                assert "oracle" not in re.findall(r'#include\s+"([^"]+)"', open(p).read()), p
