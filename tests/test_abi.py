"""CPU-side checks of the C-ABI library: it loads and exports every symbol that
include/sa.h declares; host-only calls behave (no compute without a GPU)."""
import ctypes
import re

import pytest


def test_library_exports_every_declared_symbol(sa):
    L = sa.lib()
    names = sa.exported_symbols()
    assert "sa_index_build" in names and "sa_search" in names
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing


def test_status_strings(sa):
    for code, name in enumerate(["SA_OK", "SA_ERR_INVALID_ARG", "SA_ERR_STATE", "SA_ERR_OOM",
                                 "SA_ERR_CUDA", "SA_ERR_NCCL", "SA_ERR_UNSUPPORTED"]):
        assert sa.status_string(code) == name


def test_build_opts_defaults(sa):
    o = sa._BuildOpts()
    sa.lib().sa_build_opts_default(ctypes.byref(o))
    assert (o.dtype, o.kmeans_iters, o.train_per_list, o.seed) == (0, 20, 256, 0x5A2505)


def test_invalid_args_are_rejected_before_any_device_work(sa):
    L = sa.lib()
    h = ctypes.c_void_p()
    buf = ctypes.c_void_p(1)
    assert L.sa_index_build(None, 10, 8, 0, ctypes.byref(h)) == sa.SA_ERR_INVALID_ARG
    assert L.sa_index_build(buf, 0, 8, 0, ctypes.byref(h)) == sa.SA_ERR_INVALID_ARG
    assert L.sa_index_build(buf, 10, 0, 0, ctypes.byref(h)) == sa.SA_ERR_INVALID_ARG
    assert L.sa_index_build(buf, 10, 8, 11, ctypes.byref(h)) == sa.SA_ERR_INVALID_ARG
    assert L.sa_index_build(buf, 10, 769, 0, ctypes.byref(h)) == sa.SA_ERR_UNSUPPORTED
    assert "768" in sa.last_error()
    assert L.sa_search(None, buf, 1, 10, 0, buf, buf, None) == sa.SA_ERR_INVALID_ARG


def test_header_documents_each_entry_point():
    import os
    hdr = open(os.path.join(os.path.dirname(os.path.dirname(__file__)), "include", "sa.h")).read()
    assert "PAPER.md" in hdr
    for fn in re.findall(r"\b(sa_[a-z_0-9]+)\s*\(", hdr):
        assert fn.startswith("sa_")


def test_search_mature_validates_before_device_work(sa):
    L = sa.lib()
    buf = ctypes.c_void_p(1)
    o = sa._MaturityOpts()
    o.tau, o.window, o.check_every = 0.9, 8, 1
    assert L.sa_search_mature(None, buf, 0, 1, 10, 8, ctypes.byref(o), buf, buf, None, None, None,
                              None) == sa.SA_ERR_INVALID_ARG
    assert L.sa_search_mature(buf, buf, 0, 1, 10, 8, None, buf, buf, None, None, None,
                              None) == sa.SA_ERR_INVALID_ARG


def test_graph_and_retriever_entry_points_validate(sa):
    L = sa.lib()
    buf = ctypes.c_void_p(1)
    assert L.sa_index_build_graph(None, 64, 32, 8, 0, None) == sa.SA_ERR_INVALID_ARG
    assert L.sa_search_graph(None, buf, 0, 1, 10, 64, 4, 8, 100, buf, buf, None,
                             None) == sa.SA_ERR_INVALID_ARG
    deg = ctypes.c_int32()
    assert L.sa_index_export_graph(None, ctypes.byref(deg), None, None, None) == sa.SA_ERR_INVALID_ARG
    h = ctypes.c_void_p()
    assert L.sa_retriever_create(None, 1, 1, 1, 1, ctypes.byref(h)) == sa.SA_ERR_INVALID_ARG
    assert L.sa_retriever_set_engine_ready(None, 1) == sa.SA_ERR_INVALID_ARG
    done = ctypes.c_int32()
    assert L.sa_retriever_poll(None, 0, ctypes.byref(done)) == sa.SA_ERR_INVALID_ARG
