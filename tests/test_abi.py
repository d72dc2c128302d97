"""CPU checks of the drop-in boundary: the C-ABI library loads without a GPU,
exports every symbol include/lsg.h declares, and struct layouts match."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    hdr = open(os.path.join(ROOT, "include", "lsg.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|void|const char\*|uint64_t)\s+(lsg_\w+)\(", hdr, re.M)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("lsg_generate_trace", "lsg_build_reuse_graph", "lsg_pso_order", "lsg_plan",
              "lsg_simulate", "lsg_gather", "lsg_store_fill", "lsg_last_error"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    from paper_2211_00224_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        pytest.fail("libsolar_b200.so not built (run make lib)")
    L = ctypes.CDLL(_lib.LIB_PATH)
    for s in declared_symbols():
        assert hasattr(L, s), s
    assert set(_lib.EXPORTS) <= set(declared_symbols())
    L.lsg_version.restype = ctypes.c_int
    assert L.lsg_version() == 1


def test_config_struct_matches_oracle_layout():
    from paper_2211_00224_b200._lib import LsgConfig
    import oracle as O
    assert ctypes.sizeof(LsgConfig) == ctypes.sizeof(O.OrConfig)
    assert [f[0] for f in LsgConfig._fields_] == [f[0] for f in O.OrConfig._fields_]


def test_shape_and_validation_without_gpu():
    """Host-side validation runs without touching the device."""
    import paper_2211_00224_b200 as ls
    pc = ls.PipelineConfig(trace=ls.TraceConfig(262144, 100, 8, 512, 42, True), buffer_capacity=52428)
    sh = pc.shape()
    assert (sh.global_batch, sh.steps_per_epoch, sh.keep, sh.total_steps, sh.total_items) == \
        (4096, 64, 262144, 6400, 26214400)
    for bad in (dict(buffer_capacity=0), dict(trace=ls.TraceConfig(3, 1, 2, 2, 0, True))):
        kw = dict(trace=ls.TraceConfig(64, 1, 2, 2, 0, True), buffer_capacity=4)
        kw.update(bad)
        with pytest.raises(ls.ConfigError):
            ls.PipelineConfig(**kw).validate()
    with pytest.raises(ls.ConfigError):
        ls.PipelineConfig(trace=ls.TraceConfig(64, 1, 2, 2), buffer_capacity=4,
                          pso=ls.PsoParams(inertia=1.0)).validate()
