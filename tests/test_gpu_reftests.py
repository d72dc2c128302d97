"""The reference's OWN doctest unit suites (proj/tests/test_trace.cpp,
test_prng.cpp, test_epoch_order.cpp, test_reuse_graph.cpp, test_plan.cpp),
compiled unchanged from /root/reference with a stand-in doctest.h and linked
against the B200 C++ drop-in (include/loadsched_gpu.hpp) instead of the
reference library (oracle/Makefile target `reftests`; the binaries travel in
oracle/_ref/). Every TEST_CASE must pass."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DIR = os.path.join(ROOT, "oracle", "_ref", "reftests")
SUITES = ["test_trace", "test_prng", "test_epoch_order", "test_reuse_graph", "test_plan", "test_locality",
          "test_balance", "test_chunking", "test_buffer"]


@pytest.mark.gpu
@pytest.mark.parametrize("suite", SUITES)
def test_reference_suite_passes_on_the_drop_in(ls, suite):
    exe = os.path.join(DIR, suite)
    if not os.path.exists(exe):
        pytest.skip("reference suites not built (needs /root/reference at build time)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600, cwd="/tmp")
    assert r.returncode == 0, r.stdout + r.stderr
    assert "| 0 failed |" in r.stdout, r.stdout
