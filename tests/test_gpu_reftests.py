"""The reference's OWN doctest unit suites (proj/tests/test_trace.cpp,
test_prng.cpp, test_epoch_order.cpp, test_reuse_graph.cpp, test_plan.cpp,
test_locality.cpp, test_balance.cpp, test_chunking.cpp, test_buffer.cpp,
test_store.cpp, test_pipeline.cpp), compiled unchanged from /root/reference
with a stand-in doctest.h and linked against the B200 C++ drop-in
(include/loadsched_gpu.hpp) instead of the reference library (oracle/Makefile
target `reftests`; the binaries travel in oracle/_ref/). Every TEST_CASE must
pass, except the few that exercise features out of scope for this tier
(the PFS access-pattern benchmark, the ablation ladder and the
run summary it feeds), which a test-only link shim (tests/cpp/shim/
out_of_scope.cpp) stubs with CapabilityError and EXCLUDE skips by name."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DIR = os.path.join(ROOT, "oracle", "_ref", "reftests")
SUITES = ["test_trace", "test_prng", "test_epoch_order", "test_reuse_graph", "test_plan", "test_locality",
          "test_balance", "test_chunking", "test_buffer", "test_store", "test_pipeline"]
EXCLUDE = {
    # store.cpp:160-235 bench_pattern / pattern_name: the PFS microbenchmark
    "test_store": ["benchmark patterns issue the documented read shapes",
                   "pattern names match the CLI vocabulary"],
    # pipeline.cpp:200-264 ablation_ladder / summary_text (summary.txt)
    "test_pipeline": ["run artifacts are byte-stable across reruns",
                      "the optimization ladder is cumulative and pays off",
                      "summaries carry the ladder, the spread and the chosen order"],
}


@pytest.mark.gpu
@pytest.mark.parametrize("suite", SUITES)
def test_reference_suite_passes_on_the_drop_in(ls, suite):
    exe = os.path.join(DIR, suite)
    if not os.path.exists(exe):
        pytest.skip("reference suites not built (needs /root/reference at build time)")
    env = dict(os.environ, LSG_DOCTEST_EXCLUDE="|".join(EXCLUDE.get(suite, [])))
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600, cwd="/tmp", env=env)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "| 0 failed |" in r.stdout, r.stdout
    assert f"| {len(EXCLUDE.get(suite, []))} skipped |" in r.stdout, r.stdout


@pytest.mark.gpu
def test_run_pipeline_writes_the_in_scope_artifacts(ls, tmp_path):
    """run_pipeline (pipeline.cpp:266-311) through the C++ drop-in writes the
    reference's trace/graph/order/plan/metrics/baseline_metrics files byte for
    byte and refuses the out-of-scope summary.txt (CapabilityError, exit 4)."""
    exe = os.path.join(ROOT, "tests", "cpp", "dropin_test")
    if not os.path.exists(exe):
        pytest.skip("drop-in driver not built")
    r = subprocess.run([exe, "run_pipeline", str(tmp_path / "ours")], capture_output=True, text=True, timeout=600)
    assert r.returncode == 4, r.stdout + r.stderr
    import oracle as O
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    want = O.ref_run_pipeline(str(tmp_path / "ref"))
    for name, data in want.items():
        if name == "summary.txt":
            continue
        assert (tmp_path / "ours" / name).read_bytes() == data, name
