"""The C++ loadsched drop-in (include/loadsched_gpu.hpp) on the GPU: the
reference-style checks of tests/cpp/dropin_test.cpp, and its plan/replay
output compared with the oracle on seeded configs."""
import os
import random
import subprocess
import tempfile

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "dropin_test")


@pytest.fixture(scope="module")
def binary():
    if not os.path.exists(BIN):
        subprocess.run(["make", "-C", ROOT, "host"], check=True, capture_output=True)
    return BIN


def test_cpp_dropin_reference_checks(ls, binary):
    r = subprocess.run([binary], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout


@pytest.mark.parametrize("seed", range(6))
def test_cpp_dropin_matches_oracle(ls, binary, seed):
    rnd = random.Random(500 + seed)
    N, b = rnd.choice([2, 4, 8]), rnd.choice([2, 4, 8])
    D = N * b * rnd.randint(3, 12) + rnd.randint(0, N * b - 1)
    c = O.Cfg(D, rnd.randint(2, 6), N, b, seed=seed, buffer_capacity=rnd.randint(1, D // 2),
              drop_last=rnd.random() < 0.7, optim_order=rnd.random() < 0.8,
              optim_remap=rnd.random() < 0.8, optim_balance=rnd.random() < 0.8,
              graph_mode=rnd.choice(["global", "pernode"]), pso_iters=50)
    with tempfile.TemporaryDirectory() as d:
        subprocess.run([binary, "dump", d, str(D), str(c.num_epochs), str(N), str(b), str(seed),
                        str(c.buffer_capacity), str(int(c.drop_last)), str(int(c.optim_order)),
                        str(int(c.optim_remap)), str(int(c.optim_balance)), c.graph_mode],
                       check=True, capture_output=True, timeout=300)
        rd = lambda n: np.fromfile(os.path.join(d, n), dtype=np.uint32)  # noqa: E731
        ref = O.plan(c)
        assert np.array_equal(rd("order.u32"), ref.order)
        assert np.array_equal(rd("items.u32"), ref.items)
        assert np.array_equal(rd("nodeoff.u32"), ref.node_off.ravel())
        h, m = O.simulate(ref.items, ref.node_off, N, D, c.buffer_capacity)
        rows = rd("rows.u32").reshape(-1, 2)
        assert np.array_equal(rows[:, 0], h.ravel()) and np.array_equal(rows[:, 1], m.ravel())
        if O.ref_available():  # write_metrics / cost totals byte-identical to the reference's
            ref = O.ref_text(c)
            assert open(os.path.join(d, "metrics.csv"), "rb").read() == ref["metrics"]
            assert open(os.path.join(d, "costs.txt"), "rb").read() == ref["costs"]
