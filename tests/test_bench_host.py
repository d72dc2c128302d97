"""Host-side pieces of bench.py that run without a GPU: the clock sampler
(rank 0 samples every GPU of the job with one nvidia-smi process; other ranks
do not sample) and its summary of throttle reasons."""
import importlib.util
import pathlib

ROOT = pathlib.Path(__file__).resolve().parents[1]


def _bench():
    spec = importlib.util.spec_from_file_location("bench_mod", ROOT / "bench.py")
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


def test_sampler_disabled_on_other_ranks():
    b = _bench()
    with b.ClockSampler(None) as clk:
        pass
    assert clk._t is None
    assert clk.summary()["reasons"] == ["nvidia-smi unavailable"]


def test_sampler_summary_over_all_gpus():
    b = _bench()
    clk = b.ClockSampler("0,1")
    # one nvidia-smi call returns a row per GPU; both land in rows
    clk.rows = [["0", "1965", "1965", "900", "0x0", "Not Active", "Not Active", "Not Active", "Not Active"],
                ["1", "1830", "1965", "1000", "0x4", "Not Active", "Not Active", "Not Active", "Active"],
                ["0", "1900", "1965", "950", "0x0", "Not Active", "Not Active", "Not Active", "Not Active"]]
    s = clk.summary()
    assert s["sm_mhz"] == 1900.0
    assert s["sm_max_mhz"] == 1965.0
    assert s["reasons"] == ["sw_power_cap"]
    assert s["samples"] == 3
