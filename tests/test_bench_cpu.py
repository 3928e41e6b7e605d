"""Host logic of bench.py (no GPU): both arms describe the workload with the
same config object, and the clock sampler's window selection."""

import argparse
import importlib.util
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench():
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def test_both_arms_share_the_config_object():
    B = _bench()
    args = argparse.Namespace(dims="48x48x48x96", prec=64, recon=12)
    dims = (48, 48, 48, 96)
    V = 48 * 48 * 48 * 96
    ours = B.bench_config(args, dims, V, 1, "none")
    ref = B.bench_config(args, dims, V, 1, "nccl")  # what run_reference passes
    assert ours == ref
    assert ours["workload"] == "wilson_dslash_fp64_48x48x48x96" and ours["parallelism"] == "single"
    multi = B.bench_config(args, dims, V, 4, "p2p")
    assert "t-slab x4" in multi["parallelism"] and "48x48x48x384" in multi["parallelism"]
    assert "IPC-mapped" in multi["parallelism"]
    assert "NCCL halo exchange" in B.bench_config(args, dims, V, 2, "nccl")["parallelism"]


def test_clock_sampler_windows():
    B = _bench()
    s = B.ClockSampler(0)
    # sm, max, hw_slowdown, hw_thermal, sw_thermal, sw_power_cap, timestamp
    s.samples = [["1965", "1965", "Not Active", "Not Active", "Not Active", "Not Active", 10.00],
                 ["1965", "1965", "Not Active", "Not Active", "Not Active", "Not Active", 10.10],
                 ["1500", "1965", "Not Active", "Not Active", "Not Active", "Active", 10.90],
                 ["1490", "1965", "Not Active", "Not Active", "Not Active", "Active", 11.00]]
    burst = s.summary(9.95, 10.15)
    assert burst["sm_mhz"] == 1965.0 and burst["reasons"] == [] and burst["samples"] == 2
    sus = s.summary(10.8, 11.1)
    assert sus["sm_mhz"] == 1495.0 and sus["reasons"] == ["sw_power_cap"] and sus["sm_max_mhz"] == 1965.0
    # a window shorter than one poll takes the nearest sample
    near = s.summary(10.3, 10.32)
    assert near["samples"] == 1 and near["sm_mhz"] == 1965.0
    assert B.ClockSampler(0).summary()["reasons"] == ["unsampled"]
