"""bench.py host logic that needs no GPU: the roofline arithmetic of the C5 / eval-sweep blocks,
the nvidia-smi line parser of the clock sampler and the build tag of the DRAM capture."""
import json
import os

import bench

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_roofline_of_tensor_path_arithmetic():
    bf16, _ = bench.measured_bf16_peak()
    clocks = {"sm_mhz": 1572.0, "sm_max_mhz": 1965.0, "reasons": ["sw_power_cap"], "samples": 9}
    # 2 TFLOP of algorithmic work in 10 ms = 200 TFLOP/s against bf16 / 6
    r = bench.roofline_of(2.0e12, 10.0, "tensor", 0, clocks)
    assert r["bound"] == "tensor" and r["unit"] == "TFLOP/s"
    assert abs(r["achieved"] - 200.0) < 1e-9
    assert abs(r["peak"] - bf16 / 6.0) < 1e-9
    assert abs(r["frac"] - 200.0 / (bf16 / 6.0)) < 1e-12
    # the peak rescaled to the sampled clock
    assert abs(r["frac_at_run_clock"] - r["frac"] * 1965.0 / 1572.0) < 1e-12
    # no clock samples: no run-clock fraction claimed
    r0 = bench.roofline_of(2.0e12, 10.0, "tensor", 0, None)
    assert "frac_at_run_clock" not in r0 and "clocks" not in r0


def test_clock_sampler_parses_nvidia_smi_lines():
    s = bench.ClockSampler(0)

    class P:  # a finished process
        def terminate(self):
            pass

        def wait(self, timeout=None):
            return 0

    class T:
        def join(self, timeout=None):
            pass

    s.proc, s.thread = P(), T()
    s.lines = ["0, 1965, 1965, 310.5, 0x0000000000000000, Not Active, Not Active, Not Active, Not Active",
               "0, 1575, 1965, 985.0, 0x0000000000000004, Not Active, Not Active, Not Active, Active",
               "0, 1560, 1965, 990.2, 0x0000000000000004, Not Active, Not Active, Not Active, Active",
               "garbage"]
    c = s.stop()
    assert c["sm_mhz"] == 1575.0 and c["sm_max_mhz"] == 1965.0 and c["samples"] == 3
    assert c["reasons"] == ["sw_power_cap"]
    assert c["power_w"] == 985.0


def test_dram_capture_is_tagged_with_a_build_hash():
    pj = json.load(open(os.path.join(ROOT, "profiles", "ncu_dram_per_launch.json")))
    assert set(pj) >= {"build", "capture", "per_launch"}
    assert len(pj["build"]) == 16 and len(bench.source_hash()) == 16
    assert all(k in pj["per_launch"] for k in ("fwd", "fwd_centre", "bwd", "wgrad"))
