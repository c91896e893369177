"""The bench.py contract on the CPU: the reference arm (the oracle, --impl reference) runs
without a GPU on a small workload and prints one JSON line with the keys the driver reads."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--workload", "cfg2w",
                          "--steps", "1", "--warmup", "3"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["higher_is_better"] is False and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert "workload" in d["config"]


def test_clock_sampler_parse():
    """ClockSampler.stop parses nvidia-smi's csv and reports throttle reasons."""
    sys.path.insert(0, ROOT)
    import bench

    class FakeP:
        def terminate(self):
            pass

        def communicate(self, timeout=None):
            return ("1700, 1965, Not Active, Not Active, Not Active, Active\n"
                    "1710, 1965, Not Active, Not Active, Not Active, Active\n"
                    "300, 1965, Not Active, Not Active, Not Active, Not Active\n", "")
    s = bench.ClockSampler.__new__(bench.ClockSampler)
    s.p = FakeP()
    r = bench.ClockSampler.stop(s)
    assert r["sm_mhz"] == 1705.0 and r["sm_max_mhz"] == 1965.0 and r["reasons"] == ["sw_power_cap"]
