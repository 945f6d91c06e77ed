"""The driver's bench.py contract on the CPU leg it has: `--impl reference` times the
oracle on the host cores (configs[1] formula, a bounded sample) and prints ONE JSON
line with the keys the driver reads.  (The GPU arm is exercised by the round's GPU
runs; its line is in profiles/r02/bench_round2.json.)"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "0"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["steps"] == 1 and d["value"] > 0
    assert d["unit"] == "Gsamples/s" and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["h2d_bytes_per_step"] == 0


def test_committed_bench_line_has_the_contract_keys():
    """The last GPU bench line of the round (profiles/r02) carries the keys the driver
    and the judge read: roofline, cpu_baseline, e2e, clocks, gpu_launches."""
    d = json.load(open(os.path.join(ROOT, "profiles", "r02", "bench_round2.json")))
    for k in ("metric", "value", "unit", "roofline", "cpu_baseline", "e2e", "clocks", "gpu_launches", "config"):
        assert k in d, k
    ro = d["roofline"]
    assert ro["bound"] == "hbm" and 0 < ro["frac"] < 1.2 and abs(ro["achieved"] / ro["peak"] - ro["frac"]) < 1e-9
    assert d["gpu_launches"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert "workload" in d["config"]
