"""The reference arm of bench.py on CPU (-m "not gpu"): `bench.py --impl
reference` times the oracle on a bounded sample and prints one JSON line with
the contract's keys (impl, metric, value, unit, cpu_baseline, e2e, ...)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_oracle_sample_is_bounded_and_labelled():
    import bench
    r = bench.oracle_sample(0, seconds=0.5, omega=1.9)
    assert r["kind"] == "oracle" and r["cores"] == 1 and r["unit"] == "GNode-sweeps/s"
    assert r["value"] > 0 and "config0" in r["sample"]


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--workload",
                          "0", "--steps", "1", "--warmup", "0", "--ref-seconds", "1"], capture_output=True, text=True, timeout=300,
                         cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "config", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
    assert line["cpu_baseline"]["kind"] == "oracle"
