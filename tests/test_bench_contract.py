"""CPU: bench.py --impl reference prints one JSON line with the contract's keys (tiny config)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "tiny",
                        "--steps", "1", "--warmup", "1", "--depth", "4"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
                "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "oracle"
    assert "workload" in line["config"]


def test_reference_arm_2bit_workload():
    # --sub-bits 2 (NEXT-3): the oracle sample quantizes its substitute with 2 bits and says so
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "tiny",
                        "--steps", "1", "--warmup", "0", "--depth", "4", "--sub-bits", "2"],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert "2-bit" in line["config"]["workload"] and "2-bit substitute" in line["cpu_baseline"]["sample"]


def test_reference_arm_3bit_hqq_workload():
    # --sub-bits 3 --quant hqq (NEXT-3): the oracle sample builds a 3-bit HQQ substitute and says so
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "tiny",
                        "--steps", "1", "--warmup", "0", "--depth", "4", "--sub-bits", "3", "--quant", "hqq"],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert "3-bit g64 HQQ" in line["config"]["workload"] and "3-bit substitute" in line["cpu_baseline"]["sample"]
