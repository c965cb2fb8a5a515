"""The bench's oracle leg on the CPU (no GPU needed): `bench.py --impl reference` runs the oracle as it
stands — assembly, setup and Krylov iterations timed one by one by oracle/scripts/cpu_baseline.py —
and prints the contract's JSON line for the same metric, unit and step as the GPU arm."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_line_c2():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "C2",
                        "--steps", "3", "--warmup", "1"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads(r.stdout.strip().splitlines()[-1])
    assert d["impl"] == "reference" and d["unit"] == "s/iter" and d["higher_is_better"] is False
    assert d["steps"] == 3 and d["warmup"] == 1 and d["value"] > 0
    assert d["ms_per_step"] == round(d["value"] * 1e3, 2)
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] == 1 and cb["cpu_model"] and cb["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["unit"] == "s/iter"
    # the timed steps fit the run: W + K iterations after the oracle's own setup
    c = d["consistency"]
    assert c["timed_s"] <= c["oracle_wall_s"]
    assert "FCG" in d["config"]["workload"] or "PCG" in d["config"]["workload"]


def test_cpu_baseline_script_counts_steps():
    """oracle/scripts/cpu_baseline.py times exactly W + K iterations, restarting converged solves (C1's
    PCG converges in 5 iterations; 8 steps need two solves)."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "oracle", "scripts", "cpu_baseline.py"), "--config", "C1",
                        "--warmup", "2", "--steps", "8", "--full-solve"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads(r.stdout.strip().splitlines()[-1])
    assert len(d["step_s"]) == 8 and d["krylov"] == "PCG" and d["problem"] == "manufactured"
    assert d["full_solve"]["rc"] == 0 and d["full_solve"]["iters"] >= 1
