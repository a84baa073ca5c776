"""bench.py keeps the driver's JSON contract (a short run on the GPU) and the reference arm
runs the oracle.  Checks the keys and their types, not the numbers."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                         cwd=ROOT, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_bench_json_contract():
    d = _run("--steps", "20", "--warmup", "3", "--no-cpu-baseline", "--c5-steps", "1")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 20 and d["warmup"] == 3 and d["value"] > 0
    assert d["config"]["workload"].startswith("C2") and "model" not in d["config"]
    r = d["roofline"]
    assert r["bound"] == "tensor" and r["unit"] == "TFLOP/s" and 0 < r["frac"] < 1.5 and r["peak"] > 0
    assert {"achieved", "traffic", "hbm_kernels"} <= set(r)
    assert r["peak_kind"] == "burst"  # a 20-step timed region is ~10 ms: the burst denominator
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] == 2 * 8192 * 4096 * 2
    assert e["d2h_bytes_per_step"] == 4 * 16 * 8192 + 2 * 8192 * 4096 * 2  # dA, dB fp32 + Y, dX bf16
    assert e["grads_only"]["value"] > 0
    assert d["gpu_launches"] == d["gpu_launches_per_step"] * 20 > 0
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"] and d["clocks"]["samples"] > 0
    assert d["speedup_vs_default"] > 0 and len(d["default_chain"]["ms_blocks"]) == 5
    c4 = d["c4_strong"]
    assert c4["global_tokens"] == 131072 and set(c4["runs"]) == {"r8", "r32", "r128"}
    assert all(v["tokens_per_s"] > 0 and v["speedup_vs_default"] > 0 for v in c4["runs"].values())
    c5 = d["c5"]
    assert c5["global_tokens"] == 65536 and c5["micro_batches"] == 8 and c5["tokens_per_s"] > 0


def test_reference_arm_contract():
    d = _run("--impl", "reference", "--steps", "1", "--warmup", "0")
    assert d["impl"] == "reference" and d["value"] > 0 and d["dtype"] == "f64"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0


def test_bench_two_ranks_gloo_code_path():
    """bench.py's data-parallel path (token shards, plan broadcast, overlapped exchange, the
    dX GEMM on the reduced ring) under torchrun with 2 ranks on this box's one GPU; the
    exchange uses gloo (CPU), so no rank's GPU kernel waits on another's.  Checks the JSON
    line, not the numbers (two ranks share one GPU)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29573", os.path.join(ROOT, "bench.py"), "--gpus", "2",
           "--steps", "3", "--warmup", "3", "--backend", "gloo", "--no-cpu-baseline", "--no-c5", "--blocks", "1"]
    out = subprocess.run(cmd, capture_output=True, text=True, cwd=ROOT, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "weak" and d["value"] > 0
    assert d["config"]["parallelism"].startswith("dp2")
    assert d["c4_strong"]["tokens_per_rank"] == 65536 and d["c4_strong"]["parallelism"].startswith("dp2")


def test_bench_gpus_must_match_world_size():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "3"],
                         capture_output=True, text=True, cwd=ROOT, timeout=300)
    assert out.returncode == 2 and "WORLD_SIZE" in out.stderr
