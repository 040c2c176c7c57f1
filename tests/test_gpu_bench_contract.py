"""bench.py's JSON line keeps the driver's contract (keys, types, the roofline / e2e / clocks objects)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, cwd=ROOT, capture_output=True,
                         text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_bench_line_contract(cuda_device, tmp_path):
    man = tmp_path / "manifest.jsonl"
    d = _run(["--steps", "1", "--warmup", "3", "--no-configs", "--no-cpu-baseline", "--manifest", str(man)])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
                "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks"):
        assert key in d, key
    assert d["n_gpus"] == 1 and d["steps"] == 1 and d["warmup"] == 3 and d["higher_is_better"] is True
    assert d["value"] > 0 and d["ms_per_step"] > 0 and d["gpu_launches"] > 0
    assert "workload" in d["config"]
    r = d["roofline"]
    assert r["bound"] in ("alu", "hbm", "tensor") and 0 < r["frac"] <= 1.0 and r["achieved"] > 0 and r["peak"] > 0
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]
    # the run manifest: one JSON line with the seeded inputs' and the library's SHA-256 and the same numbers
    (m,) = [json.loads(l) for l in man.read_text().splitlines()]
    assert m["value"] == d["value"] and m["config"]["name"] == "c4" and m["seeds"] == {"mu[0]": 4000}
    assert len(m["input_sha256"]["mu[0]"]) == 64 and len(m["libse2ot_sha256"]) == 64
    assert m["gpu"]["sms"] > 0 and m["clocks"]["sm_mhz"] == d["clocks"]["sm_mhz"]


def test_bench_reference_arm_contract(cuda_device):
    d = _run(["--impl", "reference", "--steps", "1", "--warmup", "0"])
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
