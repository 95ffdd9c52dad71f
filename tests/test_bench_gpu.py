"""bench.py contract on a GPU box: the JSON line's keys, the N > 1 orchestration (two ranks on one
GPU over gloo: partition, sharded generation, max-over-ranks timing, d all-gather) and the
reference arm."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def _run(cmd, env=None, timeout=900):
    e = dict(os.environ)
    e.update(env or {})
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=timeout, env=e)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_bench_line_contract():
    d = _run([sys.executable, "bench.py", "--rows", "400000", "--steps", "3", "--warmup", "3",
              "--no-cpu-baseline"])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "roofline",
              "e2e", "gpu_launches", "clocks", "cpu_baseline"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["value"] > 0 and d["dtype"] == "f64"
    assert d["roofline"]["bound"] == "hbm" and 0 < d["roofline"]["frac"] < 1.5
    assert d["e2e"]["h2d_bytes_per_step"] == 8 * 40000
    assert d["e2e"]["d2h_bytes_per_step"] == 8 * 400000
    assert d["gpu_launches"] >= 3 and d["alt_fp32"]["value"] > 0


def test_bench_two_ranks_orchestration():
    d = _run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
              "--master-addr", "127.0.0.1", "--master-port", "29533", "bench.py", "--gpus", "2",
              "--rows", "400000", "--steps", "3", "--warmup", "3", "--dist-backend", "gloo"],
             env={"DG_BENCH_ONE_DEVICE": "1"})
    assert d["n_gpus"] == 2 and d["scaling"] == "strong"
    assert d["ms_per_step_gathered"] > 0 and d["cpu_baseline"] is None
    for k in ("ms_per_step_gathered_fused", "ms_per_step_gathered_blocks"):  # IPC gathers, both modes
        assert d[k] == "unavailable: CUDA IPC" or d[k] > 0, (k, d[k])
    assert d["config"]["rows"] == 400000


def test_bench_reference_arm():
    d = _run([sys.executable, "bench.py", "--impl", "reference", "--steps", "2", "--warmup", "1",
              "--cpu-sample-rows", "20000"])
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0
