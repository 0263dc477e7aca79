"""bench.py keeps the driver's JSON contract (one line, required keys) on a
small config, both arms."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
        "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "clocks",
        "gpu_launches", "roofline", "cpu_baseline", "e2e"}


def _run(*args):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_bench_line_ours():
    d = _run("--config", "C4", "--steps", "20", "--warmup", "3", "--cpu-budget", "1")
    assert KEYS <= set(d)
    assert d["value"] > 0 and d["n_gpus"] == 1 and d["warmup"] >= 3
    assert d["gpu_launches"] > 0
    r = d["roofline"]
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= set(r)
    assert r["bound"] == "hbm" and r["unit"] == "GB/s"          # SURVEY 8(d)'s roof
    assert r["kernel_share_of_step"] <= 1.001
    assert d["repeats"]["n"] == 5 and len(d["repeats"]["region_ms"]) == 5
    assert len(d["e2e"]["final_state_digest"]) == 16
    assert r["traffic"] is None or isinstance(r["traffic"], float)   # ncu bytes per launch
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])


def test_bench_line_reference():
    d = _run("--impl", "reference", "--config", "C4", "--steps", "3", "--warmup", "3")
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle"
    assert d["e2e"]["h2d_bytes_per_step"] == 0


def test_bench_x_slab_rank_path_one_rank():
    """bench.py's N > 1 code (NCCL communicator, ghost exchange, owned-voxel
    I/O, digest summed over the group, per-rank rows) run with one rank under
    torchrun (--nccl-one): the final-state digest equals the plain run's."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    args = ["--config", "C4", "--steps", "10", "--warmup", "3", "--no-cpu", "--e2e-steps", "64"]
    plain = _run(*args)
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                          "--nproc-per-node", "1", "--master-addr", "127.0.0.1", "--master-port",
                          str(port), os.path.join(ROOT, "bench.py"), "--nccl-one", *args],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads([l for l in out.stdout.splitlines() if l.strip()][-1])
    assert line["config"]["parallelism"] == "x-slab1" and "per_rank_ms_per_step" in line
    assert "vx_set/read_state_owned" in line["e2e"]["episode"]
    assert line["e2e"]["final_state_digest"] == plain["e2e"]["final_state_digest"]
