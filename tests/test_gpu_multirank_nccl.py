"""The x-slab path over NCCL between distinct GPUs: two ranks,
one per GPU, step a strained C5-recipe block with ghost planes exchanged by
NCCL and must equal the one-GPU run bit for bit (tools/nccl_slab_check.py).
Needs >= 2 GPUs: skipped on a one-GPU box (emulated slabs and the one-rank
NCCL path cover the slab arithmetic there)."""
import os
import socket
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def _ngpu():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:   # pragma: no cover
        return 0


@pytest.mark.skipif(_ngpu() < 2, reason="needs >= 2 GPUs")
def test_two_rank_nccl_slabs_bitwise():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(ROOT, "tools", "nccl_slab_check.py"), "48", "64", "96", "80"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, (r.stdout[-3000:], r.stderr[-3000:])
    assert '"ok": true' in r.stdout
