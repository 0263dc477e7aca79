"""x-slab run over NCCL ranks (one process per GPU) against the one-GPU run:
    python -m torch.distributed.run --nproc-per-node P --master-addr 127.0.0.1 \\
        tools/nccl_slab_check.py [nx ny nz steps]
Each rank steps its slab of a strained C5-recipe block (fused engine, fp32 and
fp64) with ghost planes exchanged by NCCL, reads back its own voxels
(vx_read_state_owned) and hashes them; rank 0 also runs the whole block on its
GPU alone.  The partition-invariant digests (bench.py's) must be equal, and the
full-state read must equal the one-GPU state bit for bit.  Prints one JSON line
on rank 0; exit code 1 on a mismatch."""
import importlib.util
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import workloads as W  # noqa: E402
from paper_1212_2845_b200 import dist as vd  # noqa: E402
from paper_1212_2845_b200 import from_scene  # noqa: E402

spec = importlib.util.spec_from_file_location("bench", os.path.join(ROOT, "bench.py"))
bench = importlib.util.module_from_spec(spec)
spec.loader.exec_module(bench)


def main():
    nx, ny, nz, steps = (int(a) for a in (sys.argv[1:5] if len(sys.argv) >= 5 else (64, 64, 96, 100)))
    world, rank, local = vd.env_ranks()
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    sc = W.block(nx, ny, nz)
    st0 = W.strained(sc, seed=4, lift=False)
    out = {"world": world, "shape": [nx, ny, nz], "steps": steps}
    ok = True
    for prec in (32, 64):
        nid = vd.bootstrap_nccl_id(dist, rank)      # an NCCL unique id serves one communicator
        lat = from_scene(sc, precision=prec, rank=rank, nranks=world, nccl_id=nid,
                         init_state=False, engine="fused")
        ids = lat.owned_ids()
        lat.set_state_owned(*[a[ids] for a in st0])
        lat.step(steps // 2)
        lat.step(steps - steps // 2)
        mine = lat.read_state_owned()
        dg = vd.sum_over_ranks_u64(bench.state_digest(mine, ids), dist, "cuda")
        full = lat.read_state()                      # collective: global state on every rank
        lat.destroy()
        if rank == 0:
            one = from_scene(sc, precision=prec, init_state=False, engine="fused")
            one.set_state(*st0)
            one.step(steps // 2)
            one.step(steps - steps // 2)
            ref = one.read_state()
            one.destroy()
            same = all(np.array_equal(a, b) for a, b in ((full.pos, ref.pos), (full.quat, ref.quat),
                                                           (full.linmom, ref.linmom),
                                                           (full.angmom, ref.angmom),
                                                           (full.latch, ref.latch)))
            d1 = bench.state_digest(ref)
            out[f"fp{prec}"] = {"digest_ranks": f"{dg:016x}", "digest_one_gpu": f"{d1:016x}",
                                "bitwise_equal": bool(same)}
            ok = ok and same and dg == d1
    if rank == 0:
        out["ok"] = ok
        print(json.dumps(out), flush=True)
    flag = torch.tensor([0 if ok or rank != 0 else 1], device="cuda")
    dist.all_reduce(flag)
    dist.destroy_process_group()
    return int(flag.item())


if __name__ == "__main__":
    sys.exit(main())
