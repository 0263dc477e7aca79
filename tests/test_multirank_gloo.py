"""The N>1 path's host logic on CPU with world_size-2 (and 3) gloo process
groups: NCCL-id bootstrap, slab partition, the ghost-plane protocol (with gloo
send/recv standing in for NCCL), the self-collision surface-table protocol
(per-rank segment broadcast + motion-budget max) and the max-over-ranks
timing reduction."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    import torch
    from paper_1212_2845_b200 import dist as vd
    dist.init_process_group("gloo", rank=rank, world_size=world)
    out = {}
    # 1. NCCL bootstrap id: identical bytes on every rank
    nid = vd.bootstrap_nccl_id(dist, rank)
    ids = [None] * world
    dist.all_gather_object(ids, nid)
    out["ids_equal"] = all(x == ids[0] for x in ids) and len(ids[0]) == 128
    # 2. slab partition of a 37-plane lattice tiles [0, nx) exactly
    nx, ny, nz = 37, 3, 4
    x0, x1, xl0, xl1 = vd.ghost_planes(nx, world, rank)
    sl = [None] * world
    dist.all_gather_object(sl, (x0, x1))
    out["slabs"] = sl
    # 3. ghost-plane protocol on a box-ordered (x slowest) field, gloo for NCCL
    rng = np.random.default_rng(0)
    glob = rng.normal(size=(nx, ny, nz))
    local = np.zeros((xl1 - xl0, ny, nz))
    local[x0 - xl0:x1 - xl0] = glob[x0:x1]
    reqs = []
    bufs = {}
    if x0 > 0:
        reqs.append(dist.isend(torch.from_numpy(local[x0 - xl0].copy()), rank - 1))
        bufs["L"] = torch.zeros(ny, nz, dtype=torch.float64)
        reqs.append(dist.irecv(bufs["L"], rank - 1))
    if x1 < nx:
        reqs.append(dist.isend(torch.from_numpy(local[x1 - 1 - xl0].copy()), rank + 1))
        bufs["R"] = torch.zeros(ny, nz, dtype=torch.float64)
        reqs.append(dist.irecv(bufs["R"], rank + 1))
    for r in reqs:
        r.wait()
    if "L" in bufs:
        local[0] = bufs["L"].numpy()
    if "R" in bufs:
        local[-1] = bufs["R"].numpy()
    out["ghosts_ok"] = bool(np.array_equal(local, glob[xl0:xl1]))
    # 4. self-collision surface table, as libvoxsim runs it over
    #    NCCL: surface voxels in global box order; rank r owns the contiguous
    #    segment of its slab, packs it, and broadcasts it to every rank; the
    #    motion budget takes the max |V| over ranks (one allreduce)
    cells = rng.random((nx, ny, nz)) < 0.6
    pad = np.pad(cells, 1)
    nb = sum(np.roll(pad, s, a)[1:-1, 1:-1, 1:-1] for a in range(3) for s in (-1, 1))
    surf = np.flatnonzero((cells & (nb < 6)).ravel())          # global box ids, ascending
    state = rng.normal(size=(nx * ny * nz, 2))                  # (pos, mom) stand-ins
    plane = ny * nz
    seg = [int(np.searchsorted(surf, vd.ghost_planes(nx, world, r)[0] * plane)) for r in range(world)]
    seg.append(len(surf))
    table = torch.zeros(len(surf), 2, dtype=torch.float64)
    mine = surf[seg[rank]:seg[rank + 1]]
    assert np.all((mine // plane >= x0) & (mine // plane < x1))
    table[seg[rank]:seg[rank + 1]] = torch.from_numpy(state[mine])
    for r in range(world):
        if seg[r + 1] > seg[r]:
            part = table[seg[r]:seg[r + 1]].clone()
            dist.broadcast(part, src=r)
            table[seg[r]:seg[r + 1]] = part
    out["table_ok"] = bool(np.array_equal(table.numpy(), state[surf]))
    vmax = torch.tensor([float(np.abs(state[x0 * plane:x1 * plane, 1]).max())], dtype=torch.float64)
    dist.all_reduce(vmax, op=dist.ReduceOp.MAX)
    out["vmax_ok"] = float(vmax) == float(np.abs(state[:, 1]).max())
    # 5. max over ranks of per-rank times, the per-rank breakdown rows and the
    #    wrap-around digest sum bench.py uses (uint64 through int64 all-reduce)
    out["max"] = vd.max_over_ranks([1.0 + rank, 10.0 - rank], dist)
    out["rows"] = vd.gather_rows([float(rank), 2.0 * rank], dist)
    big = [0xFFFFFFFFFFFFFFF0 - 7 * r for r in range(world)]
    out["u64"] = (vd.sum_over_ranks_u64(big[rank], dist), sum(big) & 0xFFFFFFFFFFFFFFFF)
    dist.destroy_process_group()
    q.put((rank, out))


@pytest.mark.parametrize("world", [2, 3])
def test_multirank_host_logic_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    slabs = res[0]["slabs"]
    assert slabs[0][0] == 0 and slabs[-1][1] == 37
    assert all(slabs[i][1] == slabs[i + 1][0] for i in range(world - 1))
    sizes = [b - a for a, b in slabs]
    assert max(sizes) - min(sizes) <= 1
    for r in range(world):
        assert res[r]["ids_equal"] and res[r]["ghosts_ok"]
        assert res[r]["table_ok"] and res[r]["vmax_ok"]
        assert res[r]["max"] == [float(world), 10.0]
        assert res[r]["rows"] == [[float(q), 2.0 * q] for q in range(world)]
        assert res[r]["u64"][0] == res[r]["u64"][1]


def test_state_digest_is_partition_invariant():
    """bench.py's final-state digest: the sum over disjoint owned sets (ranks)
    equals the digest of the whole state, whatever the split; any changed bit
    changes it."""
    import importlib.util
    import os
    spec = importlib.util.spec_from_file_location("bench", os.path.join(ROOT, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    from paper_1212_2845_b200.lattice import State
    rng = np.random.default_rng(0)
    n = 1000
    st = State(rng.normal(size=(n, 3)), rng.normal(size=(n, 4)), rng.normal(size=(n, 3)),
               rng.normal(size=(n, 3)), (rng.random(n) < 0.3).astype(np.uint8))
    whole = bench.state_digest(st)
    for parts in (2, 3, 8):
        cuts = np.sort(rng.choice(np.arange(1, n), parts - 1, replace=False))
        tot = 0
        for ids in np.split(np.arange(n), cuts):
            sub = State(st.pos[ids], st.quat[ids], st.linmom[ids], st.angmom[ids], st.latch[ids])
            tot = (tot + bench.state_digest(sub, ids)) & 0xFFFFFFFFFFFFFFFF
        assert tot == whole
    st.pos[17, 1] = np.nextafter(st.pos[17, 1], np.inf)
    assert bench.state_digest(st) != whole
