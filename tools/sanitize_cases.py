"""Small runs of every kernel family for compute-sanitizer (racecheck,
memcheck, initcheck, synccheck):

    compute-sanitizer --tool racecheck python tools/sanitize_cases.py [case ...]

Cases cover both engines, the fused row pass (FULL rows, TY = 7 and TY = 1
tiles with an odd row count -- the zrec parity across planes), its z-chunk form
(nz > 256), the (y, z) pass (nz < 64), self collision (broadphase + contact),
emulated slabs, the one-rank NCCL path, batching and state I/O.  Each runs a
few steps through the C ABI and reads the state back."""
from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import workloads as W  # noqa: E402


def _run(sc, prec=32, engine="fused", steps=4, nranks=1, nccl=False, state=None, env=None):
    from paper_1212_2845_b200 import from_scene, nccl_unique_id
    for k, v in (env or {}).items():
        os.environ[k] = str(v)
    nid = nccl_unique_id() if nccl else None
    lat = from_scene(sc, precision=prec, engine=engine, nranks=nranks, nccl_id=nid,
                     init_state=state is None)
    if state is not None:
        lat.set_state(*state)
    lat.step(steps)
    st = lat.read_state()
    lat.read_voxels(np.arange(min(lat.num_voxels, 7)))
    lat.destroy()
    for k in (env or {}):
        os.environ.pop(k, None)
    assert np.all(np.isfinite(st.pos))


def c1(prec):
    _run(W.cantilever(), prec)


def c2c(prec):
    _run(W.get("C2c"), prec, steps=3)


def c3(prec):
    _run(W.hollow_sphere(), prec, steps=3)


def tall300(prec):       # z chunks (nz > 256), FULL rows
    sc = W.block(6, 5, 300, precision=prec)
    _run(sc, prec, state=W.strained(sc, lift=False))


def n96(prec):           # FULL rows, TY = 7 with an odd tile (ny = 9: tiles of 7 and 2)
    sc = W.block(8, 9, 96, precision=prec)
    _run(sc, prec, state=W.strained(sc, lift=False), env={"VX_FUSED_TY": 7, "VX_FUSED_SX": 3})


def n96_ty1(prec):       # one-row tiles: every plane's last row is adjacent to the next plane's first
    sc = W.block(5, 4, 96, precision=prec)
    _run(sc, prec, state=W.strained(sc, lift=False), env={"VX_FUSED_TY": 1, "VX_FUSED_SX": 5})


def yz(prec):            # (y, z) pass: shallow lattice
    _run(W.walker(16, 8, 8), prec)


def two_pass(prec):
    sc = W.block(8, 9, 96, precision=prec)
    _run(sc, prec, engine="two_pass", state=W.strained(sc, lift=False))
    _run(W.hollow_sphere(n=14, r_in=4, r_out=7), prec, engine="two_pass", steps=3)


def slabs(prec):
    sc = W.block(12, 6, 70, precision=prec)
    _run(sc, prec, nranks=3, state=W.strained(sc, lift=False))
    _run(W.two_bodies(n=4), prec, nranks=2, steps=3)
    _run(sc, prec, engine="two_pass", nranks=3, state=W.strained(sc, lift=False))


def nccl1(prec):
    sc = W.block(12, 6, 70, precision=prec)
    _run(sc, prec, nccl=True, env={"VX_FORCE_NCCL": 1}, state=W.strained(sc, lift=False))


def batch(prec):
    from paper_1212_2845_b200.batch import pack
    scenes = [W.cube(contact_variant=True, n=5) for _ in range(3)]
    b = pack(scenes, precision=prec, engine="fused", z_stack=2)
    b.lattice.step(3)
    b.lattice.read_state()
    b.lattice.destroy()


CASES = dict(c1=c1, c2c=c2c, c3=c3, tall300=tall300, n96=n96, n96_ty1=n96_ty1, yz=yz,
             two_pass=two_pass, slabs=slabs, nccl1=nccl1, batch=batch)

if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    for n in names:
        for prec in (32, 64):
            CASES[n](prec)
            print(f"case {n} fp{prec} ok", flush=True)
