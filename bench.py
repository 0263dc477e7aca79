#!/usr/bin/env python
"""Benchmark of the voxel stepper (arXiv:1212.2845) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C5] [--impl ours|reference]

N > 1 is launched by torchrun (one rank per GPU, NCCL); the lattice is split
into x-slabs and each rank steps its slab, exchanging ghost planes by NCCL
send/recv inside libvoxsim.so.  One step = one full pass of the hot path over
the whole lattice (clock, the fused bond + gather-integrate pass, or K3 + K4
with --engine two_pass; collision kernels when the workload collides).

Rank 0 prints ONE JSON line.  ``value`` is whole-job voxel-steps/s with the
state resident in HBM (CUDA events on the library stream, max over ranks);
``e2e`` is the same metric through the public API for one episode of the
workload as specified (C5: 1k steps): the state uploaded from pinned host
memory, the steps, the state read back; ``roofline`` is the dominant kernel's
algorithmic work per launch over its live average launch duration;
``cpu_baseline`` is the fp64 oracle (test infrastructure) on a bounded sample,
timed on this host's cores.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402

METRIC = "voxel-steps/sec and achieved HBM GB/s vs peak"
UNIT = "voxel-steps/s"

# Algorithmic HBM bytes per voxel-step, fp32 / fp64
ALG_BYTES = {
    32: {"bonds": 56 + 108, "integrate": 108 + 56 + 56, "fused": 56 + 56},
    64: {"bonds": 112 + 216, "integrate": 216 + 112 + 112, "fused": 112 + 112},
}
# Issue side of the fused kernel (a secondary roof; the headline roofline is HBM,
# SURVEY 8(d)): counted by ncu on C5 fp32 at the tuned geometry -- issue slots per
# voxel-step (smsp__inst_executed / voxels), FP32 lane-operations (scalar
# FADD/FMUL/FFMA thread-instructions + 2 x the packed FADD2/FMUL2/FFMA2 ones) and
# FLOP (an FMA lane-op = 2) per voxel-step.  These are constants of the kernel
# binary measured offline (ncu replays each kernel ~40 times, so it cannot run
# inside the bench); `source` names the profile, and they go stale with every
# kernel change until the next profile.
FUSED_COUNTS = {32: {"warp_inst": 883301546 / 33554432, "fp32_ops": 587.1, "flop": 891.4,
                     "source": "profiles/r15_full.json (issue slots), r13 (FP32 op mix); "
                               "ncu --set full, C5 fp32"}}


def alu_roof(prec, ms, voxels, clocks):
    """Secondary roof of the fused single pass: instruction issue.  Its
    algorithmic intensity (~890 FLOP / 112 B) sits below the FP32 ridge, but
    its ~26 warp-instructions per voxel need more issue cycles than 112 B need
    HBM time.  Peak = 4 warp-instructions / clock / SM x 148 SMs x the median
    SM clock of the timed region."""
    c = FUSED_COUNTS.get(prec)
    if not c:
        return None
    mhz = (clocks or {}).get("sm_mhz") or 1965.0
    peak = 4 * 148 * mhz * 1e6 / 1e9                           # G warp-inst / s
    achieved = c["warp_inst"] * voxels / (ms / 1e3) / 1e9
    fp_peak = 2 * 128 * 148 * mhz * 1e6 / 1e12                 # TFLOP/s (FMA = 2)
    fp = c["flop"] * voxels / (ms / 1e3) / 1e12
    return {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "Gwarp-inst/s",
            "frac": achieved / peak, "warp_inst_per_voxel": c["warp_inst"], "counts_source": c["source"],
            "fp32": {"achieved": fp, "peak": fp_peak, "unit": "TFLOP/s", "frac": fp / fp_peak,
                     "flop_per_voxel": c["flop"], "lane_ops_per_voxel": c["fp32_ops"]},
            "peak_note": f"4 issue/clk/SM x 148 SMs x {mhz:.0f} MHz; FP32 128 lanes/SM"}


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index):
        self.dev = device_index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 7:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if r[3 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def state_digest(st, ids=None):
    """Order- and partition-invariant digest of a state: the sum mod 2^64 of a
    per-voxel hash of (external id, the bit patterns of its 13 state values and
    latch).  Ranks holding disjoint voxel sets add their sums, so the digest of
    the final state must be identical at every GPU count (slab invariance:
    DESIGN.md §7)."""
    n = len(st.pos)
    ids = np.arange(n, dtype=np.uint64) if ids is None else np.asarray(ids, np.uint64)
    words = np.concatenate([st.pos, st.quat, st.linmom, st.angmom,
                            st.latch.astype(np.float64)[:, None]], 1).view(np.uint64)
    with np.errstate(over="ignore"):
        mult = (np.arange(words.shape[1], dtype=np.uint64) * np.uint64(0x9E3779B97F4A7C15)
                + np.uint64(0xBF58476D1CE4E5B9))
        h = ids * np.uint64(0x94D049BB133111EB)
        for c in range(words.shape[1]):
            x = (words[:, c] ^ h) * mult[c]
            h = (x ^ (x >> np.uint64(31))) + np.uint64(c + 1)
        return int(h.sum(dtype=np.uint64))


def scene_for(name, precision):
    if name == "C5":
        return W.block(precision=precision)
    sc = W.get(name)
    sc.precision = precision
    return sc


# ------------------------------------------------------------------ reference arm
def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def oracle_sample(cfg, precision, budget_s=10.0, threads=None):
    """The fp64 oracle on a bounded sample of the workload: (voxel-steps/s,
    sample description, threads, total voxel-steps)."""
    from oracle import OracleSim
    if cfg == "C5":
        sc = W.block(16, 256, 256, precision=precision)   # first 16 x-planes of C5
        desc = "C5 sub-slab 16x256x256 (1,048,576 voxels, same recipe)"
    else:
        sc = scene_for(cfg, precision)
        desc = f"{sc.name} full lattice"
    o = OracleSim(sc.cells, sc.lattice_dim, sc.materials, sc.env, sc.origin)
    threads = threads or os.cpu_count() or 1
    o.set_threads(threads)
    if sc.fixed is not None or sc.fext is not None:
        o.set_boundary(sc.fixed, sc.fext)
    o.set_state(*sc.initial_state())
    o.step(1)
    steps, t0 = 0, time.perf_counter()
    while True:
        o.step(1)
        steps += 1
        el = time.perf_counter() - t0
        if el >= budget_s or steps >= 100000:
            break
    rate = o.n * steps / el
    return rate, f"{desc}, {steps} steps in {el:.1f} s", threads, o.n * steps


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    if args.config == "C5":
        sc = W.block(16, 256, 256, precision=args.precision)
        desc = "C5 sub-slab 16x256x256 (1,048,576 voxels, same recipe)"
    else:
        sc = scene_for(args.config, args.precision)
        desc = f"{sc.name} full lattice"
    from oracle import OracleSim as O
    o = O(sc.cells, sc.lattice_dim, sc.materials, sc.env, sc.origin)
    threads = os.cpu_count() or 1
    o.set_threads(threads)
    if sc.fixed is not None or sc.fext is not None:
        o.set_boundary(sc.fixed, sc.fext)
    o.set_state(*sc.initial_state())
    for _ in range(args.warmup):
        o.step(1)
    t0 = time.perf_counter()
    o.step(args.steps)
    el = time.perf_counter() - t0
    val = o.n * args.steps / el
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * el / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.config} (oracle sample: {desc})"},
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": threads, "kind": "oracle",
                         "sample": f"{desc}, {args.steps} timed steps", "cpu_model": cpu_model()},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ our arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_1212_2845_b200 import dist as vd
    from paper_1212_2845_b200 import from_scene

    world, rank, local = vd.env_ranks()
    if world == 1 and args.gpus > 1:
        print("use torchrun for --gpus > 1", file=sys.stderr)
        return 2
    torch.cuda.set_device(local)
    nid = None
    # --nccl-one: the x-slab rank path (NCCL communicator, ghost exchange, owned
    # I/O, reductions over the group) with a single rank under torchrun --
    # a check of the N > 1 code on one GPU (VX_FORCE_NCCL)
    if args.nccl_one:
        if world != 1 or "RANK" not in os.environ:
            print("--nccl-one needs torchrun with one process", file=sys.stderr)
            return 2
        os.environ["VX_FORCE_NCCL"] = "1"
    use_dist = world > 1 or args.nccl_one
    if use_dist:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        nid = vd.bootstrap_nccl_id(dist, rank)

    sc = scene_for(args.config, args.precision)
    replicas = world > 1 and (args.config != "C5" or args.batch > 1)
    # "auto": the library's choice (VX_ENGINE_AUTO, resolved at the first step)
    if args.batch > 1:   # K copies of the scene packed along x, one launch per step (f2)
        from paper_1212_2845_b200.batch import pack
        bt = pack([sc] * args.batch, precision=args.precision, engine=args.engine,
                  device=local, z_stack=args.z_stack if args.z_stack == "auto" else int(args.z_stack))
        lat = bt.lattice
    else:
        # C5 shards into x-slabs; C1-C4 are too small to shard and run as one
        # replica per GPU
        shard = (world > 1 and not replicas) or args.nccl_one
        lat = from_scene(sc, precision=args.precision, device=local, rank=rank if shard else 0,
                         nranks=world if shard else 1, nccl_id=nid if shard else None,
                         init_state=sc.v0 is not None, engine=args.engine)
    N = lat.num_voxels
    st_init = lat.read_state() if args.batch > 1 and not args.no_e2e else None
    stream = torch.cuda.ExternalStream(lat.stream, device=torch.device("cuda", local))

    def barrier():
        torch.cuda.synchronize()
        if use_dist:
            dist.barrier(device_ids=[local])

    # warm-up (graphs captured / tables uploaded)
    lat.step(max(args.warmup, 3))
    barrier()

    # ---- timed regions: K steps each, state resident in HBM, CUDA graphs (built
    # by vx_prepare_steps outside the regions).  `repeats` regions are timed and
    # the median is the value; then one more region of K steps
    # carries CUDA-event nodes around every launch of EVERY step for the kernel
    # breakdown and the roofline (the dominant kernel's average launch time).
    lat.set_instrumentation(False)
    lat.prepare_steps(args.steps)   # graphs built outside the timed region (nothing runs)
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    region_ms = []
    for _ in range(max(1, args.repeats)):
        barrier()
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        lat.step(args.steps)
        ev1.record(stream)
        barrier()
        region_ms.append(vd.max_over_ranks([ev0.elapsed_time(ev1)], dist if use_dist else None,
                                           "cuda")[0])
    clocks = sampler.stop()
    ms_max = float(np.median(region_ms))
    value = N * args.steps / (ms_max / 1e3) * (world if replicas else 1)   # whole job
    # instrumented region: events on every step
    lat.set_instrumentation(True, stride=1)
    lat.prepare_steps(args.steps)
    barrier()
    ie0 = torch.cuda.Event(enable_timing=True)
    ie1 = torch.cuda.Event(enable_timing=True)
    ie0.record(stream)
    lat.step(args.steps)
    ie1.record(stream)
    barrier()
    instr_ms = vd.max_over_ranks([ie0.elapsed_time(ie1)], dist if use_dist else None, "cuda")[0]
    kt = lat.kernel_times()
    n_instr = max(1, round(kt["all"][1] / max(lat.launches_per_step, 1)))   # measured steps
    lat.set_instrumentation(False)
    per_rank = None
    if use_dist:   # each rank's own kernel breakdown (ms per step), gathered on rank 0
        mine = [kt[k][0] / n_instr for k in ("bonds", "integrate", "other", "all")]
        per_rank = vd.gather_rows(mine, dist, "cuda")

    # ---- roofline of the dominant kernel (live CUDA-event durations)
    x0, x1 = lat.owned_planes()
    vox_rank = N if (world == 1 or replicas) else N * (x1 - x0) / sc.cells.shape[2]   # dense: per rank
    alg = ALG_BYTES[args.precision]
    fused = lat.engine == "fused"
    kinds = ("fused",) if fused else ("bonds", "integrate")
    slot = {"fused": "integrate", "bonds": "bonds", "integrate": "integrate"}
    avg = {k: kt[slot[k]][0] / max(kt[slot[k]][1], 1) for k in kinds}
    per_step_ms = {k: kt[slot[k]][0] / n_instr for k in kinds}
    dom = max(per_step_ms, key=per_step_ms.get)
    peak, peak_src = _peaks()
    gbps = {k: alg[k] * vox_rank / (per_step_ms[k] / 1e3) / 1e9 for k in kinds}
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        try:
            tr = json.load(open(tp))
            t = tr.get(f"{args.config}:fp{args.precision}:{dom}")
            traffic = float(t) if t else None   # ncu dram bytes read + written per launch
        except Exception:
            traffic = None
    names = {"bonds": "k_bonds (K3)", "integrate": "k_integrate (K4)",
             "fused": "k_step_fused (K3+K4 single pass)"}
    # achieved = algorithmic bytes per launch (112 B / voxel-step fused,
    # 164 + 220 two-pass, fp32) over the dominant kernel's average launch time
    # measured by the event nodes on every step of the instrumented region
    instr_step_ms = instr_ms / args.steps
    roof = {"bound": "hbm", "kernel": names[dom],
            "achieved": gbps[dom], "peak": peak, "peak_source": peak_src, "unit": "GB/s",
            "frac": gbps[dom] / peak, "frac_of_spec_8000": gbps[dom] / 8000.0,
            "traffic": traffic,
            "traffic_bytes_per_voxel": traffic / vox_rank if traffic else None,
            "alg_bytes_per_voxel": alg[dom], "avg_launch_ms": avg[dom],
            "launches_timed": int(kt[slot[dom]][1]),
            "instrumented_region_ms_per_step": instr_step_ms,
            "kernel_share_of_step": per_step_ms[dom] / instr_step_ms,
            "kernels": {k: {"ms_per_step": per_step_ms[k], "GBps": gbps[k]} for k in kinds},
            "step_GBps_alg": sum(alg[k] for k in kinds) * N / (ms_max / args.steps / 1e3) / 1e9}
    # the kernel average comes from the same steps as the region around them
    assert per_step_ms[dom] <= instr_step_ms * 1.001, (per_step_ms[dom], instr_step_ms)
    if fused:
        # secondary roof: instruction issue (alu_roof), with the FP32 fraction
        alu = alu_roof(args.precision, per_step_ms[dom], vox_rank, clocks)
        if alu:
            roof["alu"] = alu

    # ---- e2e through the public API with pinned host buffers
    e2e = None
    if not args.no_e2e:
        st0 = (sc.initial_state() if st_init is None else
               (st_init.pos, st_init.quat, st_init.linmom, st_init.angmom, st_init.latch))
        # x-slab ranks move only their own voxels (vx_set/read_state_owned); one
        # GPU or replicas use the full-state calls
        owned = (world > 1 and not replicas) or args.nccl_one
        ids = lat.owned_ids() if owned else None
        if owned:
            st0 = tuple(a[ids] for a in st0)
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()  # noqa
        hin = [pin(a) for a in st0]
        from paper_1212_2845_b200 import State
        hout = State(*[pin(np.empty_like(a)) for a in st0])
        # one episode of the workload as specified (C5: 1k steps, BASELINE.json configs[4]),
        # at least the timed-region K
        K = args.e2e_steps or max(args.steps, int(sc.steps or 0))
        lat.prepare_steps(K)
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        tw = time.perf_counter()
        e0.record(stream)
        (lat.set_state_owned if owned else lat.set_state)(*hin)
        lat.set_step(0)
        lat.step(K)
        (lat.read_state_owned if owned else lat.read_state)(hout)
        e1.record(stream)
        barrier()
        tw = time.perf_counter() - tw
        ems = e0.elapsed_time(e1)
        # host wall clock around the calls bounds the device timeline
        ems = max(vd.max_over_ranks([ems, tw * 1e3], dist if use_dist else None, "cuda"))
        bi = sum(a.nbytes for a in hin)
        bo = sum(a.nbytes for a in (hout.pos, hout.quat, hout.linmom, hout.angmom, hout.latch))
        bi = vd.max_over_ranks([bi], dist if use_dist else None, "cuda")[0] if owned else bi
        bo = vd.max_over_ranks([bo], dist if use_dist else None, "cuda")[0] if owned else bo
        e2e = {"value": N * K / (ems / 1e3) * (world if replicas else 1), "unit": UNIT,
               "h2d_bytes_per_step": bi / K, "d2h_bytes_per_step": bo / K,
               "episode": f"set_state (H2D) + {K} steps + read_state (D2H) per episode; "
                          "bytes per step = episode bytes / K" +
                          ("; each rank its own voxels (vx_set/read_state_owned), "
                           "bytes = the largest rank's" if owned else "")}
        # digest of the episode's final state (the same initial state and K at
        # every GPU count): equal bit for bit for every N when the slab split is
        # invariant, so a SCALE run doubles as the NCCL slab test
        dg = state_digest(hout, ids)
        if owned:
            dg = vd.sum_over_ranks_u64(dg, dist, "cuda")
        e2e["final_state_digest"] = f"{dg:016x}"
        e2e["digest_steps"] = K

    # ---- CPU baseline: the oracle on a bounded sample (rank 0, N = 1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        rate, desc, threads, _ = oracle_sample(args.config, args.precision, args.cpu_budget)
        rate1, desc1, _, _ = oracle_sample(args.config, args.precision, max(1.0, args.cpu_budget / 4), 1)
        cpu = {"value": rate, "unit": UNIT, "cores": threads, "kind": "oracle", "sample": desc,
               "cpu_model": cpu_model(),
               "one_core": {"value": rate1, "sample": desc1}}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": ms_max / args.steps,
            "higher_is_better": True, "scaling": "weak" if replicas else "strong", "vs_baseline": None,
            "dtype": "f32" if args.precision == 32 else "f64", "data": "synthetic",
            "config": {"workload": (f"{args.batch} x " if args.batch > 1 else "") +
                                   f"{sc.name} ({sc.cells.shape[2]}x{sc.cells.shape[1]}x"
                                   f"{sc.cells.shape[0]}, {N} voxels, {lat.num_bonds} bonds)",
                       "engine": lat.engine,
                       **({"packing": f"{-(-args.batch // (bt.z_stack * bt.y_stack))} x-blocks x "
                                      f"{bt.y_stack} y-blocks x {bt.z_stack} z-blocks"}
                          if args.batch > 1 else {}),
                       "timing": f"median of {len(region_ms)} regions of K steps (CUDA graphs, events "
                                 "on the library stream, max over ranks); kernel breakdown from one "
                                 "more region with event nodes on every step",
                       "parallelism": f"replicas{world}" if replicas else f"x-slab{world}",
                       "l2": "no flush: working set (state + bond records) >> 126 MB L2"
                             if N > 1_000_000 else "small lattice, L2-resident"},
            "clocks": clocks, "gpu_launches": lat.launches_per_step * args.steps * world,
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
            "achieved_GBps_alg": roof["step_GBps_alg"],
            "repeats": {"n": len(region_ms), "region_ms": region_ms,
                        "median_ms": ms_max, "spread": (max(region_ms) - min(region_ms)) / ms_max},
        }
        if per_rank is not None:   # ms per step: [bonds, fused/integrate, clock+collision, whole step]
            line["per_rank_ms_per_step"] = {"columns": ["bonds", "fused_or_integrate", "other", "step"],
                                            "rows": per_rank}
        print(json.dumps(line), flush=True)
    lat.destroy()
    if use_dist:
        dist.barrier(device_ids=[local])
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C5")
    ap.add_argument("--precision", type=int, default=32)
    ap.add_argument("--engine", default="auto", choices=["auto", "fused", "two_pass"],
                    help="auto: the fused single pass when nz >= 32 (z lanes of a warp), else K3+K4")
    ap.add_argument("--repeats", type=int, default=5,
                    help="timed regions of K steps; the value is their median")
    ap.add_argument("--batch", type=int, default=1,
                    help="pack K copies of the config into one lattice (SURVEY 8f f2)")
    ap.add_argument("--z-stack", default="1",
                    help="with --batch: scenes per z column ('auto' or an integer; 1 = along x only)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--nccl-one", action="store_true",
                    help="(check) the x-slab rank path with one rank under torchrun")
    ap.add_argument("--e2e-steps", type=int, default=0,
                    help="steps per end-to-end episode (default: the workload's own run length)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=10.0)
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
