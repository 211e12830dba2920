#!/usr/bin/env python
"""Benchmark: batched multi-robot MotVal + FFC on B200 (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg5] [--impl mrv|reference]

A step = one pass of the whole hot path over one batch: MotVal (Alg. 1, obstacle +
robot-robot, rake-ordered early exit) and FFC (Alg. 2) over every motion of the
config (default cfg5: 4 manipulators, 2^20 motions x 128 timesteps) -- independent
queries, FFC on a second stream so it takes the SMs MotVal's tail frees (--serial: one
stream) -- followed for N > 1 by the NCCL all-gather of the per-motion results.  The
roofline times each query's kernel alone.  Motions are sharded by
index across ranks (one process per GPU, torchrun); total work is fixed
("scaling": "strong", BASELINE.json configs[4]).

value = robot-states validated per second, whole job:
        n_robots * sum_m T_m * (#queries in the step) / step time (max over ranks).
Inputs are resident in HBM when the timed region starts; L2 is flushed (256 MiB
memset, outside the CUDA-event intervals) before every timed step.
"""
import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

BJ_METRIC = "validated multi-robot states/s (MotVal, FFC) at 1/2/4/8 B200; % FP32 roofline"
# the paper's own numbers for this path, quoted with their hardware (context only: the
# paper reports speedup ratios and effort, no absolute rates)
PAPER_CONTEXT = {"motval_speedup_vs_fcl": "1109x (combined rake, 4 Pandas, Cage with obstacles, 1000 random motions; "
                                          "PAPER.md:529, :14, :97)",
                 "motval_effort": "0.2% of CC calls before termination (hierarchical rake, 16 Pandas; PAPER.md:529)",
                 "hardware": "Intel Core i7-14700F (<= 5.4 GHz), 32 GB, Linux 6.8, CPU SIMD via VAMP (PAPER.md:494)",
                 "ffc": "no FFC validation timing is reported"}
UNIT = "robot-states/s"
QUERIES = {"cfg1": ("motval", "ffc"), "cfg2": ("motval", "ffc"), "cfg3": ("motval", "ffc"), "cfg4": ("ffc",),
           "cfg5": ("motval", "ffc"), "pp5": ("pp_motval",)}
WORKLOAD = {
    "cfg1": "cfg1: 2 SE(2) bodies x 4 discs, 16 disc obstacles, 256 motions x 64 timesteps",
    "cfg2": "cfg2: 4 x 7-DOF arms (56 spheres each), 32 AABBs, 4096 motions, T = 1 + ceil(max|dq|/0.05)",
    "cfg3": "cfg3: 8 SE(3) bodies x 20 spheres, 100 spheres + 100 AABBs, 65536 motions x 96 timesteps",
    "cfg4": "cfg4: 4 arms + 8 SE(3) bodies, FFC, 16384 path sets, 10 knots, 1000 timesteps",
    "cfg5": "cfg5: 4 x 7-DOF arms (cfg2 scene), 1,048,576 motions x 128 timesteps, sharded by motion index",
    "pp5": "pp5: PP-ST-RRT MotVal variant (PAPER.md:399-406, SURVEY f2): arm 3 of the cfg2 scene vs the fixed paths "
           "of arms 0-2 (65 knots over 4096 absolute timesteps), 1,048,576 candidate motions x 128 timesteps at random "
           "start times; the partner table is rebuilt every step",
}
# FP32 cost model of the ALGORITHMIC work: the FADD / FMUL / FFMA
# operations (the 128-lane-per-SM FMA pipe that `peak` counts; one FFMA = one lane-op)
# the method's arithmetic needs per unit, counted from the kernel's work counters
# (MRV_CNT_*).  Compares, min/max, selects and MUFU sin/cos/sqrt/rcp run on other pipes
# and are not counted.
#   joint: lerp 2 + sincos range reduction 4 + DH compose 3 rows x 10 = 36
#   group_bound: link frame x local centre, 9 FFMA;  sphere_xform: 9
#   merge (one Ritter step growing a supergroup bound): d 3, d^2 3, tests 2, R' 3, f 2, C' 3 = 16
#   sphere-sphere test (rr_super / rr_broad / rr_narrow / sphere obstacles): d 3, d^2 3, (Ra+Rb)^2 2 = 8
#   sphere-box test (box obstacles): clamped e 6, e^2 3, R^2 1 = 10
#   se3_pose: position lerp 6, slerp angle 22, Taylor sines 3 x 7, weights 2, blend 8, rotation 21 = 80
#   se2_pose: lerp 6, sincos 4, = 10
#   capsule prefilter (group pair): 4 endpoint transforms 24, segment vectors 9, five dots 15,
#     closest-point step 9, D 6, |D|^2 3, gradients 8, lower bound 8, margin + radius 6 = 88
COST = {"joint": 36, "se3_pose": 80, "se2_pose": 10, "group_bound": 9, "merge": 16, "env_sphere": 8,
        "env_box": 10, "rr_test": 8, "sphere_xform": 9, "capsule": 88}
# SURVEY.md §8(d)'s original weights ("chain joint ~60 incl. sincosf; sphere transform 9;
# sphere-sphere test 7; sphere-AABB 16; SE(3) pose 45"): they count compares and MUFU work
# too and have no merge / capsule entries.  Reported beside COST.
SURVEY_COST = {"joint": 60, "se3_pose": 45, "se2_pose": 10, "group_bound": 9, "merge": 0, "env_sphere": 7,
               "env_box": 16, "rr_test": 7, "sphere_xform": 9, "capsule": 0}


def args_():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg5", choices=sorted(QUERIES))
    ap.add_argument("--impl", default="mrv", choices=["mrv", "reference"])
    ap.add_argument("--motval-order", default="combined", choices=["combined", "hierarchical"])
    ap.add_argument("--motions", type=int, default=None, help="override M (prefix of the config's motions)")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="target CPU time of the cpu_baseline sample")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--serial", action="store_true", help="MotVal then FFC on one stream (default: FFC on a second "
                    "stream, filling MotVal's launch tail)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-seconds", type=float, default=None,
                    help="--impl reference: CPU seconds per step (default: the run fits in ~2 minutes)")
    ap.add_argument("--launcher-check", action="store_true",
                    help="CPU / gloo check of the N-rank plumbing (spawn, shard, in-place all-gather, max over "
                         "ranks) with index-derived placeholder results; prints a check line, not a bench value")
    ap.add_argument("--no-roofline-nee", action="store_true",
                    help="skip the MRV_DIAG_NO_EARLY_EXIT roofline launches")
    return ap.parse_args()


# ------------------------------------------------------------------ N-rank launcher
def _free_port():
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def spawn_ranks(a):
    """``--gpus N > 1`` without torchrun's environment: start N ranks ourselves, one process
    per GPU, exactly as the driver's ``torch.distributed.run`` launch does (rank 0 prints
    the JSON line; the others print nothing)."""
    import subprocess
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={a.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def check_world(a, world):
    if a.gpus != world:
        raise SystemExit(f"bench.py: --gpus {a.gpus} but {world} rank(s) started (WORLD_SIZE); "
                         f"run `python bench.py --gpus {a.gpus}` or torchrun --nproc-per-node {a.gpus}")


def launcher_check(a):
    """The N-rank plumbing of the GPU arm on CPU (gloo): the same shard / pad / in-place
    all-gather / max-over-ranks calls, with per-motion placeholder results derived from the
    motion index (so the gathered arrays are checkable) in place of the kernels."""
    import torch

    from paper_2604_23960_b200 import dist as D
    from paper_2604_23960_b200 import gen
    rank, world, _ = D.init_from_env("gloo")
    check_world(a, world)
    sc, mo = gen.make(a.config, a.motions)
    M = mo.M
    lo, hi, per = D.shard(M, rank, world)
    valid_all = torch.full((world * per,), 255, dtype=torch.uint8)
    key_all = torch.full((world * per,), -7, dtype=torch.int32)
    m = torch.arange(rank * per, (rank + 1) * per, dtype=torch.int64)
    valid_all[rank * per:(rank + 1) * per] = (m % 3 == 0).to(torch.uint8)
    key_all[rank * per:(rank + 1) * per] = (m * 7 + 1).to(torch.int32)
    D.gather_inplace(valid_all, per, rank, world)
    D.gather_inplace(key_all, per, rank, world)
    mm = torch.arange(M, dtype=torch.int64)
    ok = bool(torch.equal(valid_all[:M], (mm % 3 == 0).to(torch.uint8)) and
              torch.equal(key_all[:M], (mm * 7 + 1).to(torch.int32)))
    per_rank = D.all_ranks(float(hi - lo), world)
    t_max = D.max_over_ranks(float(rank + 1), world)
    oks = D.all_ranks(1.0 if ok else 0.0, world)
    if rank == 0:
        print(json.dumps({"launcher_check": all(x == 1.0 for x in oks) and t_max == float(world), "n_gpus": world,
                          "backend": "gloo", "motions": M, "motions_per_rank": per_rank, "gathered_ok_per_rank": oks,
                          "max_over_ranks": t_max}), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    if not all(x == 1.0 for x in oks):
        raise SystemExit(1)


# ------------------------------------------------------------------ clocks sampler (NVML)
class Clocks:
    REASONS = {"gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4, "hw_slowdown": 0x8,
               "sync_boost": 0x10, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "hw_power_brake_slowdown": 0x80, "display_clock_setting": 0x100}

    def __init__(self, index):
        self.samples, self.reasons, self.ok = [], set(), False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max = None
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                try:
                    r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                except Exception:
                    r = self.nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                for name, bit in self.REASONS.items():
                    if r & bit and name not in ("gpu_idle",):
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.01)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        return json.load(open(p)), "measured"
    return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


def cost_ops(c, sc, query, COST=COST):
    """Algorithmic FP32 FMA-pipe lane-ops of one launch from its work counters."""
    from paper_2604_23960_b200 import gen
    n_se3 = sum(r.kind == gen.SE3 for r in sc.robots)
    n_se2 = sum(r.kind == gen.SE2 for r in sc.robots)
    groups = [int(np.ceil(np.bincount(r.sphere_link).clip(0) / 32).sum()) for r in sc.robots]
    n_groups = sum(groups)
    # supergroups of <= 3 consecutive groups: a robot with g groups merges g - ceil(g / 3) times
    merges = sum(g - -(-g // 3) for g in groups)
    states = c["states"]
    ops = c["joints"] * COST["joint"] + states * (n_se3 * COST["se3_pose"] + n_se2 * COST["se2_pose"]
                                                  + n_groups * COST["group_bound"] + merges * COST["merge"])
    nbox, nsph = len(sc.obs_boxes), len(sc.obs_spheres)
    w_env = (nbox * COST["env_box"] + nsph * COST["env_sphere"]) / max(1, nbox + nsph)
    ops += (c["env_broad"] + c["env_narrow"]) * w_env
    ops += (c["rr_super"] + c["rr_broad"] + c["rr_narrow"] + c["self_broad"]) * COST["rr_test"]
    ops += c["sphere_xform"] * COST["sphere_xform"]
    ops += c.get("rr_capsule", 0) * COST["capsule"]
    return float(ops)


# ------------------------------------------------------------------ CPU oracle timing
def load_workload(a):
    """(scene, motions, pp) of --config: pp = the PP-ST-RRT workload's fixed paths and
    start times (pp5), else None."""
    from paper_2604_23960_b200 import gen
    if a.config == "pp5":
        sc, paths, cand, t0 = gen.make_pp(a.motions)
        return sc, cand, {"paths": paths, "t0": t0}
    sc, mo = gen.make(a.config, a.motions)
    return sc, mo, None


def time_oracle(sc, mo, queries, seconds, check_env=True, n_fixed=None, pp=None):
    """Oracle (as it stands, sequential linear scan with early exit -- the paper's
    'sphere-based' baseline shape) on a bounded prefix sample (sized to
    `seconds`, or exactly `n_fixed` motions)."""
    import oracle
    from paper_2604_23960_b200 import gen
    oracle.build()
    n = min(mo.M, n_fixed or 256)
    while True:
        sub = mo.subset(np.arange(n))
        t0 = time.perf_counter()
        if "motval" in queries:
            oracle.baseline_motval(sc, sub, check_env=check_env)
        if "ffc" in queries:
            oracle.baseline_ffc(sc, sub)
        if "pp_motval" in queries:   # the plain-definition PP variant (stops at a definite hit)
            oracle.pp_motval(sc, gen.PP_FOCUS, gen.PP_PARTNERS, sub, pp["t0"][:n], pp["paths"], gen.PP_HORIZON,
                             check_env=check_env)
        dt = time.perf_counter() - t0
        if n_fixed or dt >= seconds * 0.8 or n >= mo.M:   # the timed sample: ~10-20 s of CPU work at 12 s
            break
        n = min(mo.M, max(n * 2, int(n * 1.1 * seconds / max(dt, 1e-3))))
    states = sub.total_states() * sc.n_robots * len(queries)
    return {"value": states / dt, "unit": UNIT, "cores": oracle.threads(), "kind": "oracle", "n": n,
            "seconds": dt, "robot_states": int(states),
            "sample": f"first {n} of {mo.M} motions of the same config ({sub.total_states()} composite states), "
                      f"queries {'+'.join(queries)}, fp64 scalar C, early exit at first strict hit, "
                      f"{oracle.threads()} threads, {dt:.2f} s"}


def config_dict(a, sc, mo, queries, n_ranks):
    """The ``config`` object of the JSON line -- identical for the GPU and the reference arm."""
    from paper_2604_23960_b200 import gen
    d = {"workload": WORKLOAD[a.config], "queries": list(queries), "motions": int(mo.M),
            "composite_states": int(mo.T_array().astype(np.int64).sum()), "n_robots": sc.n_robots,
            "parallelism": f"motion-index dp{n_ranks}",
            "motval_flags": (("check_env|combined (default flags: spread packing, DESIGN.md reading c.28)"
                              if a.motval_order == "combined" else "check_env|hierarchical (Alg. 1 rake batches)")
                             if "motval" in queries else
                             "check_env|combined|rake" if "pp_motval" in queries else None),
            "l2": "flushed before every timed step (256 MiB memset outside the event interval)",
            "scene_sha256": gen.scene_digest(sc)[:16]}
    if a.config == "pp5":
        d.update(horizon=gen.PP_HORIZON, focus=gen.PP_FOCUS, partners=list(gen.PP_PARTNERS))
    return d


def run_reference(a):
    """--impl reference: the oracle on the box's host cores (rank 0 only; the other ranks
    of a torchrun launch exit without work).  Each step times the same bounded prefix
    sample of the workload; ``ms_per_step`` is that sample's measured time."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    sc, mo, pp = load_workload(a)
    q = QUERIES[a.config]
    # calibrate a per-step sample so the whole run stays within a few minutes
    per_step = a.ref_seconds or max(1.0, min(20.0, 120.0 / max(1, a.steps + a.warmup)))
    cal = time_oracle(sc, mo, q, per_step, pp=pp)
    vals, secs = [], []
    for i in range(a.warmup + a.steps):   # every step times the same calibrated sample
        r = time_oracle(sc, mo, q, per_step, n_fixed=cal["n"], pp=pp)
        if i >= a.warmup:
            vals.append(r["value"])
            secs.append(r["seconds"])
    v = float(statistics.median(vals))
    n_ranks = int(os.environ.get("WORLD_SIZE", str(a.gpus)))
    line = {"impl": "reference", "metric": BJ_METRIC, "value": v, "unit": UNIT,
            "n_gpus": 0, "n_gpus_note": f"CPU oracle on rank 0's host cores (launched with --gpus {a.gpus})",
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": float(statistics.median(secs)) * 1e3,
            "ms_per_step_note": f"measured time of one step = the oracle over the first {cal['n']} of {mo.M} motions",
            "sample_robot_states_per_step": cal["robot_states"],
            "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded generators, paper_2604_23960_b200/gen.py)",
            "config": config_dict(a, sc, mo, q, n_ranks),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cal["cores"], "kind": "oracle", "sample": cal["sample"]},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "paper_context": PAPER_CONTEXT}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU arm
def main():
    a = args_()
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ and (a.impl == "mrv" or a.launcher_check):
        sys.exit(spawn_ranks(a))
    if a.launcher_check:
        launcher_check(a)
        return
    if a.impl == "reference":
        run_reference(a)
        return
    import torch

    from paper_2604_23960_b200 import dist as D
    from paper_2604_23960_b200 import gen, mrv

    rank, world, local = D.init_from_env("nccl")
    check_world(a, world)
    torch.cuda.set_device(local)
    if a.config == "pp5":
        return main_pp(a, rank, world, local)
    dev = torch.device("cuda", local)
    queries = QUERIES[a.config]
    sc, mo = gen.make(a.config, a.motions)
    M = mo.M
    lo, hi, per = D.shard(M, rank, world)
    wp_local = torch.from_numpy(np.ascontiguousarray(mo.waypoints[lo:hi]))
    T_all = mo.T_array()
    if mo.n_timesteps is None:
        T_arg = int(mo.fixed_timesteps)
        T_local_host = None
    else:
        T_local_host = D.pad_rows(torch.from_numpy(np.ascontiguousarray(mo.n_timesteps[lo:hi])), per)
        T_arg = T_local_host.to(dev)
    wp_host = D.pad_rows(wp_local, per).pin_memory()
    wp = wp_host.to(dev)
    gs = mrv.Scene(sc, device=local)
    flags = mrv.CHECK_ENV | (mrv.ORDER_HIERARCHICAL if a.motval_order == "hierarchical" else 0)
    valid_all = torch.empty(world * per, dtype=torch.uint8, device=dev)
    key_all = torch.empty(world * per, dtype=torch.int32, device=dev)
    my_valid = valid_all[rank * per:(rank + 1) * per]
    my_key = key_all[rank * per:(rank + 1) * per]
    stream = torch.cuda.current_stream()

    # MotVal and FFC are independent queries over the same batch: FFC runs on a second
    # stream so its CTAs take each SM as MotVal's persistent CTAs drain (no idle launch
    # tail between them); --serial runs them back to back on one stream.
    s2 = torch.cuda.Stream(device=dev)
    fork = torch.cuda.Event()

    def step(ev=None):
        concurrent = not a.serial and len(queries) == 2
        if concurrent:
            fork.record(stream)
            s2.wait_event(fork)
        if "motval" in queries:
            gs.motval(wp, T_arg, flags, out=my_valid, stream=stream)
        if ev is not None:
            ev[0].record(stream)
        if "ffc" in queries:
            gs.ffc(wp, T_arg, out=my_key, stream=s2 if concurrent else stream)
            if concurrent:
                if ev is not None:
                    ev[1].record(s2)
                stream.wait_stream(s2)
            elif ev is not None:
                ev[1].record(stream)
        if world > 1:
            if ev is not None:
                ev[2].record(stream)
            if "motval" in queries:
                D.gather_inplace(valid_all, per, rank, world)
            if "ffc" in queries:
                D.gather_inplace(key_all, per, rank, world)

    for _ in range(max(3, a.warmup)):
        step()
    torch.cuda.synchronize()

    # algorithmic work of one launch of each query (untimed counting launch, same flags)
    counts = {}
    for q in queries:
        c = torch.zeros(mrv.NUM_COUNTERS, dtype=torch.int64, device=dev)
        if q == "motval":
            gs.motval(wp, T_arg, flags, counters=c)
        else:
            gs.ffc(wp, T_arg, counters=c)
        counts[q] = dict(zip(mrv.COUNTER_NAMES, (int(x) for x in c.cpu().tolist())))
    torch.cuda.synchronize()

    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    K = a.steps
    ev = [tuple(torch.cuda.Event(enable_timing=True) for _ in range(5)) for _ in range(K)]
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    wall0 = time.perf_counter()
    with Clocks(local) as clk:
        for k in range(K):
            flush.zero_()
            ev[k][0].record(stream)
            step(ev[k][1:3] + ev[k][4:5])   # MotVal end, FFC end, gather start (N > 1)
            ev[k][3].record(stream)
        torch.cuda.synchronize()
    wall = time.perf_counter() - wall0
    if world > 1:
        torch.distributed.barrier()
    concurrent = not a.serial and len(queries) == 2
    step_ms = [e[0].elapsed_time(e[3]) for e in ev]
    mv_ms = [e[0].elapsed_time(e[1]) for e in ev] if "motval" in queries else [0.0] * K
    # FFC: from the step start when it runs beside MotVal, else after MotVal
    ffc_ms = [(e[0] if (concurrent or "motval" not in queries) else e[1]).elapsed_time(e[2]) for e in ev]
    per_rank_ms = D.all_ranks(sum(step_ms) / K, world, dev)
    # N > 1: the in-place all-gather's share of the step (gather start -> step end) and
    # each rank's kernel-only time (SURVEY §8(d) multi-GPU protocol)
    gather_ms = [e[4].elapsed_time(e[3]) for e in ev] if world > 1 else [0.0] * K
    per_rank_kernel_ms = D.all_ranks(sum(t - g for t, g in zip(step_ms, gather_ms)) / K, world, dev)
    allgather_ms = D.max_over_ranks(sum(gather_ms) / K, world, dev)
    step_sorted = sorted(step_ms)
    total_ms = D.max_over_ranks(sum(step_ms), world, dev)
    ms_per_step = total_ms / K
    mv_avg = D.max_over_ranks(sum(mv_ms) / K, world, dev) if "motval" in queries else 0.0
    ffc_avg = D.max_over_ranks(sum(ffc_ms) / K, world, dev) if "ffc" in queries else 0.0

    # each query's kernel alone (untimed w.r.t. the step, L2 flushed): the roofline's
    # duration, since inside the step FFC shares the SMs with MotVal's tail
    alone = {}
    for q in queries:
        ts = []
        for _ in range(3):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            if q == "motval":
                gs.motval(wp, T_arg, flags, out=my_valid, stream=stream)
            else:
                gs.ffc(wp, T_arg, out=my_key, stream=stream)
            e1.record(stream)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        alone[q] = D.max_over_ranks(sum(ts) / len(ts), world, dev)

    n = sc.n_robots
    state_bytes = int(wp_host.numel()) * 4 + (0 if T_local_host is None else int(T_local_host.numel()) * 4)
    comp_states = int(T_all.astype(np.int64).sum())
    robot_states_step = comp_states * n * len(queries)
    value = robot_states_step / (ms_per_step / 1e3)

    # roofline of the dominant kernel (FP32 ALU-bound)
    peaks, peak_src = measured_peaks()
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    clk_s = clk.summary()
    f_max = float(clk_s["sm_max_mhz"] or peaks.get("sm_max_mhz", 1965.0))
    peak = sms * 128 * f_max * 1e6 / 1e12          # T lane-ops/s
    dom = max(alone, key=alone.get)
    dom_ms = alone[dom]
    ops_local = cost_ops(counts[dom], sc, dom)
    achieved = ops_local / (dom_ms / 1e3) / 1e12   # per launch on this rank / its max-over-ranks duration
    ops_survey = cost_ops(counts[dom], sc, dom, SURVEY_COST)
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get(a.config, {}).get(dom)
        except Exception:
            traffic = None
    roof = {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "Tlane-ops/s", "frac": achieved / peak,
            "traffic": traffic, "kernel": f"mrv_query_kernel<{dom}>", "kernel_ms": dom_ms,
            "peak_source": f"{sms} SMs x 128 FP32 lanes x {f_max:.0f} MHz (NVML max SM clock)",
            "frac_at_observed_clock": (achieved / (sms * 128 * clk_s['sm_mhz'] * 1e6 / 1e12)) if clk_s["sm_mhz"] else None,
            "ops_per_launch": ops_local, "counters": counts[dom],
            "weights": {"fma_pipe": COST, "survey": SURVEY_COST},
            "frac_survey_weights": ops_survey / (dom_ms / 1e3) / 1e12 / peak}

    # SURVEY §8(d) headline: the same kernel with MRV_DIAG_NO_EARLY_EXIT, so every state of
    # every motion is evaluated (deterministic work, independent of where conflicts fall)
    if not a.no_roofline_nee:
        nee = {}
        for q in queries:
            fl = (flags if q == "motval" else 0) | mrv.DIAG_NO_EARLY_EXIT
            c = torch.zeros(mrv.NUM_COUNTERS, dtype=torch.int64, device=dev)
            if q == "motval":
                gs.motval(wp, T_arg, fl, counters=c)
            else:
                gs.ffc(wp, T_arg, fl, counters=c)
            cq = dict(zip(mrv.COUNTER_NAMES, (int(x) for x in c.cpu().tolist())))
            ts = []
            for _ in range(2):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                if q == "motval":
                    gs.motval(wp, T_arg, fl, out=my_valid, stream=stream)
                else:
                    gs.ffc(wp, T_arg, fl, out=my_key, stream=stream)
                e1.record(stream)
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            ms_q = D.max_over_ranks(sum(ts) / len(ts), world, dev)
            o = cost_ops(cq, sc, q)
            nee[q] = {"kernel_ms": ms_q, "states_evaluated": cq["states"], "ops_per_launch": o,
                      "achieved": o / (ms_q / 1e3) / 1e12, "frac": o / (ms_q / 1e3) / 1e12 / peak,
                      "frac_survey_weights": cost_ops(cq, sc, q, SURVEY_COST) / (ms_q / 1e3) / 1e12 / peak,
                      "evaluated_robot_states_per_s": cq["states"] * n * world / (ms_q / 1e3)}
        roof["no_early_exit"] = nee

    # end to end through the public API with host buffers
    e2e = None
    if not a.no_e2e:
        out_v = torch.empty(world * per, dtype=torch.uint8).pin_memory()
        out_k = torch.empty(world * per, dtype=torch.int32).pin_memory()
        ee = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
        h2d = wp_host.numel() * 4 + (0 if T_local_host is None else T_local_host.numel() * 4)
        d2h = (world * per if "motval" in queries else 0) + (4 * world * per if "ffc" in queries else 0)
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        T_host_arg = T_arg if T_local_host is None else T_local_host.pin_memory()
        # one GPU: the results land in pinned host memory straight from the call (each chunk's
        # results copied back as its kernel ends); several: device outputs, the all-gather,
        # then one copy to the host
        host_out = world == 1
        ov = (out_v if host_out else my_valid) if "motval" in queries else None
        ok = (out_k if host_out else my_key) if "ffc" in queries else None
        for _ in range(2):   # untimed: the first call allocates the staging buffers and streams
            gs.run_host(wp_host, T_host_arg, flags, ov, 0, ok, stream=stream)
        torch.cuda.synchronize()
        for k in range(K):
            flush.zero_()
            ee[k][0].record(stream)
            # the end-to-end call: host inputs, chunked H2D overlapped with the kernels
            gs.run_host(wp_host, T_host_arg, flags, ov, 0, ok, stream=stream)
            if not host_out:
                if "motval" in queries:
                    D.gather_inplace(valid_all, per, rank, world)
                    out_v.copy_(valid_all, non_blocking=True)
                if "ffc" in queries:
                    D.gather_inplace(key_all, per, rank, world)
                    out_k.copy_(key_all, non_blocking=True)
            ee[k][1].record(stream)
        torch.cuda.synchronize()
        if host_out:   # the end-to-end results are the device path's
            assert "motval" not in queries or torch.equal(out_v, valid_all.cpu()), "end-to-end MotVal results differ"
            assert "ffc" not in queries or torch.equal(out_k, key_all.cpu()), "end-to-end FFC results differ"
        e_ms = D.max_over_ranks(sum(e[0].elapsed_time(e[1]) for e in ee), world, dev) / K
        e2e = {"value": robot_states_step / (e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": e_ms,
               "path": "mrv_run_host_batch: pinned host waypoints, chunks growing x4 from min(32768, max(M/8, 8192)) up to "
                       "1048576 motions, H2D "
                       "of chunk i+1 overlapped with the kernels of chunk i (each query's chunks alternating between two compute "
                       "streams); results written to pinned host memory chunk by chunk (one GPU) or gathered "
                       "and copied back (several)"}

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        cpu = time_oracle(sc, mo, queries, a.cpu_seconds)

    if rank == 0:
        vv = valid_all[:M].float().mean().item() if "motval" in queries else None
        kk = key_all[:M]
        cf = (kk == -1).float().mean().item() if "ffc" in queries else None
        deciles = None
        if "ffc" in queries:   # first-conflict time t* / T in deciles, conflicting motions only
            keys = kk.cpu().numpy().view(np.uint32)
            hit = keys != 0xFFFFFFFF
            tstar = (keys[hit] // max(1, sc.n_pairs)).astype(np.float64)
            frac_t = tstar / np.maximum(T_all[:M][hit].astype(np.float64) - 1.0, 1.0)
            deciles = np.histogram(np.clip(frac_t, 0, 1), bins=10, range=(0, 1))[0].tolist()
        # per-query rates first: the nominal value counts every state of every motion, but
        # MotVal's early exit evaluates only a fraction of them
        rates = {"motval_robot_states_per_s": (comp_states * n / (alone["motval"] / 1e3)
                                               if "motval" in alone else None),
                 "ffc_robot_states_per_s": (comp_states * n / (alone["ffc"] / 1e3)
                                            if "ffc" in alone else None),
                 "motval_evaluated_robot_states_per_s": (counts["motval"]["states"] * n * world / (alone["motval"] / 1e3)
                                                         if "motval" in alone else None),
                 "ffc_evaluated_robot_states_per_s": (counts["ffc"]["states"] * n * world / (alone["ffc"] / 1e3)
                                                      if "ffc" in alone else None),
                 "motions_per_s": M / (ms_per_step / 1e3),
                 "note": "each query's kernel timed alone; 'evaluated' counts only the states a query computed "
                         "before its early exit (work counters)"}
        line = {
            "metric": BJ_METRIC, "value": value, "unit": UNIT, "rates": rates, "n_gpus": world, "steps": K, "warmup": max(3, a.warmup),
            "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic (seeded generators, paper_2604_23960_b200/gen.py)",
            "config": config_dict(a, sc, mo, queries, world),
            "breakdown": {"motval_ms": mv_avg, "ffc_ms": ffc_avg, "per_rank_step_ms": per_rank_ms,
                          "per_rank_kernel_ms": per_rank_kernel_ms, "allgather_ms": allgather_ms,
                          "step_ms_min": step_sorted[0], "step_ms_median": step_sorted[len(step_sorted) // 2],
                          "queries_concurrent": concurrent,
                          "motval_alone_ms": alone.get("motval"), "ffc_alone_ms": alone.get("ffc"),
                          "motval_robot_states_per_s": (comp_states * n / (alone["motval"] / 1e3)
                                                        if "motval" in alone else None),
                          "ffc_robot_states_per_s": (comp_states * n / (alone["ffc"] / 1e3) if "ffc" in alone else None),
                          # states each query actually evaluated before its early exit (work counters,
                          # this rank's shard; whole job under equal shards)
                          "motval_evaluated_states_per_s": (counts["motval"]["states"] * world / (alone["motval"] / 1e3)
                                                            if "motval" in alone else None),
                          "ffc_prefix_states_per_s": (counts["ffc"]["states"] * world / (alone["ffc"] / 1e3)
                                                      if "ffc" in alone else None),
                          "composite_states_per_s": comp_states * len(queries) / (ms_per_step / 1e3),
                          "motions_per_s": M / (ms_per_step / 1e3), "valid_frac": vv, "conflict_free_frac": cf,
                          "ffc_first_conflict_deciles": deciles,
                          # the state stream (BJ.north_star: achieved HBM GB/s): every launch reads
                          # each motion's waypoint block once (+ per-motion T); the path is ALU-bound,
                          # so this is a small fraction of HBM bandwidth by design
                          "state_stream": {
                              "bytes_per_launch": state_bytes,
                              "motval_gbs": (state_bytes / (alone["motval"] / 1e3) / 1e9 if "motval" in alone else None),
                              "ffc_gbs": (state_bytes / (alone["ffc"] / 1e3) / 1e9 if "ffc" in alone else None),
                              "hbm_peak_gbs": peaks.get("hbm_gbs"), "peak_source": peak_src},
                          "wall_s_timed_loop": wall},
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": K * len(queries),
            "clocks": clk_s, "peaks": peak_src, "paper_context": PAPER_CONTEXT,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


# ------------------------------------------------------------------ PP-ST-RRT variant (pp5)
def main_pp(a, rank, world, local):
    """One step = the PP-ST-RRT MotVal variant's whole path: build the partner table from
    the fixed paths (mrv_pp_build_table), then validate every candidate against it
    (mrv_pp_motval_batch), then (N > 1) the all-gather of the per-candidate flags.
    Candidates are sharded by index; the table is rebuilt on every rank.  Beside it the
    same candidates through the replicated-waypoint MRV_FOCUS path (every candidate
    carries the partners' waypoints and re-runs their FK), timed alone."""
    import torch

    from paper_2604_23960_b200 import dist as D
    from paper_2604_23960_b200 import gen, mrv
    dev = torch.device("cuda", local)
    sc, cand, pp = load_workload(a)
    paths, t0_all = pp["paths"], pp["t0"]
    H, focus, partners = gen.PP_HORIZON, gen.PP_FOCUS, gen.PP_PARTNERS
    M = cand.M
    lo, hi, per = D.shard(M, rank, world)
    cw_host = D.pad_rows(torch.from_numpy(np.ascontiguousarray(cand.waypoints[lo:hi])), per).pin_memory()
    t0_host = D.pad_rows(torch.from_numpy(np.ascontiguousarray(t0_all[lo:hi])), per).pin_memory()
    pw_host = torch.from_numpy(np.ascontiguousarray(paths.waypoints)).pin_memory()
    pT_host = torch.from_numpy(np.ascontiguousarray(paths.robot_timesteps)).pin_memory()
    cw, t0, pw, pT = (x.to(dev) for x in (cw_host, t0_host, pw_host, pT_host))
    T = int(cand.fixed_timesteps)
    gs = mrv.Scene(sc, device=local)
    flags = mrv.CHECK_ENV
    valid_all = torch.empty(world * per, dtype=torch.uint8, device=dev)
    my_valid = valid_all[rank * per:(rank + 1) * per]
    nb = gs.pp_table(pw, pT, partners, H).numel()
    table = torch.empty(nb, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()

    def build_table():
        b = gs._batch(pw, pT)
        mrv._check(mrv.lib().mrv_pp_build_table(gs._h, mrv.C.byref(b), gs._mask(partners), H, table.data_ptr(),
                                                stream.cuda_stream), "mrv_pp_build_table")

    def step(ev=None):
        build_table()
        if ev is not None:
            ev[0].record(stream)
        gs.pp_motval(cw, T, t0, focus, partners, table, H, flags, out=my_valid, stream=stream)
        if ev is not None:
            ev[1].record(stream)
        if world > 1:
            D.gather_inplace(valid_all, per, rank, world)

    for _ in range(max(3, a.warmup)):
        step()
    torch.cuda.synchronize()
    cnt = torch.zeros(mrv.NUM_COUNTERS, dtype=torch.int64, device=dev)
    gs.pp_motval(cw, T, t0, focus, partners, table, H, flags, counters=cnt)
    counts = dict(zip(mrv.COUNTER_NAMES, (int(x) for x in cnt.cpu().tolist())))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    K = a.steps
    ev = [tuple(torch.cuda.Event(enable_timing=True) for _ in range(4)) for _ in range(K)]
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    with Clocks(local) as clk:
        for k in range(K):
            flush.zero_()
            ev[k][0].record(stream)
            step(ev[k][1:3])
            ev[k][3].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    step_ms = [e[0].elapsed_time(e[3]) for e in ev]
    table_ms = D.max_over_ranks(sum(e[0].elapsed_time(e[1]) for e in ev) / K, world, dev)
    kern_ms = D.max_over_ranks(sum(e[1].elapsed_time(e[2]) for e in ev) / K, world, dev)
    ms_per_step = D.max_over_ranks(sum(step_ms), world, dev) / K

    # the replicated-waypoint MRV_FOCUS path on the same candidates: each motion carries all
    # four arms, the partners' rows = their path knots nearest the window's ends (a cost
    # comparison: a straight segment between those knots, not the piecewise path)
    Kp = paths.K
    kk0 = np.rint(t0_all[lo:hi].astype(np.float64) * (Kp - 1) / (H - 1)).astype(np.int64)
    kk1 = np.rint((t0_all[lo:hi] + T - 1).astype(np.float64) * (Kp - 1) / (H - 1)).astype(np.int64)
    rep = np.empty((hi - lo, sc.n_robots, 2, 7), np.float32)
    rep[:, focus] = cand.waypoints[lo:hi, 0]
    for r in partners:
        rep[:, r, 0] = paths.waypoints[0, r, kk0]
        rep[:, r, 1] = paths.waypoints[0, r, kk1]
    rep_d = D.pad_rows(torch.from_numpy(rep), per).to(dev)
    del rep
    rep_out = torch.empty(per, dtype=torch.uint8, device=dev)
    alone = {}
    for name in ("pp", "replicated"):
        ts = []
        for _ in range(3):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            if name == "pp":
                gs.pp_motval(cw, T, t0, focus, partners, table, H, flags, out=my_valid, stream=stream)
            else:
                gs.motval(rep_d, T, flags, out=rep_out, stream=stream, focus=focus, partners=partners)
            e1.record(stream)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        alone[name] = D.max_over_ranks(sum(ts) / len(ts), world, dev)
    c_rep = torch.zeros(mrv.NUM_COUNTERS, dtype=torch.int64, device=dev)
    gs.motval(rep_d, T, flags, out=rep_out, counters=c_rep, focus=focus, partners=partners)
    c_rep = dict(zip(mrv.COUNTER_NAMES, (int(x) for x in c_rep.cpu().tolist())))
    del rep_d

    n = sc.n_robots   # robots whose geometry each candidate state checks: the focus + 3 partners
    comp_states = M * T
    value = comp_states * n / (ms_per_step / 1e3)
    peaks, peak_src = measured_peaks()
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    clk_s = clk.summary()
    f_max = float(clk_s["sm_max_mhz"] or peaks.get("sm_max_mhz", 1965.0))
    peak = sms * 128 * f_max * 1e6 / 1e12
    ops = cost_ops(counts, sc, "motval")
    achieved = ops / (alone["pp"] / 1e3) / 1e12
    table_bytes = counts["table_bytes"]
    wp_bytes = int(cw_host.numel()) * 4 + int(t0_host.numel()) * 4
    roof = {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "Tlane-ops/s", "frac": achieved / peak,
            "traffic": None, "kernel": "mrv_query_kernel<motval> (PP table mode)", "kernel_ms": alone["pp"],
            "peak_source": f"{sms} SMs x 128 FP32 lanes x {f_max:.0f} MHz (NVML max SM clock)",
            "ops_per_launch": ops, "counters": counts,
            "frac_survey_weights": cost_ops(counts, sc, "motval", SURVEY_COST) / (alone["pp"] / 1e3) / 1e12 / peak}

    # end to end through the public API: host candidates / start times / fixed paths copied
    # in, table built, candidates validated, flags copied out -- every step
    out_v = torch.empty(world * per, dtype=torch.uint8).pin_memory()
    ee = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    torch.cuda.synchronize()
    for k in range(K):
        flush.zero_()
        ee[k][0].record(stream)
        cw.copy_(cw_host, non_blocking=True)
        t0.copy_(t0_host, non_blocking=True)
        pw.copy_(pw_host, non_blocking=True)
        pT.copy_(pT_host, non_blocking=True)
        step()
        out_v.copy_(valid_all, non_blocking=True)
        ee[k][1].record(stream)
    torch.cuda.synchronize()
    e_ms = D.max_over_ranks(sum(e[0].elapsed_time(e[1]) for e in ee), world, dev) / K
    h2d = wp_bytes + int(pw_host.numel()) * 4 + int(pT_host.numel()) * 4
    e2e = {"value": comp_states * n / (e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": h2d,
           "d2h_bytes_per_step": int(world * per), "ms_per_step": e_ms,
           "path": "pinned host candidates + start times + fixed paths -> device (torch copies), mrv_pp_build_table, "
                   "mrv_pp_motval_batch, flags -> host"}
    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        cpu = time_oracle(sc, cand, QUERIES["pp5"], a.cpu_seconds, pp=pp)
    if rank == 0:
        vv = valid_all[:M].float().mean().item()
        line = {
            "metric": BJ_METRIC, "value": value, "unit": UNIT,
            "rates": {"pp_robot_states_per_s": comp_states * n / (alone["pp"] / 1e3),
                      "pp_evaluated_robot_states_per_s": counts["states"] * n * world / (alone["pp"] / 1e3),
                      "replicated_focus_robot_states_per_s": comp_states * n / (alone["replicated"] / 1e3),
                      "candidates_per_s": M / (ms_per_step / 1e3),
                      "note": "robot-states = candidate states x 4 (the focus arm + the 3 partner arms it is checked "
                              "against); kernels timed alone"},
            "n_gpus": world, "steps": K, "warmup": max(3, a.warmup), "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded generators, paper_2604_23960_b200/gen.py make_pp)",
            "config": config_dict(a, sc, cand, QUERIES["pp5"], world),
            "breakdown": {"table_build_ms": table_ms, "pp_kernel_ms": kern_ms, "pp_alone_ms": alone["pp"],
                          "replicated_focus_alone_ms": alone["replicated"],
                          "speedup_vs_replicated": alone["replicated"] / alone["pp"],
                          "replicated_counters": c_rep, "valid_frac": vv,
                          "table": {"bytes": nb, "rows": H, "bytes_read_per_launch": table_bytes,
                                    "read_gbs": table_bytes / (alone["pp"] / 1e3) / 1e9,
                                    "bytes_per_evaluated_state": table_bytes / max(1, counts["states"])},
                          "state_stream": {"bytes_per_launch": wp_bytes,
                                           "gbs": wp_bytes / (alone["pp"] / 1e3) / 1e9,
                                           "hbm_peak_gbs": peaks.get("hbm_gbs"), "peak_source": peak_src},
                          "per_rank_step_ms": D.all_ranks(sum(step_ms) / K, world, dev)},
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": 2 * K, "clocks": clk_s,
            "peaks": peak_src, "paper_context": PAPER_CONTEXT,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
