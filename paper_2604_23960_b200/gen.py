"""Seeded synthetic input generators for the five BASELINE.json configs.

This module is the ONLY code shared by the CUDA path (bench, tests) and the
oracle (tests).  It builds input tables -- robot sphere sets, joint origins,
obstacles, waypoints, timestep counts -- and holds none of the method's
arithmetic: no forward kinematics, no interpolation, no collision test.
Recipes follow SURVEY.md §8(d) (table "Generator") and the readings
c.4/c.5/c.7/c.8/c.9/c.23/c.24/c.25 listed in DESIGN.md.

Endpoint validity (reading c.25) is NOT decided here: the accepted candidate
indices are read from ``pools/*.npz``, which ``oracle/make_pools.py`` (a
committed script that calls only ``oracle/``) wrote.  The candidate streams
themselves are generated here, block by block, so the file only stores indices.

Determinism: every random draw comes from ``numpy.random.Generator(PCG64)``
seeded by ``SeedSequence([cfg_seed, purpose, block])``; motion ``m`` depends only
on its block, so a prefix of ``M`` motions is identical for every ``M``.
"""
from __future__ import annotations

import dataclasses
import hashlib
import os
from typing import List, Optional

import numpy as np

CHAIN, SE2, SE3 = 0, 1, 2
REVOLUTE, PRISMATIC = 0, 1

BLOCK = 65536           # candidates / motions per independently seeded block
POOL_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "pools")

# purposes (second SeedSequence word)
_P_SCENE, _P_OBST, _P_CAND, _P_MOT, _P_PAIR, _P_FORCE = 1, 2, 3, 4, 5, 6


@dataclasses.dataclass
class Robot:
    """One robot in ABI form (include/mrv.h, mrv_robot_desc)."""
    kind: int
    dof: int
    sphere_link: np.ndarray                   # [ns] int32
    sphere: np.ndarray                        # [ns][4] float32 (ox, oy, oz, r)
    joint_origin: Optional[np.ndarray] = None  # chain: [dof][12] float32 row-major 3x4
    joint_type: Optional[np.ndarray] = None    # chain: [dof] int32
    base: Optional[np.ndarray] = None          # chain: [12] float32 or None (identity)
    self_pairs: Optional[np.ndarray] = None    # chain: [n][2] int32 link pairs for self-collision (MRV_CHECK_SELF)

    @property
    def n_spheres(self) -> int:
        return int(self.sphere.shape[0])


@dataclasses.dataclass
class Scene:
    robots: List[Robot]
    obs_spheres: np.ndarray   # [n][4] float32 (x, y, z, R)
    obs_boxes: np.ndarray     # [n][6] float32 (lo xyz, hi xyz)

    @property
    def n_robots(self) -> int:
        return len(self.robots)

    @property
    def n_pairs(self) -> int:
        n = self.n_robots
        return n * (n - 1) // 2

    @property
    def total_spheres(self) -> int:
        return sum(r.n_spheres for r in self.robots)


@dataclasses.dataclass
class Motions:
    waypoints: np.ndarray                  # [M][n_robots][K][S] float32
    n_timesteps: Optional[np.ndarray]      # [M] int32, or None -> fixed_timesteps
    fixed_timesteps: int = 0
    robot_timesteps: Optional[np.ndarray] = None   # [M][n_robots] int32 per-robot lengths (stay at goal)

    @property
    def M(self) -> int:
        return int(self.waypoints.shape[0])

    @property
    def K(self) -> int:
        return int(self.waypoints.shape[2])

    @property
    def S(self) -> int:
        return int(self.waypoints.shape[3])

    def T_array(self) -> np.ndarray:
        if self.robot_timesteps is not None:
            return self.robot_timesteps.max(axis=1).astype(np.int32)
        if self.n_timesteps is not None:
            return self.n_timesteps
        return np.full(self.M, self.fixed_timesteps, dtype=np.int32)

    def total_states(self) -> int:
        return int(self.T_array().astype(np.int64).sum())

    def subset(self, idx) -> "Motions":
        idx = np.asarray(idx)
        nt = None if self.n_timesteps is None else np.ascontiguousarray(self.n_timesteps[idx])
        rt = None if self.robot_timesteps is None else np.ascontiguousarray(self.robot_timesteps[idx])
        return Motions(np.ascontiguousarray(self.waypoints[idx]), nt, self.fixed_timesteps, rt)


def _rng(*words) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence(list(words))))


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float32))


def _affine(rot3x3, trans3) -> np.ndarray:
    """Pack a rotation and translation into the ABI's row-major 3x4 (12 floats)."""
    m = np.zeros((3, 4), dtype=np.float64)
    m[:, :3] = rot3x3
    m[:, 3] = trans3
    return m.reshape(12)


# --------------------------------------------------------------------------
# scenes
# --------------------------------------------------------------------------

def arm_robots(seed: int = 1002) -> List[Robot]:
    """cfg2's four 7-DOF revolute arms (BASELINE.json configs[1]).

    Standard DH with d_j = 0, a_j ~ U[0.1, 0.4] m, alpha_j in {+-pi/2}; converted
    to the ABI chain T_j = T_{j-1} O_j Rz(q_j) (reading c.9): O_1 = I (the base is
    the separate ``base`` field), O_j = Tx(a_{j-1}) Rx(alpha_{j-1}).  With
    alpha = +-pi/2 the rotation entries are exactly 0 / +-1.  8 spheres per link at
    ((k+0.5)/8) * (a_j, 0, 0), r ~ U[0.03, 0.08].  Bases at (+-0.6, +-0.6, 0) with
    yaw facing the centre.
    """
    rng = _rng(seed, _P_SCENE)
    robots = []
    for (bx, by) in [(0.6, 0.6), (-0.6, 0.6), (-0.6, -0.6), (0.6, -0.6)]:
        a = rng.uniform(0.1, 0.4, size=7)
        sgn = rng.choice([-1.0, 1.0], size=7)
        radii = rng.uniform(0.03, 0.08, size=56)
        origins = []
        for j in range(7):
            if j == 0:
                origins.append(_affine(np.eye(3), np.zeros(3)))
            else:
                s = sgn[j - 1]
                rx = np.array([[1.0, 0.0, 0.0], [0.0, 0.0, -s], [0.0, s, 0.0]])
                origins.append(_affine(rx, np.array([a[j - 1], 0.0, 0.0])))
        yaw = np.arctan2(-by, -bx)
        c, s = np.cos(yaw), np.sin(yaw)
        base = _affine(np.array([[c, -s, 0.0], [s, c, 0.0], [0.0, 0.0, 1.0]]), np.array([bx, by, 0.0]))
        sph, link = [], []
        for j in range(7):
            for k in range(8):
                sph.append([(k + 0.5) / 8.0 * a[j], 0.0, 0.0, radii[8 * j + k]])
                link.append(j)
        # self-collision pairs: links at least 3 apart (SPEC.md:23 excludes adjacent links; in these
        # synthetic arms links two apart always overlap through the shortest middle links)
        pairs = np.array([(i, j) for i in range(7) for j in range(i + 3, 7)], np.int32)
        robots.append(Robot(kind=CHAIN, dof=7, sphere_link=np.asarray(link, np.int32), sphere=_f32(sph),
                            joint_origin=_f32(origins), joint_type=np.zeros(7, np.int32), base=_f32(base),
                            self_pairs=pairs))
    return robots


def arm_boxes(seed: int = 1002) -> np.ndarray:
    """cfg2's 32 AABBs: centre U([-1.8,1.8]^2 x [0.1,1.6]), half-extents U[0.05,0.25]^3,
    redrawn while the centre is within 0.45 m (xy) of a base."""
    rng = _rng(seed, _P_OBST)
    bases = np.array([(0.6, 0.6), (-0.6, 0.6), (-0.6, -0.6), (0.6, -0.6)])
    boxes = []
    while len(boxes) < 32:
        c = np.array([rng.uniform(-1.8, 1.8), rng.uniform(-1.8, 1.8), rng.uniform(0.1, 1.6)])
        h = rng.uniform(0.05, 0.25, size=3)
        if np.min(np.hypot(bases[:, 0] - c[0], bases[:, 1] - c[1])) < 0.45:
            continue
        boxes.append(np.concatenate([c - h, c + h]))
    return _f32(boxes)


def body_robots(seed: int, n: int, n_spheres: int = 20) -> List[Robot]:
    """cfg3-style SE(3) bodies: spheres r ~ U[0.05, 0.2], centre uniform in the ball of
    radius 0.5 - r (reading c.23: ||o|| + r <= 0.5)."""
    rng = _rng(seed, _P_SCENE, 3)
    robots = []
    for _ in range(n):
        sph = []
        for _k in range(n_spheres):
            r = rng.uniform(0.05, 0.2)
            while True:
                o = rng.uniform(-1.0, 1.0, size=3)
                if o @ o <= 1.0:
                    break
            o = o * (0.5 - r)
            sph.append([o[0], o[1], o[2], r])
        robots.append(Robot(kind=SE3, dof=7, sphere_link=np.zeros(n_spheres, np.int32), sphere=_f32(sph)))
    return robots


def scene_cfg1(seed: int = 1001) -> Scene:
    """cfg1: 2 SE(2) bodies x 4 discs (r ~ U[0.05,0.15], offset rho = 0.3 sqrt(U),
    phi ~ U[0, 2pi), z = 0) and 16 obstacle discs (R ~ U[0.1,0.3], centres U([0,4]^2))."""
    rng = _rng(seed, _P_SCENE)
    robots = []
    for _ in range(2):
        r = rng.uniform(0.05, 0.15, size=4)
        rho = 0.3 * np.sqrt(rng.uniform(size=4))
        phi = rng.uniform(0.0, 2 * np.pi, size=4)
        sph = np.stack([rho * np.cos(phi), rho * np.sin(phi), np.zeros(4), r], axis=1)
        robots.append(Robot(kind=SE2, dof=3, sphere_link=np.zeros(4, np.int32), sphere=_f32(sph)))
    ro = _rng(seed, _P_OBST)
    obs = np.stack([ro.uniform(0, 4, 16), ro.uniform(0, 4, 16), np.zeros(16), ro.uniform(0.1, 0.3, 16)], axis=1)
    return Scene(robots, _f32(obs), np.zeros((0, 6), np.float32))


def scene_cfg2(seed: int = 1002) -> Scene:
    return Scene(arm_robots(seed), np.zeros((0, 4), np.float32), arm_boxes(seed))


def scene_cfg3(seed: int = 1003) -> Scene:
    """cfg3: 8 SE(3) bodies x 20 spheres; 100 sphere obstacles (centre U[0,10]^3,
    R ~ U[0.1,0.5]) + 100 AABBs (centre U[0,10]^3, half-extents U[0.1,0.5]^3)."""
    robots = body_robots(seed, 8)
    ro = _rng(seed, _P_OBST)
    sph = np.concatenate([ro.uniform(0, 10, (100, 3)), ro.uniform(0.1, 0.5, (100, 1))], axis=1)
    c = ro.uniform(0, 10, (100, 3))
    h = ro.uniform(0.1, 0.5, (100, 3))
    return Scene(robots, _f32(sph), _f32(np.concatenate([c - h, c + h], axis=1)))


def scene_cfg4(seed: int = 1004) -> Scene:
    """cfg4: robots 0-3 = the cfg2 arms (same parameters), 4-11 = cfg3-style bodies; no obstacles."""
    return Scene(arm_robots(1002) + body_robots(seed, 8), np.zeros((0, 4), np.float32),
                 np.zeros((0, 6), np.float32))


# --------------------------------------------------------------------------
# candidate endpoint streams (accepted subsets come from pools/*.npz)
# --------------------------------------------------------------------------

def _shoemake(rng, n) -> np.ndarray:
    """Uniform unit quaternions (Shoemake), layout (qw, qx, qy, qz)."""
    u1, u2, u3 = rng.uniform(size=n), rng.uniform(size=n), rng.uniform(size=n)
    a, b = np.sqrt(1.0 - u1), np.sqrt(u1)
    return np.stack([b * np.cos(2 * np.pi * u3), a * np.sin(2 * np.pi * u2),
                     a * np.cos(2 * np.pi * u2), b * np.sin(2 * np.pi * u3)], axis=1)


def candidate_block(stream: str, block: int) -> np.ndarray:
    """Block ``block`` of a candidate composite-state stream, [BLOCK][n_robots][7] float32.

    'arm' (seeds 1002/1005): 4 arms, joints U[-2.9, 2.9]^7.
    'body' (seed 1003): 8 bodies, position U[0.5, 9.5]^3 + Shoemake quaternion.
    """
    name, seed = stream.split(":")
    seed = int(seed)
    rng = _rng(seed, _P_CAND, block)
    if name == "arm":
        return _f32(rng.uniform(-2.9, 2.9, size=(BLOCK, 4, 7)))
    if name == "body":
        pos = rng.uniform(0.5, 9.5, size=(BLOCK * 8, 3))
        q = _shoemake(rng, BLOCK * 8)
        return _f32(np.concatenate([pos, q], axis=1).reshape(BLOCK, 8, 7))
    raise ValueError(stream)


def candidates(stream: str, idx: np.ndarray) -> np.ndarray:
    idx = np.asarray(idx, dtype=np.int64)
    out = None
    for b in np.unique(idx // BLOCK):
        blk = candidate_block(stream, int(b))
        sel = idx // BLOCK == b
        if out is None:
            out = np.empty((idx.size,) + blk.shape[1:], np.float32)
        out[sel] = blk[idx[sel] % BLOCK]
    return out


POOLS = {  # pool name -> (candidate stream, scene builder used for acceptance, accepted count)
    "cfg2": ("arm:1002", "cfg2", 2 * 4096),
    "cfg3": ("body:1003", "cfg3", 2 * 65536),
    "cfg5": ("arm:1005", "cfg2", 65536),
}


def pool_path(name: str) -> str:
    return os.path.join(POOL_DIR, f"{name}_accepted.npz")


def load_pool(name: str, count: Optional[int] = None) -> np.ndarray:
    """First ``count`` accepted candidate composite states of a pool, [count][n][7] float32."""
    p = pool_path(name)
    if not os.path.exists(p):
        raise FileNotFoundError(f"{p} missing: run `python oracle/make_pools.py {name}` (test infrastructure)")
    acc = np.load(p)["accepted"].astype(np.int64)
    if count is not None:
        if count > acc.size:
            raise ValueError(f"pool {name} has {acc.size} accepted states, {count} requested")
        acc = acc[:count]
    return candidates(POOLS[name][0], acc)


# --------------------------------------------------------------------------
# motions
# --------------------------------------------------------------------------

def _align_quats(wp: np.ndarray) -> None:
    """ABI contract (reading c.8): consecutive SE(3) knots satisfy q_{k+1} . q_k >= 0.
    wp: [..., K, 7] with quaternion in [3:7]; flips signs in place (a sign flip
    leaves the rotation unchanged)."""
    for k in range(1, wp.shape[-2]):
        d = np.sum(wp[..., k, 3:7].astype(np.float64) * wp[..., k - 1, 3:7], axis=-1)
        wp[..., k, 3:7] = np.where((d < 0)[..., None], -wp[..., k, 3:7], wp[..., k, 3:7])


def motions_cfg1(M: int = 256, seed: int = 1001) -> Motions:
    """cfg1: K=2, (x,y) ~ U([0,4]^2), theta_s ~ U[-pi,pi), goal unwrapped into
    [theta_s - pi, theta_s + pi) (reading c.7); T = 64; no endpoint rejection."""
    rng = _rng(seed, _P_MOT, 0)
    xy = rng.uniform(0, 4, size=(M, 2, 2, 2))
    th = rng.uniform(-np.pi, np.pi, size=(M, 2, 2))
    th[:, :, 1] = th[:, :, 0] + np.mod(th[:, :, 1] - th[:, :, 0] + np.pi, 2 * np.pi) - np.pi
    wp = np.concatenate([xy, th[..., None]], axis=-1)
    return Motions(_f32(wp), None, 64)


def resolution_T(start: np.ndarray, goal: np.ndarray, res: float) -> np.ndarray:
    """Reading c.5: T = 1 + ceil(max |dq| / res), in fp64 on the fp32 endpoints."""
    d = np.abs(goal.astype(np.float64) - start.astype(np.float64)).reshape(start.shape[0], -1).max(axis=1)
    return (1 + np.ceil(d / res)).astype(np.int32)


def motions_cfg2(M: int = 4096) -> Motions:
    """cfg2: K=2, endpoints = consecutive accepted pool states, T per reading c.5 (res 0.05 rad)."""
    pool = load_pool("cfg2", 2 * M)
    s, g = pool[0::2], pool[1::2]
    wp = np.stack([s, g], axis=2)  # [M][4][2][7]
    return Motions(_f32(wp), resolution_T(s, g, 0.05), 0)


def motions_cfg3(M: int = 65536) -> Motions:
    """cfg3: K=2, endpoints = consecutive accepted pool states, quaternions sign-aligned, T=96."""
    pool = load_pool("cfg3", 2 * M)
    wp = np.stack([pool[0::2], pool[1::2]], axis=2).copy()  # [M][8][2][7]
    _align_quats(wp)
    return Motions(_f32(wp), None, 96)


def motions_cfg5(M: int = 1 << 20, pool_size: int = 65536) -> Motions:
    """cfg5: endpoints paired at random (distinct) from a pool of 65,536 accepted states; T=128."""
    pool = load_pool("cfg5", pool_size)
    wp = np.empty((M, 4, 2, 7), np.float32)
    for b in range((M + BLOCK - 1) // BLOCK):
        lo, hi = b * BLOCK, min(M, (b + 1) * BLOCK)
        rng = _rng(1005, _P_PAIR, b)
        i = rng.integers(0, pool_size, size=BLOCK)
        j = (i + rng.integers(1, pool_size, size=BLOCK)) % pool_size
        wp[lo:hi, :, 0] = pool[i[: hi - lo]]
        wp[lo:hi, :, 1] = pool[j[: hi - lo]]
    return Motions(wp, None, 128)


# cfg4 tuning knobs (stated in DESIGN.md)
CFG4_ARM_HOME = np.array([2.6, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0])
CFG4_ARM_STEP = 0.25
CFG4_BODY_LO = np.array([-6.0, -6.0, 0.0])
CFG4_BODY_HI = np.array([6.0, 6.0, 3.0])
CFG4_BODY_STEP = 0.75
CFG4_FORCE_FRAC = 0.30


def motions_cfg4(M: int = 16384, seed: int = 1004) -> Motions:
    """cfg4: K=10 knots, T=1000 (knots at t = 111k).  Arms: bounded random walk from an
    outward-facing home posture (step U[-s, s] per DOF, clipped +-2.9).  Bodies:
    bounded random walk of positions from U(box) (step U[-0.75, 0.75] m per axis,
    clipped to the box), Shoemake orientations per knot, sign-aligned.  Reading c.24: in ~30%
    of path sets one seeded body pair (a, b) gets waypoint k of a := waypoint k of
    b (identical pose) at a seeded knot k in 1..8 -> a definite hit at t = 111k."""
    K = 10
    wp = np.empty((M, 12, K, 7), np.float32)
    for blk in range((M + BLOCK - 1) // BLOCK):
        lo, hi = blk * BLOCK, min(M, (blk + 1) * BLOCK)
        n = hi - lo
        rng = _rng(seed, _P_MOT, blk)
        steps = rng.uniform(-CFG4_ARM_STEP, CFG4_ARM_STEP, size=(n, 4, K, 7))
        steps[:, :, 0] = 0.0
        q = np.empty((n, 4, K, 7))
        q[:, :, 0] = CFG4_ARM_HOME
        for k in range(1, K):
            q[:, :, k] = np.clip(q[:, :, k - 1] + steps[:, :, k], -2.9, 2.9)
        pos = np.empty((n, 8, K, 3))
        pos[:, :, 0] = rng.uniform(CFG4_BODY_LO, CFG4_BODY_HI, size=(n, 8, 3))
        bsteps = rng.uniform(-CFG4_BODY_STEP, CFG4_BODY_STEP, size=(n, 8, K, 3))
        for k in range(1, K):
            pos[:, :, k] = np.clip(pos[:, :, k - 1] + bsteps[:, :, k], CFG4_BODY_LO, CFG4_BODY_HI)
        quat = _shoemake(rng, n * 8 * K).reshape(n, 8, K, 4)
        body = np.concatenate([pos, quat], axis=-1)
        rf = _rng(seed, _P_FORCE, blk)
        force = rf.uniform(size=n) < CFG4_FORCE_FRAC
        a = rf.integers(0, 8, size=n)
        b = (a + rf.integers(1, 8, size=n)) % 8
        kk = rf.integers(1, 9, size=n)
        for m in np.nonzero(force)[0]:
            body[m, a[m], kk[m]] = body[m, b[m], kk[m]]
        body32 = _f32(body)
        _align_quats(body32)
        wp[lo:hi, :4] = _f32(q)
        wp[lo:hi, 4:] = body32
    return Motions(wp, None, 1000)


CONFIGS = {
    "cfg1": (scene_cfg1, motions_cfg1, 256),
    "cfg2": (scene_cfg2, motions_cfg2, 4096),
    "cfg3": (scene_cfg3, motions_cfg3, 65536),
    "cfg4": (scene_cfg4, motions_cfg4, 16384),
    "cfg5": (scene_cfg2, motions_cfg5, 1 << 20),
}


# --------------------------------------------------------------------------
# PP-ST-RRT MotVal variant workload: the cfg2/cfg5
# 4-arm scene; arms 0-2 (higher priority) follow fixed paths over PP_HORIZON absolute
# timesteps, the candidates are motions of arm 3 (the robot being planned) between pool
# states, each starting at a random absolute timestep (ST-RRT samples in space-time)
# --------------------------------------------------------------------------
PP_FOCUS, PP_PARTNERS = 3, (0, 1, 2)
PP_HORIZON, PP_KNOTS, PP_T, PP_STEP = 4096, 65, 128, 0.25


def pp_paths(seed: int = 1006) -> Motions:
    """The fixed paths: one motion [1][4][PP_KNOTS][7]; every arm starts at a seeded pool
    state and random-walks in joint space (step U[-0.25, 0.25] rad per knot and DOF, clipped
    to +-2.9); all paths span the horizon (per-robot lengths = PP_HORIZON)."""
    pool = load_pool("cfg5", 65536)
    rng = _rng(seed, _P_MOT, 0)
    q = np.empty((4, PP_KNOTS, 7))
    q[:, 0] = pool[int(rng.integers(0, 65536))]
    steps = rng.uniform(-PP_STEP, PP_STEP, size=(4, PP_KNOTS, 7))
    for k in range(1, PP_KNOTS):
        q[:, k] = np.clip(q[:, k - 1] + steps[:, k], -2.9, 2.9)
    return Motions(_f32(q[None]), None, 0, np.full((1, 4), PP_HORIZON, np.int32))


def pp_candidates(M: int = 1 << 20, seed: int = 1006):
    """(Motions [M][1][2][7] of arm PP_FOCUS between two random pool states, T = PP_T;
    t_start [M] int32 uniform in [0, PP_HORIZON - PP_T])."""
    pool = load_pool("cfg5", 65536)[:, PP_FOCUS]
    wp = np.empty((M, 1, 2, 7), np.float32)
    t0 = np.empty(M, np.int32)
    for b in range((M + BLOCK - 1) // BLOCK):
        lo, hi = b * BLOCK, min(M, (b + 1) * BLOCK)
        rng = _rng(seed, _P_PAIR, b)
        i = rng.integers(0, 65536, size=BLOCK)
        j = (i + rng.integers(1, 65536, size=BLOCK)) % 65536
        ts = rng.integers(0, PP_HORIZON - PP_T + 1, size=BLOCK)
        wp[lo:hi, 0, 0] = pool[i[: hi - lo]]
        wp[lo:hi, 0, 1] = pool[j[: hi - lo]]
        t0[lo:hi] = ts[: hi - lo]
    return Motions(wp, None, PP_T), t0


def make_pp(M: Optional[int] = None):
    """(Scene, fixed paths, candidates, t_start) of the PP-ST-RRT workload ("pp5")."""
    cand, t0 = pp_candidates(1 << 20 if M is None else M)
    return scene_cfg2(), pp_paths(), cand, t0


def make(cfg: str, M: Optional[int] = None):
    """(Scene, Motions) for a BASELINE.json config; ``M`` takes a prefix of the motions."""
    scene_fn, mot_fn, full = CONFIGS[cfg]
    return scene_fn(), mot_fn(full if M is None else min(M, full) if cfg != "cfg5" else M)


def digest(*arrays) -> str:
    """SHA-256 over the raw bytes of the given arrays (recorded in result records)."""
    h = hashlib.sha256()
    for a in arrays:
        if a is not None:
            h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def scene_digest(scene: Scene) -> str:
    parts = []
    for r in scene.robots:
        parts += [np.int32([r.kind, r.dof]), r.sphere_link, r.sphere, r.joint_origin, r.joint_type, r.base,
                  r.self_pairs]
    return digest(*parts, scene.obs_spheres, scene.obs_boxes)


# --------------------------------------------------------------------------
# Fig. 7-shaped arm teams: n arms in two facing rows ("Cage"-like,
# PAPER.md:552), random start/goal motions without endpoint rejection (the paper's
# "1000 randomly sampled motions")
# --------------------------------------------------------------------------

def scene_arm_team(n_arms: int, obstacles: bool = True, seed: int = 2001) -> Scene:
    """n_arms 7-DOF DH arms (cfg2's link/sphere recipe) in two facing rows 1.2 m apart,
    1.0 m spacing along x; 8 boxes per arm pair in the shared volume when obstacles."""
    rng = _rng(seed, _P_SCENE)
    per_row = (n_arms + 1) // 2
    robots = []
    for k in range(n_arms):
        row, col = k % 2, k // 2
        bx = (col - (per_row - 1) / 2.0) * 1.0
        by = -0.6 if row == 0 else 0.6
        a = rng.uniform(0.1, 0.4, size=7)
        sgn = rng.choice([-1.0, 1.0], size=7)
        radii = rng.uniform(0.03, 0.08, size=56)
        origins = [_affine(np.eye(3), np.zeros(3))]
        for j in range(1, 7):
            s = sgn[j - 1]
            origins.append(_affine(np.array([[1.0, 0.0, 0.0], [0.0, 0.0, -s], [0.0, s, 0.0]]),
                                   np.array([a[j - 1], 0.0, 0.0])))
        yaw = np.pi / 2 if row == 0 else -np.pi / 2
        c, s = np.cos(yaw), np.sin(yaw)
        base = _affine(np.array([[c, -s, 0.0], [s, c, 0.0], [0.0, 0.0, 1.0]]), np.array([bx, by, 0.0]))
        sph, link = [], []
        for j in range(7):
            for q in range(8):
                sph.append([(q + 0.5) / 8.0 * a[j], 0.0, 0.0, radii[8 * j + q]])
                link.append(j)
        pairs = np.array([(i, j) for i in range(7) for j in range(i + 3, 7)], np.int32)
        robots.append(Robot(kind=CHAIN, dof=7, sphere_link=np.asarray(link, np.int32), sphere=_f32(sph),
                            joint_origin=_f32(origins), joint_type=np.zeros(7, np.int32), base=_f32(base),
                            self_pairs=pairs))
    boxes = np.zeros((0, 6), np.float32)
    if obstacles:
        ro = _rng(seed, _P_OBST, n_arms)
        nb = 8 * per_row
        half_x = per_row * 0.5 + 0.5
        cen = np.stack([ro.uniform(-half_x, half_x, nb), ro.uniform(-1.4, 1.4, nb), ro.uniform(0.1, 1.6, nb)], 1)
        h = ro.uniform(0.05, 0.2, (nb, 3))
        boxes = _f32(np.concatenate([cen - h, cen + h], axis=1))
    return Scene(robots, np.zeros((0, 4), np.float32), boxes)


def motions_arm_team(n_arms: int, M: int = 1000, seed: int = 2001, res: float = 0.05) -> Motions:
    """Uniform joint-space endpoints in +-2.9 rad (no rejection), T per reading c.5."""
    rng = _rng(seed, _P_MOT, n_arms)
    q = _f32(rng.uniform(-2.9, 2.9, size=(M, n_arms, 2, 7)))
    return Motions(q, resolution_T(q[:, :, 0], q[:, :, 1], res), 0)
