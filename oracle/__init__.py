"""Python (ctypes) wrapper of the fp64 scalar CPU oracle in ``orc.c``.

TEST INFRASTRUCTURE ONLY: only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  It never imports the CUDA path (``paper_2604_23960_b200``) and the CUDA
path never imports it; the only shared module is the seeded generator
``paper_2604_23960_b200.gen`` that the *callers* use to build inputs.

Every function restates the plain definition of PAPER.md's queries (see
``orc.h`` for citations); DESIGN.md §3 lists the readings.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liborc.so")
NONE = 0xFFFFFFFF
BAND = 1e-4   # BASELINE.json north_star: states within 1e-4 m of contact are "ambiguous"


def build(force: bool = False) -> str:
    src = os.path.join(HERE, "orc.c")
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(
            os.path.getmtime(src), os.path.getmtime(os.path.join(HERE, "orc.h"))):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fPIC", "-shared", "-pthread",
                               "-Wall", "-o", LIB, src, "-lm"])
    return LIB


class _Robot(C.Structure):
    _fields_ = [("kind", C.c_int32), ("dof", C.c_int32), ("joint_origin", C.c_void_p),
                ("joint_type", C.c_void_p), ("base", C.c_void_p), ("n_spheres", C.c_int32),
                ("sphere_link", C.c_void_p), ("sphere", C.c_void_p), ("n_self_pairs", C.c_int32),
                ("self_pairs", C.c_void_p)]


class _Scene(C.Structure):
    _fields_ = [("n_robots", C.c_int32), ("robots", C.POINTER(_Robot)), ("n_obs_spheres", C.c_int32),
                ("obs_spheres", C.c_void_p), ("n_boxes", C.c_int32), ("boxes", C.c_void_p)]


class _Motions(C.Structure):
    _fields_ = [("M", C.c_int64), ("K", C.c_int32), ("S", C.c_int32), ("waypoints", C.c_void_p),
                ("n_timesteps", C.c_void_p), ("fixed_timesteps", C.c_int32), ("robot_timesteps", C.c_void_p)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB)
        vp, i32, i64, f64 = C.c_void_p, C.c_int32, C.c_int64, C.c_double
        L.orc_interp.argtypes = [vp, vp, i64, i32, i32, vp]
        L.orc_fk.argtypes = [vp, vp, vp]
        L.orc_centres_at.argtypes = [vp, vp, i64, i32, vp]
        L.orc_state_tables.argtypes = [vp, vp, i64, i32, vp, vp, vp, vp]
        L.orc_config_eval.argtypes = [vp, vp, i64, i32, i32, i32, vp, vp]
        L.orc_motval_batch.argtypes = [vp, vp, i32, f64, i32, vp, vp, vp]
        L.orc_ffc_batch.argtypes = [vp, vp, f64, i32, vp, vp, vp, vp]
        L.orc_pp_motval_batch.argtypes = [vp, i32, C.c_uint64, vp, vp, vp, i32, i32, f64, i32, vp, vp, vp]
        L.orc_motval_batch_ex.argtypes = [vp, vp, i32, f64, i32, i32, vp, vp, vp, vp, vp]
        L.orc_ffc_batch_ex.argtypes = [vp, vp, f64, i32, i32, vp, vp, vp, vp, vp, vp]
        L.orc_pair_sep.argtypes = [vp, vp, i64, i32, i32, i32]
        L.orc_pair_sep.restype = f64
        L.orc_baseline_motval.argtypes = [vp, vp, i32, i32, vp]
        L.orc_baseline_motval.restype = i64
        L.orc_baseline_ffc.argtypes = [vp, vp, i32, vp]
        L.orc_baseline_ffc.restype = i64
        _lib = L
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data


def threads() -> int:
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)


class OScene:
    """Oracle-side view of a scene (any object with ``robots``/``obs_spheres``/``obs_boxes``)."""

    def __init__(self, scene):
        self._keep = []
        rbs = (_Robot * max(1, len(scene.robots)))()
        for i, r in enumerate(scene.robots):
            arrs = [np.ascontiguousarray(x) if x is not None else None for x in
                    (r.joint_origin, r.joint_type, r.base, r.sphere_link, r.sphere)]
            arrs[0] = None if arrs[0] is None else arrs[0].astype(np.float32)
            arrs[1] = None if arrs[1] is None else arrs[1].astype(np.int32)
            arrs[2] = None if arrs[2] is None else arrs[2].astype(np.float32)
            arrs[3] = arrs[3].astype(np.int32)
            arrs[4] = arrs[4].astype(np.float32)
            sp = getattr(r, "self_pairs", None)
            sp = None if sp is None else np.ascontiguousarray(sp, dtype=np.int32).reshape(-1, 2)
            self._keep += arrs + [sp]
            if not 1 <= r.dof <= 64:   # ORC_MAX_DOF: the oracle's per-robot frame and configuration buffers
                raise ValueError(f"oracle supports 1..64 joints per robot, got {r.dof}")
            rbs[i] = _Robot(r.kind, r.dof, _ptr(arrs[0]), _ptr(arrs[1]), _ptr(arrs[2]), arrs[4].shape[0],
                            _ptr(arrs[3]), _ptr(arrs[4]), 0 if sp is None else sp.shape[0], _ptr(sp))
        osph = np.ascontiguousarray(scene.obs_spheres, dtype=np.float32).reshape(-1, 4)
        box = np.ascontiguousarray(scene.obs_boxes, dtype=np.float32).reshape(-1, 6)
        self._keep += [rbs, osph, box]
        self.s = _Scene(len(scene.robots), rbs, osph.shape[0], _ptr(osph), box.shape[0], _ptr(box))
        self.n = len(scene.robots)
        self.P = self.n * (self.n - 1) // 2
        self.n_spheres = [int(r.sphere.shape[0]) for r in scene.robots]
        self.robots = rbs

    @property
    def ref(self):
        return C.byref(self.s)


class OMotions:
    def __init__(self, mot):
        self.wp = np.ascontiguousarray(mot.waypoints, dtype=np.float32)
        self.T = None if mot.n_timesteps is None else np.ascontiguousarray(mot.n_timesteps, dtype=np.int32)
        rt = getattr(mot, "robot_timesteps", None)
        self.RT = None if rt is None else np.ascontiguousarray(rt, dtype=np.int32)
        M, _, K, S = self.wp.shape
        self.s = _Motions(M, K, S, _ptr(self.wp), _ptr(self.T), int(mot.fixed_timesteps), _ptr(self.RT))
        self.M = M

    @property
    def ref(self):
        return C.byref(self.s)


def interp(scene, mot, m, r, t):
    os_, om = OScene(scene), OMotions(mot)
    q = np.zeros(max(1, int(scene.robots[r].dof)))   # orc_interp writes dof doubles
    lib().orc_interp(os_.ref, om.ref, m, r, t, _ptr(q))
    return q


def fk(robot, q):
    """World sphere centres of one robot at configuration q (fp64), [ns][3]."""
    class _S:  # minimal scene wrapper (FK only)
        robots = [robot]
        obs_spheres = np.zeros((0, 4), np.float32)
        obs_boxes = np.zeros((0, 6), np.float32)
    os_ = OScene(_S)
    q = np.ascontiguousarray(np.asarray(q, dtype=np.float64))
    out = np.zeros((robot.sphere.shape[0], 3))
    lib().orc_fk(C.byref(os_.robots[0]), _ptr(q), _ptr(out))
    return out


def centres_at(scene, mot, m, t, _os=None, _om=None):
    os_ = _os or OScene(scene)
    om = _om or OMotions(mot)
    out = np.zeros((sum(os_.n_spheres), 3))
    lib().orc_centres_at(os_.ref, om.ref, m, t, _ptr(out))
    return out


def env_mask(check_env=True, check_self=False):
    """Oracle bit mask: 1 = robot-obstacle, 2 = self-collision link pairs."""
    return (1 if check_env else 0) | (2 if check_self else 0)


def state_tables(scene, mot, m, check_env=True, check_self=False):
    """Per-timestep strict hits / separations of motion m: env [T][n], pair [T][P]."""
    os_, om = OScene(scene), OMotions(mot)
    check_env = env_mask(check_env, check_self)
    T = int(mot.T_array()[m])
    eh = np.zeros((T, os_.n), np.int32)
    es = np.zeros((T, os_.n))
    ph = np.zeros((T, max(os_.P, 1)), np.int32)
    ps = np.zeros((T, max(os_.P, 1)))
    lib().orc_state_tables(os_.ref, om.ref, m, int(check_env), _ptr(eh), _ptr(es), _ptr(ph), _ptr(ps))
    return eh.astype(bool), es, ph[:, : os_.P].astype(bool), ps[:, : os_.P]


def config_eval(scene, q, check_env=True, n_threads=None, check_self=False):
    """Composite configurations q [N][n][S] -> (min signed separation, strict hit)."""
    os_ = OScene(scene)
    check_env = env_mask(check_env, check_self)
    q = np.ascontiguousarray(q, dtype=np.float32)
    N, S = q.shape[0], q.shape[2]
    ms = np.zeros(N)
    hit = np.zeros(N, np.uint8)
    lib().orc_config_eval(os_.ref, _ptr(q), N, S, int(check_env), n_threads or threads(), _ptr(ms), _ptr(hit))
    return ms, hit.astype(bool)


def motval(scene, mot, check_env=True, band=BAND, n_threads=None, check_self=False):
    """Plain-definition MotVal: (valid, ambiguous_motion, definite_hit) per motion."""
    os_, om = OScene(scene), OMotions(mot)
    check_env = env_mask(check_env, check_self)
    v = np.zeros(om.M, np.uint8)
    c = np.zeros(om.M, np.uint8)
    d = np.zeros(om.M, np.uint8)
    lib().orc_motval_batch(os_.ref, om.ref, int(check_env), band, n_threads or threads(), _ptr(v), _ptr(c), _ptr(d))
    return v, c.astype(bool), d.astype(bool)


def motval_counts(scene, mot, check_env=True, band=BAND, n_threads=None, check_self=False, full_scan=True):
    """MotVal with per-motion state counts: (valid, ambiguous_motion, definite_hit,
    ambiguous_states, scanned_states); full_scan classifies every state of every motion."""
    os_, om = OScene(scene), OMotions(mot)
    check_env = env_mask(check_env, check_self)
    v = np.zeros(om.M, np.uint8)
    c = np.zeros(om.M, np.uint8)
    d = np.zeros(om.M, np.uint8)
    na = np.zeros(om.M, np.int32)
    ns = np.zeros(om.M, np.int32)
    lib().orc_motval_batch_ex(os_.ref, om.ref, int(check_env), band, int(full_scan), n_threads or threads(),
                              _ptr(v), _ptr(c), _ptr(d), _ptr(na), _ptr(ns))
    return v, c.astype(bool), d.astype(bool), na, ns


def ffc_counts(scene, mot, band=BAND, n_threads=None, full_scan=True):
    """FFC with per-motion counts: (key, k_lo, k_hi, ambiguous, ambiguous_states, scanned_states)."""
    os_, om = OScene(scene), OMotions(mot)
    k = np.zeros(om.M, np.uint32)
    lo = np.zeros(om.M, np.uint32)
    hi = np.zeros(om.M, np.uint32)
    a = np.zeros(om.M, np.uint8)
    na = np.zeros(om.M, np.int32)
    ns = np.zeros(om.M, np.int32)
    lib().orc_ffc_batch_ex(os_.ref, om.ref, band, int(full_scan), n_threads or threads(), _ptr(k), _ptr(lo),
                           _ptr(hi), _ptr(a), _ptr(na), _ptr(ns))
    return k, lo, hi, a.astype(bool), na, ns


def pp_motval(scene, focus, partners, cand, t_start, paths, horizon, check_env=True, band=BAND, n_threads=None,
              check_self=False):
    """PP-ST-RRT MotVal variant (orc_pp_motval_batch): candidates ``cand`` (waypoints
    [M][1][K][S], robot ``focus``) starting at absolute timesteps ``t_start`` against the
    fixed ``paths`` (one motion [1][n][Kp][S], per-robot lengths) of the ``partners``
    (iterable of robot indices).  Returns (valid, ambiguous_motion, definite_hit)."""
    os_ = OScene(scene)
    oc, op = OMotions(cand), OMotions(paths)
    ts = np.ascontiguousarray(t_start, dtype=np.int32)
    assert ts.shape == (oc.M,) and op.M == 1
    mask = 0
    for j in partners:
        mask |= 1 << int(j)
    v = np.zeros(oc.M, np.uint8)
    c = np.zeros(oc.M, np.uint8)
    d = np.zeros(oc.M, np.uint8)
    lib().orc_pp_motval_batch(os_.ref, int(focus), mask, oc.ref, _ptr(ts), op.ref, int(horizon),
                              env_mask(check_env, check_self), band, n_threads or threads(), _ptr(v), _ptr(c),
                              _ptr(d))
    return v, c.astype(bool), d.astype(bool)


def ffc(scene, mot, band=BAND, n_threads=None):
    """Plain-definition FFC: (key, k_lo, k_hi, ambiguous) per motion; NONE = 0xFFFFFFFF."""
    os_, om = OScene(scene), OMotions(mot)
    k = np.zeros(om.M, np.uint32)
    lo = np.zeros(om.M, np.uint32)
    hi = np.zeros(om.M, np.uint32)
    a = np.zeros(om.M, np.uint8)
    lib().orc_ffc_batch(os_.ref, om.ref, band, n_threads or threads(), _ptr(k), _ptr(lo), _ptr(hi), _ptr(a))
    return k, lo, hi, a.astype(bool)


def pair_sep(scene, mot, m, t, i, j, _os=None, _om=None):
    os_ = _os or OScene(scene)
    om = _om or OMotions(mot)
    return lib().orc_pair_sep(os_.ref, om.ref, m, t, i, j)


def baseline_motval(scene, mot, check_env=True, n_threads=None, check_self=False):
    os_, om = OScene(scene), OMotions(mot)
    check_env = env_mask(check_env, check_self)
    v = np.zeros(om.M, np.uint8)
    n = lib().orc_baseline_motval(os_.ref, om.ref, int(check_env), n_threads or threads(), _ptr(v))
    return v, int(n)


def baseline_ffc(scene, mot, n_threads=None):
    os_, om = OScene(scene), OMotions(mot)
    k = np.zeros(om.M, np.uint32)
    n = lib().orc_baseline_ffc(os_.ref, om.ref, n_threads or threads(), _ptr(k))
    return k, int(n)


def decode(key, n_robots):
    """key = t*P + rank(i,j) (lexicographic pair rank) -> (t, i, j); None for NONE."""
    key = int(key)
    if key == NONE:
        return None
    P = n_robots * (n_robots - 1) // 2
    t, p = divmod(key, P)
    for i in range(n_robots):
        for j in range(i + 1, n_robots):
            if p == 0:
                return t, i, j
            p -= 1
    raise ValueError(key)
