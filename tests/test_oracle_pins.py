"""Pins of the fp64 CPU oracle against things other than itself:
values the paper/SPEC print for worked examples (tests/golden/paper_examples.json),
closed forms, a different FK formulation (standard DH), library routines (scipy
Rotation/Slerp), brute-force transcriptions of Alg. 1/2, and invariants.
All CPU-only."""
import json
import math
import os

import numpy as np
import pytest

import oracle
from alg_transcriptions import ffc_alg2, motval_alg1, pack_linear, pack_rake
from helpers import ball, knots_motion, motions, pose, rand_tiny_case, scene
from paper_2604_23960_b200 import gen

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_examples.json")))


def key_of(t, i, j, n):
    P = n * (n - 1) // 2
    rank = i * n - i * (i + 1) // 2 + (j - i - 1)
    return t * P + rank


# ---------------------------------------------------------------- P1 packing
def test_packing_formulas_paper_fig1():
    g = GOLD["packing"]
    for b, ts in g["rake"].items():
        assert pack_rake(int(b), g["t_max"], g["batch_size"]) == ts
    for b, ts in g["linear"].items():
        assert pack_linear(int(b), g["t_max"], g["batch_size"]) == ts
    # Fig. 1: the first rake is {0, t/4, 2t/4, 3t/4}
    assert pack_rake(0, 16, 4) == [0, 16 // 4, 2 * 16 // 4, 3 * 16 // 4]
    # coverage equality: rake and linear visit every timestep exactly once
    for t_max in range(1, 60):
        for W in (1, 3, 4, 8, 32):
            nb = math.ceil(t_max / W)
            r = sorted(sum((pack_rake(b, t_max, W) for b in range(nb)), []))
            l_ = sorted(sum((pack_linear(b, t_max, W) for b in range(nb)), []))
            assert r == l_ == list(range(t_max))


# ---------------------------------------------------------------- P2 crossing
def test_crossing_spec_example():
    g = GOLD["crossing"]
    sc = scene([ball(g["radius"]), ball(g["radius"])])
    mo = motions([[[pose(p) for p in g["A"]], [pose(p) for p in g["B"]]]], g["T"])
    v, amb, _ = oracle.motval(sc, mo)
    assert bool(v[0]) == g["motval"] and not amb[0]
    k, lo, hi, a = oracle.ffc(sc, mo)
    assert oracle.decode(k[0], 2) == tuple(g["ffc"])
    eh, es, ph, ps = oracle.state_tables(sc, mo, 0)
    assert not ph[4, 0] and abs(ps[4, 0]) < 1e-12       # t=4: exactly touching -> free
    assert ph[5, 0] and ph[6, 0] is not None


# ---------------------------------------------------------------- P3 contact time
def test_contact_time_closed_form():
    g = GOLD["contact_time"]
    sc = scene([ball(g["rA"]), ball(g["rB"])])
    mo = motions([[[pose(p) for p in g["A"]], [pose(g["B"]), pose(g["B"])]]], g["T"])
    eh, es, ph, ps = oracle.state_tables(sc, mo, 0)
    hits = np.nonzero(ph[:, 0])[0]
    assert hits.min() == g["colliding_t"][0] and hits.max() == g["colliding_t"][1]
    assert len(hits) == g["colliding_t"][1] - g["colliding_t"][0] + 1
    assert abs(ps[25, 0] - g["sep_t25"]) < 1e-5 and abs(ps[26, 0] - g["sep_t26"]) < 1e-5
    k, lo, hi, a = oracle.ffc(sc, mo)
    assert oracle.decode(k[0], 2) == tuple(g["ffc"]) and not a[0]
    assert oracle.motval(sc, mo)[0][0] == 0
    tv = g["touching_variant"]
    mo2 = motions([[[pose(p) for p in g["A"]], [pose(tv["B"]), pose(tv["B"])]]], g["T"])
    eh, es, ph, ps = oracle.state_tables(sc, mo2, 0)
    assert not ph.any() and abs(ps[tv["touch_t"], 0]) < 1e-12
    v, amb, d = oracle.motval(sc, mo2)
    assert bool(v[0]) == tv["motval"] and amb[0]     # touching state is inside the band


# ---------------------------------------------------------------- P4 general two-sphere
def test_two_sphere_first_contact_closed_form():
    rng = np.random.default_rng(7)
    checked = 0
    while checked < 300:
        a0, a1, b0, b1 = (rng.uniform(-2, 2, 3) for _ in range(4))
        ra, rb = rng.uniform(0.1, 0.6, 2)
        T = int(rng.integers(2, 80))
        a0, a1, b0, b1 = (np.float32(x).astype(np.float64) for x in (a0, a1, b0, b1))
        ra, rb = float(np.float32(ra)), float(np.float32(rb))
        d0, dv, R = a0 - b0, (a1 - a0) - (b1 - b0), ra + rb
        # |d0 + s dv|^2 = R^2  ->  A s^2 + B s + C = 0
        A, B, Cc = dv @ dv, 2 * d0 @ dv, d0 @ d0 - R * R
        s = np.arange(T) / (T - 1)
        sep = np.sqrt(np.maximum(A * s * s + B * s + Cc + R * R, 0)) - R
        if np.min(np.abs(sep)) < 1e-6:
            continue
        disc = B * B - 4 * A * Cc
        expect = None
        if disc > 0 and A > 0:
            sm, sp = (-B - math.sqrt(disc)) / (2 * A), (-B + math.sqrt(disc)) / (2 * A)
            t = 0 if sm < 0 else math.floor((T - 1) * sm) + 1
            if t <= T - 1 and t / (T - 1) < sp:
                expect = t
        sc = scene([ball(ra), ball(rb)])
        mo = motions([[[pose(a0), pose(a1)], [pose(b0), pose(b1)]]], T)
        k = oracle.ffc(sc, mo)[0][0]
        got = None if k == oracle.NONE else int(k)
        assert got == expect, (a0, a1, b0, b1, ra, rb, T)
        checked += 1


# ---------------------------------------------------------------- P5 planar arm (hand FK)
def _planar_arm(L1, L2):
    o1 = np.eye(3, 4).reshape(12)
    o2 = np.eye(3, 4)
    o2[0, 3] = L1
    return gen.Robot(kind=gen.CHAIN, dof=2, sphere_link=np.array([0, 1], np.int32),
                     sphere=np.array([[L1, 0, 0, 0.05], [L2, 0, 0, 0.05]], np.float32),
                     joint_origin=np.stack([o1, o2.reshape(12)]).astype(np.float32),
                     joint_type=np.zeros(2, np.int32), base=None)


def test_planar_arm_hand_fk():
    g = GOLD["planar_arm"]
    rb = _planar_arm(g["L1"], g["L2"])
    for c in g["cases"]:
        xyz = oracle.fk(rb, c["q"])
        assert np.allclose(xyz[0], c["elbow"], atol=1e-12)
        assert np.allclose(xyz[1], c["tip"], atol=1e-12)


# ---------------------------------------------------------------- P6 prismatic sphere-bot
def test_prismatic_spherebot_pure_translation():
    """sphere-bot q=(1,2,3) -> centre offset by (1,2,3)."""
    # joint axes: local z rotated onto world x, then y, then z (exact 0/+-1 rotations)
    Ry90 = np.array([[0, 0, 1], [0, 1, 0], [-1, 0, 0]], float)      # z -> x
    R1 = Ry90
    O2 = R1.T @ np.array([[1, 0, 0], [0, 0, 1], [0, -1, 0]], float)  # cumulative z -> y
    R2 = R1 @ O2
    O3 = R2.T                                                        # cumulative -> identity
    origins = [np.concatenate([R, np.zeros((3, 1))], 1).reshape(12) for R in (R1, O2, O3)]
    assert np.allclose((R1 @ O2)[:, 2], [0, 1, 0]) and np.allclose((R1 @ O2 @ O3), np.eye(3))
    rb = gen.Robot(kind=gen.CHAIN, dof=3, sphere_link=np.array([2], np.int32),
                   sphere=np.array([[0.1, -0.2, 0.3, 0.15]], np.float32),
                   joint_origin=np.asarray(origins, np.float32), joint_type=np.ones(3, np.int32), base=None)
    assert np.allclose(oracle.fk(rb, [0, 0, 0])[0], [0.1, -0.2, 0.3], atol=1e-7)
    assert np.allclose(oracle.fk(rb, [1, 2, 3])[0], [1.1, 1.8, 3.3], atol=1e-7)


# ---------------------------------------------------------------- P15 DH vs ABI chain
def _dh_chain(rng, dof, base_rot):
    a = rng.uniform(0.1, 0.4, dof).astype(np.float32)
    d = rng.uniform(-0.2, 0.2, dof).astype(np.float32)
    alpha_choices = [(0.0, 1.0), (1.0, 0.0), (-1.0, 0.0), (0.0, -1.0)]   # (sin, cos) for +-pi/2, 0, pi
    sc = [alpha_choices[i] for i in rng.integers(0, 4, dof)]
    origins = [np.eye(3, 4).reshape(12)]
    for j in range(1, dof):
        s, c = sc[j - 1]
        origins.append(np.array([[1, 0, 0, a[j - 1]], [0, c, -s, 0], [0, s, c, d[j - 1]]], float).reshape(12))
    base = np.concatenate([base_rot, rng.uniform(-1, 1, (3, 1))], 1).astype(np.float32)
    ns = 3 * dof
    link = np.repeat(np.arange(dof), 3).astype(np.int32)
    off = rng.uniform(-0.2, 0.2, (ns, 3))
    sph = np.concatenate([off, rng.uniform(0.02, 0.1, (ns, 1))], 1).astype(np.float32)
    rb = gen.Robot(kind=gen.CHAIN, dof=dof, sphere_link=link, sphere=sph,
                   joint_origin=np.asarray(origins, np.float32), joint_type=np.zeros(dof, np.int32),
                   base=base.reshape(12))
    return rb, a, d, sc


def _h(R=None, p=None):
    H = np.eye(4)
    if R is not None:
        H[:3, :3] = R
    if p is not None:
        H[:3, 3] = p
    return H


def test_chain_fk_matches_standard_dh_product():
    """the standard distal-DH product Rz(theta) Tz(d) Tx(a) Rx(alpha) and the
    ABI chain T_j = T_{j-1} O_j Rz(q_j) agree to <= 1e-12 m."""
    from scipy.spatial.transform import Rotation
    rng = np.random.default_rng(11)
    for trial in range(50):
        dof = int(rng.integers(1, 17))   # up to MRV_MAX_DOF = 16 joints
        Rb = Rotation.random(random_state=trial).as_matrix()
        rb, a, d, sc = _dh_chain(rng, dof, Rb)
        q = rng.uniform(-np.pi, np.pi, dof)
        base = rb.base.astype(np.float64).reshape(3, 4)
        T = _h(base[:, :3], base[:, 3])
        expect = np.zeros((rb.n_spheres, 3))
        for j in range(dof):
            cz, sz = math.cos(q[j]), math.sin(q[j])
            Tj = T @ _h(np.array([[cz, -sz, 0], [sz, cz, 0], [0, 0, 1]]))    # frame after Rz(theta_j)
            for k in np.nonzero(rb.sphere_link == j)[0]:
                expect[k] = (Tj @ np.append(rb.sphere[k, :3].astype(np.float64), 1.0))[:3]
            s, c = sc[j]
            T = Tj @ _h(p=[0, 0, float(d[j])]) @ _h(p=[float(a[j]), 0, 0]) @ _h(np.array([[1, 0, 0], [0, c, -s], [0, s, c]]))
        got = oracle.fk(rb, q)
        assert np.max(np.abs(got - expect)) <= 1e-12


def test_multi_robot_centres_equal_per_robot_fk_long_chains():
    """A scene's composite sphere centres are the concatenation of every robot's own FK
    at its own configuration -- with 16-joint chains next to other robots (the oracle's
    per-robot configuration buffers must not overlap: a 16-DOF chain's joints 8..15
    once overwrote the next robot's pose)."""
    from helpers import ball, motions, scene
    rng = np.random.default_rng(21)
    chains = []
    for dof in (16, 11, 16):
        rb, _, _, _ = _dh_chain(rng, dof, np.eye(3))
        chains.append(rb)
    robots = [chains[0], ball(0.2, (0.1, 0.0, 0.0)), chains[1], chains[2], ball(0.3)]
    sc = scene(robots)
    wp = np.zeros((1, len(robots), 1, 16), np.float32)
    for r, rb in enumerate(robots):
        if rb.kind == gen.CHAIN:
            wp[0, r, 0, :rb.dof] = rng.uniform(-np.pi, np.pi, rb.dof)
        else:
            wp[0, r, 0, :3] = rng.uniform(-1, 1, 3)
            qv = rng.normal(size=4)
            wp[0, r, 0, 3:7] = qv / np.linalg.norm(qv)
    mo = motions(wp, 5)
    got = oracle.centres_at(sc, mo, 0, 3)
    expect = np.concatenate([oracle.fk(rb, wp[0, r, 0, :rb.dof].astype(np.float64)) for r, rb in enumerate(robots)])
    assert np.max(np.abs(got - expect)) <= 1e-12


# ---------------------------------------------------------------- SE(2) / SE(3) poses
def test_se2_closed_form():
    rb = gen.Robot(kind=gen.SE2, dof=3, sphere_link=np.zeros(2, np.int32),
                   sphere=np.array([[1, 0, 0.25, 0.1], [0, 2, 0, 0.1]], np.float32))
    xyz = oracle.fk(rb, [2.0, 3.0, math.pi / 2])
    assert np.allclose(xyz, [[2, 4, 0.25], [0, 3, 0]], atol=1e-12)


def test_se3_quaternion_rotation_library():
    from scipy.spatial.transform import Rotation
    rng = np.random.default_rng(3)
    rb = gen.Robot(kind=gen.SE3, dof=7, sphere_link=np.zeros(5, np.int32),
                   sphere=np.concatenate([rng.uniform(-1, 1, (5, 3)), np.full((5, 1), 0.1)], 1).astype(np.float32))
    # 90 deg about x maps y to z
    c = math.sqrt(0.5)
    assert np.allclose(oracle.fk(rb, [0, 0, 0, c, c, 0, 0])[:, :], rb.sphere[:, :3] @ np.array([[1, 0, 0], [0, 0, 1], [0, -1, 0]]), atol=1e-7)
    for _ in range(50):
        p = rng.uniform(-3, 3, 3)
        q = rng.normal(size=4)
        s = rng.uniform(0.5, 2.0)          # non-unit quaternions: s = 2/(q.q) normalises
        got = oracle.fk(rb, np.concatenate([p, s * q]))
        R = Rotation.from_quat([q[1], q[2], q[3], q[0]])
        assert np.allclose(got, R.apply(rb.sphere[:, :3].astype(np.float64)) + p, atol=1e-12)


# ---------------------------------------------------------------- P7 slerp
def test_single_axis_slerp_closed_form():
    phi, rho, T = 2.0, 0.75, 33
    qz = [math.cos(phi / 2), 0, 0, math.sin(phi / 2)]
    sc = scene([ball(0.1, (rho, 0, 0))])
    p0, p1 = np.array([1.0, -2.0, 0.5]), np.array([3.0, 1.0, -1.0])
    mo = motions([[[pose(p0), pose(p1, qz)]]], T)
    q32 = np.float32(qz).astype(np.float64)
    phi32 = 2 * math.atan2(q32[3], q32[0])
    for t in range(T):
        u = t / (T - 1)
        pu = np.float32(p0) + u * (np.float32(p1).astype(np.float64) - np.float32(p0))
        expect = pu + rho * np.array([math.cos(u * phi32), math.sin(u * phi32), 0.0])
        assert np.allclose(oracle.centres_at(sc, mo, 0, t)[0], expect, atol=1e-12)


def test_slerp_matches_scipy():
    from scipy.spatial.transform import Rotation, Slerp
    rng = np.random.default_rng(5)
    sc = scene([ball(0.1, (0.4, -0.2, 0.3))])
    for trial in range(40):
        q0, q1 = Rotation.random(2, random_state=trial).as_quat()   # (x, y, z, w)
        if q0 @ q1 < 0:
            q1 = -q1
        w0 = [q0[3], q0[0], q0[1], q0[2]]
        w1 = [q1[3], q1[0], q1[1], q1[2]]
        p0, p1 = rng.uniform(-2, 2, 3), rng.uniform(-2, 2, 3)
        T = int(rng.integers(2, 50))
        mo = motions([[[pose(p0, w0), pose(p1, w1)]]], T)
        w32 = np.float32([w0, w1]).astype(np.float64)
        sl = Slerp([0, 1], Rotation.from_quat(w32[:, [1, 2, 3, 0]]))
        for t in range(T):
            u = t / (T - 1)
            pu = np.float32(p0) + u * (np.float32(p1).astype(np.float64) - np.float32(p0))
            expect = sl([u]).apply(np.float32([0.4, -0.2, 0.3]).astype(np.float64))[0] + pu
            assert np.allclose(oracle.centres_at(sc, mo, 0, t)[0], expect, atol=1e-9)


# ---------------------------------------------------------------- interpolation knots
def test_interpolation_knots_and_piecewise_linear():
    """Reading c.4: knots at t_k = k (T-1)/(K-1), exact; linear in between.  With
    w_k = 111 k and T = 1000, K = 10 (BASELINE cfg4 shape), q(t) = t exactly."""
    rb = gen.Robot(kind=gen.SE2, dof=3, sphere_link=np.zeros(1, np.int32), sphere=np.array([[0, 0, 0, 0.1]], np.float32))
    sc = scene([rb])
    wp = np.zeros((1, 1, 10, 3), np.float32)
    wp[0, 0, :, 0] = 111.0 * np.arange(10)
    wp[0, 0, :, 1] = np.arange(10) ** 2          # non-linear knot values: exact at knots
    mo = gen.Motions(wp, None, 1000)
    for t in list(range(0, 1000, 37)) + [999, 998, 1, 111, 444, 555]:
        q = oracle.interp(sc, mo, 0, 0, t)
        assert abs(q[0] - t) < 1e-9
        if t % 111 == 0:
            assert q[1] == float((t // 111) ** 2)
    # T == 1 and K == 1 -> first waypoint
    for wpk, T in ((wp, 1), (wp[:, :, :1], 7)):
        mo1 = gen.Motions(np.ascontiguousarray(wpk), None, T)
        assert np.all(oracle.interp(sc, mo1, 0, 0, 0) == wpk[0, 0, 0].astype(np.float64))


# ---------------------------------------------------------------- P8 / P9 predicates
def test_sphere_box_closed_forms():
    g = GOLD["sphere_box"]
    sc = scene([ball(g["r"])], boxes=[g["box"]])
    q = np.asarray([[pose(c["c"])] for c in g["cases"]], np.float32)
    ms, hit = oracle.config_eval(sc, q)
    for c, s, h in zip(g["cases"], ms, hit):
        assert bool(h) == c["hit"]
        assert abs(s - c["sep"]) < 1e-6


def test_sphere_sphere_obstacle_closed_forms():
    g = GOLD["sphere_sphere_obstacle"]
    for c in g["cases"]:
        sc = scene([ball(g["r"])], obs_spheres=[c["o"] + [g["R"]]])
        ms, hit = oracle.config_eval(sc, np.asarray([[pose([0, 0, 0])]], np.float32))
        assert bool(hit[0]) == c["hit"]
        assert abs(ms[0] - (np.linalg.norm(c["o"]) - 2.0)) < 1e-12


def test_check_env_off_skips_obstacles():
    sc = scene([ball(1.0)], obs_spheres=[[0, 0, 0, 1.0]])
    mo = motions([[[pose([0, 0, 0])]]], 5)
    assert oracle.motval(sc, mo, check_env=True)[0][0] == 0
    assert oracle.motval(sc, mo, check_env=False)[0][0] == 1


# ---------------------------------------------------------------- P10 / P11
def test_first_lane_timestep():
    g = GOLD["first_lane"]
    A = [[0, 0, 0]] * g["T"]
    B = [[10.0 * (t + 1), 0, 0] for t in range(7)] + [[0, 0, 0]]
    sc = scene([ball(g["radius"]), ball(g["radius"])])
    mo = gen.Motions(knots_motion([A, B]), None, g["T"])
    assert oracle.decode(oracle.ffc(sc, mo)[0][0], 2) == tuple(g["ffc"])


def test_three_robot_tie_spec():
    g = GOLD["three_robot_tie"]
    T = g["T"]
    far = lambda k: [[5.0 * (k + 1), 5.0 * (t + 1), 0] for t in range(T)]  # noqa: E731
    A = [[0, 0, 0]] * T
    B = [([0, 0, 0] if t == 7 else p) for t, p in enumerate(far(1))]   # (0,1) at t=7
    Cc = [([0, 0, 0] if t == 3 else p) for t, p in enumerate(far(2))]  # (0,2) at t=3
    sc = scene([ball(g["radius"])] * 3)
    mo = gen.Motions(knots_motion([A, B, Cc]), None, T)
    assert oracle.decode(oracle.ffc(sc, mo)[0][0], 3) == tuple(g["ffc"])
    for W in (1, 3, 4, 32):
        eh, es, ph, ps = oracle.state_tables(sc, mo, 0)
        assert ffc_alg2(ph, 3, W)[0] == tuple(g["ffc"])


# ---------------------------------------------------------------- P14 Cross scenario
@pytest.mark.parametrize("n", GOLD["cross"]["n"])
def test_cross_scenario_n_over_2_conflicts(n):
    half = n // 2
    robots = [ball(0.5) for _ in range(n)]
    wp = []
    for k in range(half):
        wp.append([pose([2.0 * k, 0, 0]), pose([2.0 * k, 10, 0])])
    for k in range(half):
        wp.append([pose([2.0 * k, 10, 0]), pose([2.0 * k, 0, 0])])
    sc = scene(robots)
    mo = motions([wp], 21)
    eh, es, ph, ps = oracle.state_tables(sc, mo, 0)
    assert int(ph.any(axis=0).sum()) == half
    t, i, j = oracle.decode(oracle.ffc(sc, mo)[0][0], n)
    assert (i, j) == (0, half) and t == 10   # head-on at the midpoint; t=9 is exact touching


# ---------------------------------------------------------------- P12 brute force vs Alg. 1 / Alg. 2
def _plain_from_tables(eh, ph, check_env):
    valid = not (ph.any() or (check_env and eh.any()))
    first = None
    n_pairs = ph.shape[1]
    for t in range(ph.shape[0]):
        hits = np.nonzero(ph[t])[0]
        if hits.size:
            first = (t, int(hits[0]))
            break
    return valid, first, n_pairs


@pytest.mark.parametrize("seed", range(4))
def test_alg1_alg2_transcriptions_equal_plain_definition(seed):
    rng = np.random.default_rng(1000 + seed)
    n_cases = 2500
    for _ in range(n_cases):
        sc, mo = rand_tiny_case(rng)
        n = sc.n_robots
        eh, es, ph, ps = oracle.state_tables(sc, mo, 0)
        for check_env in (True, False):
            v_or = bool(oracle.motval(sc, mo, check_env=check_env, n_threads=1)[0][0])
            valid, _, _ = _plain_from_tables(eh, ph, check_env)
            assert v_or == valid
            for W in (1, 3, 4, 8, 32):
                for hier in (True, False):
                    for packing in ("rake", "linear"):
                        assert motval_alg1(eh, ph, n, W, hier, check_env, packing)[0] == v_or
        k = oracle.ffc(sc, mo, n_threads=1)[0][0]
        expect = oracle.decode(k, n)
        for W in (1, 3, 4, 32):
            assert ffc_alg2(ph, n, W)[0] == expect


# ---------------------------------------------------------------- P13 cross-query invariant
@pytest.mark.parametrize("cfg", ["cfg1", "cfg2"])
def test_motval_equals_not_ffc_or_obstacle(cfg):
    sc, mo = gen.make(cfg, 96)
    v_env = oracle.motval(sc, mo, check_env=True)[0]
    v_noenv = oracle.motval(sc, mo, check_env=False)[0]
    k = oracle.ffc(sc, mo)[0]
    for m in range(mo.M):
        eh, es, ph, ps = oracle.state_tables(sc, mo, m, check_env=True)
        obstacle_hit = bool(eh.any())
        assert bool(v_env[m]) == (not (k[m] != oracle.NONE or obstacle_hit))
        assert bool(v_noenv[m]) == (k[m] == oracle.NONE)


# ---------------------------------------------------------------- P16 symmetry / equivariance
def test_symmetry_and_permutation_equivariance():
    sc, mo = gen.make("cfg1")
    k = oracle.ffc(sc, mo)[0]
    # swap the two robots: FFC t unchanged
    sc2 = gen.Scene(sc.robots[::-1], sc.obs_spheres, sc.obs_boxes)
    mo2 = gen.Motions(np.ascontiguousarray(mo.waypoints[:, ::-1]), None, mo.fixed_timesteps)
    k2 = oracle.ffc(sc2, mo2)[0]
    assert np.array_equal(k == oracle.NONE, k2 == oracle.NONE)
    assert np.array_equal(k[k != oracle.NONE] // 1, k2[k2 != oracle.NONE] // 1)
    # permute motions: outputs permute
    perm = np.random.default_rng(0).permutation(mo.M)
    v = oracle.motval(sc, mo)[0]
    vp = oracle.motval(sc, mo.subset(perm))[0]
    assert np.array_equal(v[perm], vp)
    assert np.array_equal(k[perm], oracle.ffc(sc, mo.subset(perm))[0])


# ---------------------------------------------------------------- library SE(3) brute force
def test_state_tables_match_scipy_brute_force():
    """Centres via scipy Slerp + Rotation.apply and brute-force pair distances (numpy)
    agree with the oracle's strict pair predicates away from the band."""
    from scipy.spatial.transform import Rotation, Slerp
    rng = np.random.default_rng(21)
    for _ in range(200):
        sc, mo = rand_tiny_case(rng, env=False)
        if sc.n_robots < 2 or mo.K != 2:
            continue
        T = mo.fixed_timesteps
        eh, es, ph, ps = oracle.state_tables(sc, mo, 0, check_env=False)
        cen = []
        for r, rb in enumerate(sc.robots):
            w = mo.waypoints[0, r].astype(np.float64)
            sl = Slerp([0, 1], Rotation.from_quat(w[:, [4, 5, 6, 3]]))
            rows = []
            for t in range(T):
                u = 0.0 if T == 1 else t / (T - 1)
                p = w[0, :3] + u * (w[1, :3] - w[0, :3])
                rows.append(sl([u]).apply(rb.sphere[:, :3].astype(np.float64)) + p)
            cen.append(np.asarray(rows))
        p = 0
        for i in range(sc.n_robots):
            for j in range(i + 1, sc.n_robots):
                d = np.linalg.norm(cen[i][:, :, None, :] - cen[j][:, None, :, :], axis=-1)
                R = sc.robots[i].sphere[:, 3][:, None].astype(np.float64) + sc.robots[j].sphere[:, 3][None, :]
                sep = (d - R).reshape(T, -1).min(axis=1)
                ok = np.abs(sep) > 1e-6
                assert np.array_equal((sep < 0)[ok], ph[ok, p])
                assert np.allclose(sep, ps[:, p], atol=1e-6)
                p += 1


# ---------------------------------------------------------------- band classification
def test_band_classification():
    """BASELINE north_star: states within 1e-4 m of contact are ambiguous, counted not compared."""
    sc = scene([ball(0.5), ball(0.5)])
    for gap, amb_expect, valid_expect in ((5e-5, True, True), (-5e-5, True, False), (2e-4, False, True),
                                          (-2e-4, False, False)):
        x = 1.0 + gap
        mo = motions([[[pose([0, 0, 0])], [pose([x, 0, 0])]]], 3)
        v, amb, d = oracle.motval(sc, mo)
        assert bool(amb[0]) == amb_expect and bool(v[0]) == valid_expect
        k, lo, hi, a = oracle.ffc(sc, mo)
        assert bool(a[0]) == amb_expect
        if gap < 0:
            assert k[0] == 0
        if gap <= -2e-4:
            assert hi[0] == 0


# ---------------------------------------------------------------- f1 self-collision
def _fold_arm(pairs):
    """3-link planar chain, unit links; one r=0.3 sphere at the origin of links 0 and 2.
    Link 2's origin sits at Rz(q0)[(1,0,0) + Rz(q1)(1,0,0)], so its distance to the link-0
    sphere is sqrt(2 + 2 cos q1) (closed form) and the pair overlaps iff that is < 0.6."""
    o = [np.eye(3, 4).reshape(12)]
    for _ in range(2):
        m = np.eye(3, 4)
        m[0, 3] = 1.0
        o.append(m.reshape(12))
    return gen.Robot(kind=gen.CHAIN, dof=3, sphere_link=np.array([0, 2], np.int32),
                     sphere=np.array([[0, 0, 0, 0.3], [0, 0, 0, 0.3]], np.float32),
                     joint_origin=np.asarray(o, np.float32), joint_type=np.zeros(3, np.int32), base=None,
                     self_pairs=None if pairs is None else np.asarray(pairs, np.int32))


def test_self_collision_closed_form():
    rb = _fold_arm([[0, 2]])
    sc = scene([rb])
    qs = np.linspace(0.0, math.pi, 41)
    q = np.zeros((qs.size, 1, 3), np.float32)
    q[:, 0, 0] = 0.7
    q[:, 0, 1] = qs
    ms, hit = oracle.config_eval(sc, q, check_env=False, check_self=True)
    q1 = q[:, 0, 1].astype(np.float64)
    expect = np.sqrt(np.maximum(2 + 2 * np.cos(q1), 0)) - 0.6
    assert np.allclose(ms, expect, atol=1e-6)
    ok = np.abs(expect) > 1e-6
    assert np.array_equal(hit[ok], (expect < 0)[ok])
    assert hit[-1] and not hit[0]
    # not listed -> never checked; obstacle mode alone ignores self pairs
    ms2, hit2 = oracle.config_eval(scene([_fold_arm(None)]), q, check_env=False, check_self=True)
    assert not hit2.any()
    ms3, hit3 = oracle.config_eval(sc, q, check_env=True, check_self=False)
    assert not hit3.any()


def test_self_collision_in_motval_and_not_in_ffc():
    rb = _fold_arm([[0, 2]])
    sc = scene([rb, ball(0.1)])
    wp = np.zeros((1, 2, 2, 7), np.float32)
    wp[0, 0, 0, :3] = [0.0, 0.0, 0.0]
    wp[0, 0, 1, :3] = [0.0, math.pi, 0.0]        # folds onto itself at the end
    wp[0, 1, :, :] = pose([50.0, 50.0, 0.0])      # far-away ball: no robot-robot contact
    mo = gen.Motions(wp, None, 33)
    assert oracle.motval(sc, mo, check_env=False, check_self=True)[0][0] == 0
    assert oracle.motval(sc, mo, check_env=True, check_self=False)[0][0] == 1
    assert oracle.ffc(sc, mo)[0][0] == oracle.NONE
    eh, es, ph, ps = oracle.state_tables(sc, mo, 0, check_env=False, check_self=True)
    t_first = int(np.nonzero(eh[:, 0])[0][0])
    # closed form: q1(t) = pi t / 32, first t with sqrt(2 + 2 cos q1) < 0.6
    t_expect = next(t for t in range(33) if math.sqrt(max(2 + 2 * math.cos(math.pi * t / 32), 0)) < 0.6)
    assert t_first == t_expect


# ---------------------------------------------------------------- f3: per-robot path lengths (stay at goal)
def test_stay_at_goal_closed_form():
    """t_max = max |p_i|; a robot whose path ended stays at its goal.
    A: 0 -> 4 over 5 timesteps then parked at x = 4; B: 10 -> 0 over 11.  |x_A - x_B| < 2
    first at t = 5 (t = 4: exactly touching)."""
    sc = scene([ball(1.0), ball(1.0)])
    wp = np.asarray([[[pose([0, 0, 0]), pose([4, 0, 0])], [pose([10, 0, 0]), pose([0, 0, 0])]]], np.float32)
    mo = gen.Motions(wp, None, 0, np.array([[5, 11]], np.int32))
    assert mo.T_array()[0] == 11
    assert np.allclose(oracle.interp(sc, mo, 0, 0, 7)[:3], [4, 0, 0])
    assert np.allclose(oracle.interp(sc, mo, 0, 1, 7)[:3], [3, 0, 0])
    assert oracle.decode(oracle.ffc(sc, mo)[0][0], 2) == (5, 0, 1)
    eh, es, ph, ps = oracle.state_tables(sc, mo, 0)
    assert ph.shape[0] == 11 and np.nonzero(ph[:, 0])[0].tolist() == [5, 6, 7]


# ---------------------------------------------------------------- round 2: pins of the remaining outputs
def _chain16():
    """A 16-joint chain (more joints than any BASELINE arm): one sphere per link."""
    o = np.tile(np.eye(3, 4).reshape(12), (16, 1))
    o[1:, 3] = 0.1
    return gen.Robot(kind=gen.CHAIN, dof=16, sphere_link=np.arange(16, dtype=np.int32),
                     sphere=np.tile(np.array([[0.05, 0, 0, 0.02]], np.float32), (16, 1)),
                     joint_origin=o.astype(np.float32), joint_type=np.zeros(16, np.int32), base=None)


def test_interp_16_joint_chain_matches_numpy_interp():
    """orc_interp writes all 16 joints (the wrapper's buffer is sized by dof) and equals
    numpy's piecewise-linear interpolation through the knots t_k = k (T-1)/(K-1) (reading
    c.4, "discretizing them into intermediate configurations")."""
    rng = np.random.default_rng(16)
    sc = scene([_chain16(), _chain16()])
    K, T = 4, 31
    wp = rng.uniform(-2.9, 2.9, (1, 2, K, 16)).astype(np.float32)
    mo = gen.Motions(wp, None, T)
    tk = np.arange(K) * (T - 1) / (K - 1)
    for r in range(2):
        for t in range(T):
            q = oracle.interp(sc, mo, 0, r, t)
            assert q.shape == (16,)
            expect = [np.interp(t, tk, wp[0, r, :, d].astype(np.float64)) for d in range(16)]
            assert np.allclose(q, expect, rtol=0, atol=1e-12), (r, t)


def _first_hit_tables(eh, ph, check_env):
    """Brute force over the per-state tables: first timestep with a strict hit (or None)."""
    any_t = ph.any(axis=1) | (eh.any(axis=1) if check_env else False)
    hits = np.nonzero(any_t)[0]
    return None if hits.size == 0 else int(hits[0])


@pytest.mark.parametrize("seed", range(2))
def test_baseline_scan_equals_plain_definition(seed):
    """The timed CPU baseline (sequential linear scan, exit at the first
    strict hit) returns the plain-definition verdicts (PAPER.md:36 for MotVal,
    the lexmin conflict of PAPER.md:355 for FFC) and evaluates exactly first-hit + 1 states
    (all T when there is none) -- an early break that skipped states would fail here."""
    rng = np.random.default_rng(4000 + seed)
    for _ in range(5000):
        sc, mo = rand_tiny_case(rng)
        n, T = sc.n_robots, mo.fixed_timesteps
        eh, es, ph, ps = oracle.state_tables(sc, mo, 0)
        for check_env in (True, False):
            v, work = oracle.baseline_motval(sc, mo, check_env=check_env, n_threads=1)
            first = _first_hit_tables(eh, ph, check_env)
            assert bool(v[0]) == (first is None)
            assert work == (T if first is None else first + 1)
            assert bool(v[0]) == bool(oracle.motval(sc, mo, check_env=check_env, n_threads=1)[0][0])
        k, work = oracle.baseline_ffc(sc, mo, n_threads=1)
        first = _first_hit_tables(eh, ph, False)
        if n < 2:
            assert k[0] == oracle.NONE and work == 0
            continue
        expect = oracle.NONE if first is None else first * (n * (n - 1) // 2) + int(np.nonzero(ph[first])[0][0])
        assert k[0] == expect == oracle.ffc(sc, mo, n_threads=1)[0][0]
        assert work == (T if first is None else first + 1)


def test_ffc_band_keys_closed_form():
    """k_lo / k_hi (SURVEY §8(c) comparison rule): two r = 0.5 balls, 5e-5 m apart at t = 0
    (inside the 1e-4 m band, free), 4 m apart at t = 1, overlapping by 0.5 m at t = 2 (knots
    at t = 0, 1, 2): key = 2 (t = 2), k_lo = 0, k_hi = 2P = 2, ambiguous."""
    sc = scene([ball(0.5), ball(0.5)])
    mo = motions([[[pose([0, 0, 0])] * 3, [pose([1.00005, 0, 0]), pose([5, 0, 0]), pose([0.5, 0, 0])]]], 3)
    k, lo, hi, a = oracle.ffc(sc, mo)
    assert (int(k[0]), int(lo[0]), int(hi[0]), bool(a[0])) == (2, 0, 2, True)
    # three robots: (0,2) inside the band at t = 1, (0,1) deep at t = 2, (1,2) never close;
    # P = 3, rank(0,1) = 0, rank(0,2) = 1 -> k_lo = 1*3 + 1 = 4, key = k_hi = 2*3 + 0 = 6
    sc3 = scene([ball(0.5), ball(0.5), ball(0.5)])
    far = pose([0, 50, 0])
    mo3 = motions([[[pose([0, 0, 0])] * 3,
                    [pose([9, 0, 0]), pose([9, 0, 0]), pose([0.25, 0, 0])],
                    [pose([0, -9, 0]), pose([0, -1.00005, 0]), far]]], 3)
    k, lo, hi, a = oracle.ffc(sc3, mo3)
    assert (int(k[0]), int(lo[0]), int(hi[0]), bool(a[0])) == (6, 4, 6, True)
    assert oracle.decode(lo[0], 3) == (1, 0, 2) and oracle.decode(k[0], 3) == (2, 0, 1)
    # outside the band on both sides: k_lo = k_hi = key, not ambiguous
    mo4 = motions([[[pose([0, 0, 0])] * 3, [pose([1.0003, 0, 0]), pose([5, 0, 0]), pose([0.5, 0, 0])]]], 3)
    k, lo, hi, a = oracle.ffc(sc, mo4)
    assert (int(k[0]), int(lo[0]), int(hi[0]), bool(a[0])) == (2, 2, 2, False)


def test_pair_sep_closed_form_and_tables():
    """orc_pair_sep (the GPU band check's separation) equals the closed-form separations of
    the contact-time example (golden P3: +0.0753 m at t = 25, -0.0237 m at t = 26) and, on
    random tiny cases, the numpy brute force over the oracle's own centres and the
    per-state tables for every (t, pair)."""
    g = GOLD["contact_time"]
    sc = scene([ball(g["rA"]), ball(g["rB"])])
    mo = motions([[[pose(p) for p in g["A"]], [pose(g["B"]), pose(g["B"])]]], g["T"])
    A0, A1, B = (np.asarray(x, np.float32).astype(np.float64) for x in (g["A"][0], g["A"][1], g["B"]))
    R = float(np.float32(g["rA"])) + float(np.float32(g["rB"]))
    for t in range(g["T"]):
        a = A0 + t / (g["T"] - 1) * (A1 - A0)
        assert abs(oracle.pair_sep(sc, mo, 0, t, 0, 1) - (np.linalg.norm(a - B) - R)) < 1e-12
    assert abs(oracle.pair_sep(sc, mo, 0, 25, 0, 1) - g["sep_t25"]) < 1e-4
    assert abs(oracle.pair_sep(sc, mo, 0, 26, 0, 1) - g["sep_t26"]) < 1e-4
    rng = np.random.default_rng(77)
    for _ in range(200):
        sc, mo = rand_tiny_case(rng, env=False)
        if sc.n_robots < 2:
            continue
        eh, es, ph, ps = oracle.state_tables(sc, mo, 0, check_env=False)
        off = np.cumsum([0] + [r.sphere.shape[0] for r in sc.robots])
        for t in range(mo.fixed_timesteps):
            c = oracle.centres_at(sc, mo, 0, t)
            p = 0
            for i in range(sc.n_robots):
                for j in range(i + 1, sc.n_robots):
                    d = np.linalg.norm(c[off[i]:off[i + 1], None] - c[None, off[j]:off[j + 1]], axis=-1)
                    rr = sc.robots[i].sphere[:, 3, None].astype(np.float64) + sc.robots[j].sphere[None, :, 3]
                    s = oracle.pair_sep(sc, mo, 0, t, i, j)
                    assert s == ps[t, p]
                    assert abs(s - (d - rr).min()) < 1e-12
                    p += 1


def test_ambiguous_state_counts_closed_form():
    """Ambiguous-state counts (BASELINE north_star: states within 1e-4 m of contact are
    counted and reported).  Ball A (r = 0.5) moves (0,0,0) -> (8,0,0) over T = 65 (x = t/8);
    ball B (r = 0.5) sits at (4, y, 0).  The separation at t is sqrt((t/8 - 4)^2 + y^2) - 1,
    so for y = 1.00005 only t = 32 is inside the band (+5e-5 m) and no state collides."""
    sc = scene([ball(0.5), ball(0.5)])
    for y, n_band in ((1.00005, 1), (1.0003, 0), (1.0, 1)):
        mo = motions([[[pose([0, 0, 0]), pose([8, 0, 0])], [pose([4, y, 0])] * 2]], 65)
        yy = float(np.float32(y))
        sep = np.sqrt((np.arange(65) / 8 - 4) ** 2 + yy ** 2) - 1.0
        assert int((np.abs(sep) < oracle.BAND).sum()) == n_band
        v, amb, d, na, ns = oracle.motval_counts(sc, mo)
        assert (int(na[0]), int(ns[0]), bool(v[0]), bool(amb[0])) == (n_band, 65, True, n_band > 0)
        k, lo, hi, a, fa, fs = oracle.ffc_counts(sc, mo)
        assert (int(fa[0]), int(fs[0]), int(k[0]), bool(a[0])) == (n_band, 65, oracle.NONE, n_band > 0)
    # a definite hit first (t = 0..2, y = 0.2), then a band state (t = 32): the early-stopping
    # scan classifies 1 state, the full scan all 65 and finds the band state
    wp = np.zeros((1, 2, 3, 7), np.float32)
    wp[0, :, :, 3] = 1.0
    wp[0, 0, :, 0] = [0.0, 4.0, 8.0]                # A: x = t/8 with knots at t = 0, 32, 64
    wp[0, 1, :, 0] = [0.2, 4.0, 20.0]               # B: overlaps A at t = 0, 1.00005 m off at t = 32
    wp[0, 1, 1, 1] = 1.00005
    mo = gen.Motions(wp, None, 65)
    v, amb, d, na, ns = oracle.motval_counts(sc, mo, full_scan=False)
    assert (int(na[0]), int(ns[0]), bool(v[0]), bool(d[0])) == (0, 1, False, True)
    v, amb, d, na, ns = oracle.motval_counts(sc, mo, full_scan=True)
    assert (int(na[0]), int(ns[0]), bool(amb[0])) == (1, 65, False)   # a definite hit: not an ambiguous motion
    k, lo, hi, a, fa, fs = oracle.ffc_counts(sc, mo, full_scan=True)
    assert (int(k[0]), int(fa[0]), int(fs[0]), bool(a[0])) == (0, 1, 65, False)


# ---------------------------------------------------------------- f2: PP-ST-RRT MotVal variant
def test_pp_variant_closed_form_start_times():
    """A partner ball (r = 0.5) moves x = t along the fixed path 0 -> 100 over 101 absolute
    timesteps; the focus ball (r = 0.5) is parked at x = 50 for T = 10 local timesteps
    starting at absolute t_start = s.  They overlap iff |t_abs - 50| < 1, i.e. only at
    t_abs = 50 (49 and 51 touch exactly: free), so the candidate is invalid iff
    41 <= s <= 50.  With the horizon cut to 60 the partner is held at x = 59 from then on."""
    sc = scene([ball(0.5), ball(0.5)])
    paths = gen.Motions(np.asarray([[[pose([0, 0, 0]), pose([100, 0, 0])], [pose([0, 0, 0])] * 2]], np.float32),
                        None, 0, np.array([[101, 1]], np.int32))
    starts = np.arange(0, 91, dtype=np.int32)
    cand = gen.Motions(np.tile(np.asarray([[[pose([50, 0, 0])]]], np.float32), (starts.size, 1, 1, 1)), None, 10)
    v, amb, d = oracle.pp_motval(sc, 1, [0], cand, starts, paths, horizon=101)
    expect = ~((starts >= 41) & (starts <= 50))
    assert np.array_equal(v.astype(bool), expect)
    assert np.nonzero(amb)[0].tolist() == [40, 51]   # exact touching (sep 0) at t_abs = 49 / 51, no hit
    # the same with robot 0 not a partner: nothing to collide with
    v2, _, _ = oracle.pp_motval(sc, 1, [], cand, starts, paths, horizon=101)
    assert v2.all()
    # horizon 60: the partner stops at x = 59; a focus ball at x = 59 collides from t_abs = 59 on
    cand59 = gen.Motions(np.asarray([[[pose([59, 0, 0])]]] * 3, np.float32), None, 10)
    v3, _, _ = oracle.pp_motval(sc, 1, [0], cand59, np.array([40, 55, 80], np.int32), paths, horizon=60)
    assert v3.tolist() == [1, 0, 0]


def test_pp_variant_equals_restricted_composite_motval():
    """With knots at every timestep (exact states on both sides), the variant over the
    window [s, s + T) equals the plain composite definition restricted to the focus robot's
    obstacle / self checks and its pairs with the partners (state tables pinned by scipy),
    for random tiny scenes, focus robots, partner sets and start times."""
    rng = np.random.default_rng(399)
    checked = 0
    while checked < 300:
        sc, _ = rand_tiny_case(rng, max_robots=4)
        n = sc.n_robots
        if n < 2:
            continue
        H, T = int(rng.integers(8, 40)), int(rng.integers(1, 8))
        s = int(rng.integers(0, H))
        focus = int(rng.integers(0, n))
        partners = [r for r in range(n) if r != focus and rng.uniform() < 0.7]
        # fixed paths: a knot at every absolute timestep (random walk), per-robot lengths <= H
        pos = np.cumsum(rng.uniform(-0.15, 0.15, (n, H, 3)), axis=1) + rng.uniform(0.5, 2.5, (n, 1, 3))
        q = rng.normal(size=(n, H, 4))
        q /= np.linalg.norm(q, axis=-1, keepdims=True)
        for k in range(1, H):
            q[:, k] *= np.sign(np.sum(q[:, k] * q[:, k - 1], axis=-1, keepdims=True) + 1e-30)
        pw = np.concatenate([pos, q], -1)[None].astype(np.float32)
        lens = rng.integers(1, H + 1, n).astype(np.int32)
        for r in range(n):   # knot k at t = k: the path has lens[r] knots, then stays at the goal
            pw[0, r, lens[r]:] = pw[0, r, lens[r] - 1]
        paths = gen.Motions(pw, None, 0, np.full((1, n), H, np.int32))
        cw = np.concatenate([rng.uniform(0.5, 2.5, (T, 3)), q[focus, :T] if T <= H else q[focus, :1].repeat(T, 0)], -1)
        cand = gen.Motions(cw[None, None].astype(np.float32), None, T)
        check_env = bool(rng.uniform() < 0.5)
        v, amb, d = oracle.pp_motval(sc, focus, partners, cand, np.array([s], np.int32), paths, horizon=H,
                                     check_env=check_env)
        # the composite motion with the same states: focus = the candidate, partner r = its
        # path's knots at min(s + t, H - 1), t = 0..T-1 (K = T knots, one per timestep)
        comp = np.zeros((1, n, T, 7), np.float32)
        comp[..., 3] = 1.0
        comp[0, focus] = cand.waypoints[0, 0]
        ta = np.minimum(s + np.arange(T), H - 1)
        for r in partners:
            comp[0, r] = pw[0, r, ta]
        eh, es, ph, ps = oracle.state_tables(sc, gen.Motions(comp, None, T), 0, check_env=check_env)
        pairs = [(i, j) for i in range(n) for j in range(i + 1, n)]
        cols = [p for p, (i, j) in enumerate(pairs) if (i == focus and j in partners) or (j == focus and i in partners)]
        hit = (eh[:, focus] if check_env else np.zeros(T, bool)) | ph[:, cols].any(axis=1)
        assert bool(v[0]) == (not hit.any()), (focus, partners, s, T, H)
        checked += 1
