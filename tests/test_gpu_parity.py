"""GPU parity: the CUDA path (through the C ABI) against the fp64 CPU oracle on the
same seeded inputs (BASELINE.json north_star tolerances):
  * sphere centres (K3 SpheresFK export) within 1e-5 m;
  * MotVal flags bit-exact except motions whose only collisions-or-near-misses lie
    within 1e-4 m of contact (counted, reported);
  * FFC keys (t, i, j) bit-exact except when a (t, pair) at or before the oracle's
    answer is within the band; then k_lo <= k_gpu <= k_hi and the GPU's own pair
    must be within the band or overlapping (SURVEY §8(c) comparison rules).
Plus result-neutrality of every strategy/diagnostic flag, batch width and slice
count, and edge cases."""
import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from helpers import ball, general_chain, motions, pose, random_motions, random_scene, scene  # noqa: E402
from paper_2604_23960_b200 import gen, mrv  # noqa: E402

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_examples.json")))
from parity_report import REPORT  # noqa: E402  (dumped to gpurun_out/parity_report.json at session end)


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2604_23960_b200 import build
    build.build()
    yield


_cache = {}


def data(cfg, M=None):
    key = (cfg, M)
    if key not in _cache:
        sc, mo = gen.make(cfg, M)
        gs = mrv.Scene(sc)
        wp, T = mrv.to_device(mo)
        _cache[key] = (sc, mo, gs, wp, T)
    return _cache[key]


def check_motval(sc, mo, gpu_valid, check_env=True, tag="", idx=None):
    """MotVal parity; ``idx`` = the motions of a sampled full-size launch that are compared
    (the oracle evaluates ``mo.subset(idx)``).  Records the ambiguity counts (BASELINE
    north_star: ambiguous states are counted and reported)."""
    sub = mo if idx is None else mo.subset(idx)
    v, amb, d, na, ns = oracle.motval_counts(sc, sub, check_env=check_env, full_scan=False)
    g = gpu_valid.cpu().numpy() if hasattr(gpu_valid, "cpu") else np.asarray(gpu_valid)
    if idx is not None:
        g = g[idx]
    exact = ~amb
    bad = np.nonzero(g[exact] != v[exact])[0]
    REPORT[f"motval{tag}"] = {"M": int(mo.M), "compared_motions": int(sub.M), "exact_compared": int(exact.sum()),
                              "ambiguous_motions": int(amb.sum()), "mismatch": int(bad.size),
                              "ambiguous_states": int(na.sum()), "classified_states": int(ns.sum()),
                              "definite_hit_motions": int(d.sum()), "valid_frac": float(v.mean())}
    assert bad.size == 0, f"MotVal mismatches at {np.nonzero(exact)[0][bad][:10]}"
    return v, amb


def check_ffc(sc, mo, gpu_keys, tag="", idx=None):
    """FFC parity: bit-exact keys where no (t, pair) at or before the oracle's answer is in
    the band; otherwise k_lo <= k_gpu <= k_hi and the GPU's own pair within the band or
    overlapping."""
    sub = mo if idx is None else mo.subset(idx)
    k, lo, hi, amb, na, ns = oracle.ffc_counts(sc, sub, full_scan=False)
    g = mrv.keys_u32(gpu_keys) if hasattr(gpu_keys, "cpu") else np.asarray(gpu_keys, np.uint32)
    if idx is not None:
        g = g[idx]
    exact = ~amb
    bad = np.nonzero(g[exact] != k[exact])[0]
    assert bad.size == 0, f"FFC mismatches at {np.nonzero(exact)[0][bad][:10]}: gpu {g[exact][bad][:5]} or {k[exact][bad][:5]}"
    os_, om = oracle.OScene(sc), oracle.OMotions(sub)
    for m in np.nonzero(amb)[0]:
        assert lo[m] <= g[m] <= hi[m], (m, g[m], lo[m], hi[m])
        if g[m] != oracle.NONE:
            t, i, j = oracle.decode(g[m], sc.n_robots)
            assert oracle.pair_sep(sc, sub, int(m), t, i, j, os_, om) < oracle.BAND
    REPORT[f"ffc{tag}"] = {"M": int(mo.M), "compared_motions": int(sub.M), "exact_compared": int(exact.sum()),
                           "ambiguous_ffc": int(amb.sum()), "ambiguous_ffc_equal_oracle": int((g[amb] == k[amb]).sum()),
                           "ambiguous_states": int(na.sum()), "classified_states": int(ns.sum()),
                           "none_frac": float((k == oracle.NONE).mean())}
    return k, amb


# ------------------------------------------------------------------ K3 SpheresFK
@pytest.mark.parametrize("cfg", ["cfg1", "cfg2", "cfg3", "cfg4"])
def test_fk_centres_within_1e5(cfg):
    sc, mo, gs, wp, T = data(cfg, 512)
    rng = np.random.default_rng(0)
    Q = 400
    m = rng.integers(0, mo.M, Q)
    Tm = mo.T_array()
    t = (rng.uniform(size=Q) * Tm[m]).astype(np.int32)
    t[:20] = 0
    t[20:40] = Tm[m[20:40]] - 1
    xyz = gs.fk_states(wp, T, torch.from_numpy(m.astype(np.int64)).cuda(), torch.from_numpy(t).cuda()).cpu().numpy()
    os_, om = oracle.OScene(sc), oracle.OMotions(mo)
    err = 0.0
    for q in range(Q):
        ref = oracle.centres_at(sc, mo, int(m[q]), int(t[q]), os_, om)
        err = max(err, float(np.max(np.abs(xyz[q] - ref))))
    REPORT[f"fk_{cfg}"] = {"max_abs_err_m": err, "queries": Q}
    assert err <= 1e-5


def test_fk_out_of_range_rows_are_nan():
    sc, mo, gs, wp, T = data("cfg1")
    xyz = gs.fk_states(wp, T, torch.tensor([0, -1, 10 ** 9], dtype=torch.int64).cuda(),
                       torch.tensor([64, 0, 0], dtype=torch.int32).cuda()).cpu().numpy()
    assert np.isnan(xyz).all()


# ------------------------------------------------------------------ MotVal / FFC parity per config
@pytest.mark.parametrize("cfg,M", [("cfg1", None), ("cfg2", None), ("cfg3", 4096), ("cfg5", 8192)])
def test_motval_parity(cfg, M):
    sc, mo, gs, wp, T = data(cfg, M)
    for flags in (mrv.CHECK_ENV, 0):
        g = gs.motval(wp, T, flags)
        check_motval(sc, mo, g, check_env=bool(flags & mrv.CHECK_ENV), tag=f"_{cfg}_{flags}")


@pytest.mark.parametrize("cfg,M", [("cfg1", None), ("cfg2", None), ("cfg3", 2048), ("cfg4", 384), ("cfg5", 8192)])
def test_ffc_parity(cfg, M):
    sc, mo, gs, wp, T = data(cfg, M)
    check_ffc(sc, mo, gs.ffc(wp, T), tag=f"_{cfg}")


def test_full_size_cfg5_sampled_parity():
    """cfg5 at its full 2^20 motions in the bench launch configuration; sampled
    motions compared with the oracle one by one."""
    sc, mo, gs, wp, T = data("cfg5")
    gv = gs.motval(wp, T, mrv.CHECK_ENV).cpu().numpy()
    gk = mrv.keys_u32(gs.ffc(wp, T))
    rng = np.random.default_rng(5)
    idx = np.sort(rng.choice(mo.M, 3000, replace=False))
    idx = np.concatenate([idx, [0, mo.M - 1]])
    check_motval(sc, mo, gv, tag="_cfg5_full_sampled", idx=idx)
    check_ffc(sc, mo, gk, tag="_cfg5_full_sampled", idx=idx)
    REPORT["cfg5_full_sampled"] = {"M": int(mo.M), "sampled": int(idx.size), "valid_frac_gpu": float(gv.mean()),
                                   "conflict_free_frac_gpu": float((gk == oracle.NONE).mean())}


def test_full_size_cfg3_sampled_parity():
    """cfg3 at its full 65,536 motions (the bench's launch configuration: general W = 8
    instance, FFC level-2 rows); 2,000 sampled motions compared with the oracle."""
    sc, mo, gs, wp, T = data("cfg3")
    gv = gs.motval(wp, T, mrv.CHECK_ENV).cpu().numpy()
    gk = mrv.keys_u32(gs.ffc(wp, T))
    rng = np.random.default_rng(3)
    idx = np.concatenate([np.sort(rng.choice(mo.M, 2000, replace=False)), [0, mo.M - 1]])
    check_motval(sc, mo, gv, tag="_cfg3_full_sampled", idx=idx)
    check_ffc(sc, mo, gk, tag="_cfg3_full_sampled", idx=idx)
    REPORT["cfg3_full_sampled"] = {"M": int(mo.M), "sampled": int(idx.size), "valid_frac_gpu": float(gv.mean()),
                                   "conflict_free_frac_gpu": float((gk == oracle.NONE).mean())}


def test_cfg4_full_size_sampled():
    sc, mo, gs, wp, T = data("cfg4")
    gk = mrv.keys_u32(gs.ffc(wp, T))
    rng = np.random.default_rng(6)
    idx = np.sort(rng.choice(mo.M, 256, replace=False))
    check_ffc(sc, mo, gk, tag="_cfg4_full_sampled", idx=idx)
    tstar = np.where(gk == oracle.NONE, -1, gk // sc.n_pairs)
    REPORT["cfg4_full"] = {"none_frac": float((tstar < 0).mean()),
                           "t_ge_500_or_none": float(((tstar < 0) | (tstar >= 500)).mean()),
                           "deciles": np.percentile(np.where(tstar < 0, 1000, tstar), np.arange(0, 101, 10)).tolist()}


# ------------------------------------------------------------------ result neutrality
STRATS = [mrv.CHECK_ENV, mrv.CHECK_ENV | mrv.ORDER_HIERARCHICAL, mrv.CHECK_ENV | mrv.PACK_LINEAR,
          mrv.CHECK_ENV | mrv.ORDER_HIERARCHICAL | mrv.PACK_LINEAR, mrv.CHECK_ENV | mrv.DIAG_NO_EARLY_EXIT,
          mrv.CHECK_ENV | mrv.DIAG_NO_BROADPHASE]


@pytest.mark.parametrize("cfg", ["cfg1", "cfg2", "cfg3"])
def test_motval_flags_batch_widths_slices_bit_identical(cfg):
    sc, mo, gs, wp, T = data(cfg, 2048)
    ref = gs.motval(wp, T, mrv.CHECK_ENV).cpu()
    for f in STRATS:
        assert torch.equal(gs.motval(wp, T, f).cpu(), ref), f
    for W in (4, 8, 16, 32):
        assert torch.equal(gs.motval(wp, T, mrv.CHECK_ENV, states_per_batch=W).cpu(), ref), W
    for ns in (2, 3, 7):
        assert torch.equal(gs.motval(wp, T, mrv.CHECK_ENV, n_slices=ns).cpu(), ref), ns


@pytest.mark.parametrize("cfg", ["cfg1", "cfg2", "cfg4"])
def test_ffc_flags_batch_widths_slices_bit_identical(cfg):
    sc, mo, gs, wp, T = data(cfg, 256 if cfg == "cfg4" else 2048)
    ref = gs.ffc(wp, T).cpu()
    for f in (mrv.DIAG_NO_EARLY_EXIT, mrv.DIAG_NO_BROADPHASE):
        assert torch.equal(gs.ffc(wp, T, f).cpu(), ref), f
    for W in (4, 8, 16, 32):
        assert torch.equal(gs.ffc(wp, T, states_per_batch=W).cpu(), ref), W
    for ns in (2, 5, 32):
        assert torch.equal(gs.ffc(wp, T, n_slices=ns).cpu(), ref), ns


@pytest.mark.parametrize("cfg", ["cfg1", "cfg2"])
def test_motval_equals_not_ffc_without_env(cfg):
    """P13 on the GPU: MotVal(check_env=0) == (FFC == none), bit-exact."""
    sc, mo, gs, wp, T = data(cfg)
    v = gs.motval(wp, T, 0).cpu().numpy()
    k = mrv.keys_u32(gs.ffc(wp, T))
    assert np.array_equal(v.astype(bool), k == mrv.NO_CONFLICT)


def test_permutation_equivariance():
    sc, mo, gs, wp, T = data("cfg2")
    perm = torch.randperm(mo.M, generator=torch.Generator().manual_seed(3)).cuda()
    Tp = T[perm].contiguous() if not isinstance(T, int) else T
    v = gs.motval(wp, T).cpu()
    vp = gs.motval(wp[perm].contiguous(), Tp).cpu()
    assert torch.equal(v[perm.cpu()], vp)
    k = gs.ffc(wp, T).cpu()
    kp = gs.ffc(wp[perm].contiguous(), Tp).cpu()
    assert torch.equal(k[perm.cpu()], kp)


# ------------------------------------------------------------------ golden examples + edge cases
def run_small(sc, mo, flags=mrv.CHECK_ENV):
    gs = mrv.Scene(sc)
    wp, T = mrv.to_device(mo)
    return gs, gs.motval(wp, T, flags).cpu().numpy(), mrv.keys_u32(gs.ffc(wp, T))


def test_golden_crossing_and_contact_time():
    g = GOLD["crossing"]
    sc = scene([ball(g["radius"]), ball(g["radius"])])
    mo = motions([[[pose(p) for p in g["A"]], [pose(p) for p in g["B"]]]], g["T"])
    gs, v, k = run_small(sc, mo)
    assert bool(v[0]) == g["motval"] and gs.decode(k[0]) == tuple(g["ffc"])
    g = GOLD["contact_time"]
    sc = scene([ball(g["rA"]), ball(g["rB"])])
    mo = motions([[[pose(p) for p in g["A"]], [pose(g["B"]), pose(g["B"])]]], g["T"])
    gs, v, k = run_small(sc, mo)
    assert v[0] == 0 and gs.decode(k[0]) == tuple(g["ffc"])


def test_golden_three_robot_tie():
    g = GOLD["three_robot_tie"]
    T = g["T"]
    far = lambda k: [[5.0 * (k + 1), 5.0 * (t + 1), 0] for t in range(T)]  # noqa: E731
    A = [[0, 0, 0]] * T
    B = [([0, 0, 0] if t == 7 else p) for t, p in enumerate(far(1))]
    Cc = [([0, 0, 0] if t == 3 else p) for t, p in enumerate(far(2))]
    from helpers import knots_motion
    sc = scene([ball(g["radius"])] * 3)
    mo = gen.Motions(knots_motion([A, B, Cc]), None, T)
    gs, v, k = run_small(sc, mo)
    assert gs.decode(k[0]) == tuple(g["ffc"])


def test_golden_obstacle_predicates():
    g = GOLD["sphere_box"]
    sc = scene([ball(g["r"])], boxes=[g["box"]])
    mo = motions([[[pose(c["c"])]] for c in g["cases"]], 3)
    gs, v, k = run_small(sc, mo)
    assert [not bool(x) for x in v] == [c["hit"] for c in g["cases"]]
    assert (k == mrv.NO_CONFLICT).all()          # one robot: no pairs
    g = GOLD["sphere_sphere_obstacle"]
    for c in g["cases"]:
        sc = scene([ball(g["r"])], obs_spheres=[c["o"] + [g["R"]]])
        gs, v, k = run_small(sc, motions([[[pose([0, 0, 0])]]], 1))
        assert (not bool(v[0])) == c["hit"]


def test_edge_cases_empty_T1_K1():
    sc, mo = gen.make("cfg1", 16)
    gs = mrv.Scene(sc)
    wp, T = mrv.to_device(mo)
    empty = wp[:0].contiguous()
    assert gs.motval(empty, T).numel() == 0 and gs.ffc(empty, T).numel() == 0
    for TT in (1, 2, 3, 31, 32, 33):
        mo2 = gen.Motions(mo.waypoints, None, TT)
        g = gs.motval(wp, TT).cpu()
        check_motval(sc, mo2, g, tag=f"_T{TT}")
        check_ffc(sc, mo2, gs.ffc(wp, TT), tag=f"_T{TT}")
    mo1 = gen.Motions(np.ascontiguousarray(mo.waypoints[:, :, :1]), None, 40)
    wp1, _ = mrv.to_device(mo1)
    check_motval(sc, mo1, gs.motval(wp1, 40), tag="_K1")
    check_ffc(sc, mo1, gs.ffc(wp1, 40), tag="_K1")


def test_ragged_timesteps_and_many_knots():
    sc, mo = gen.make("cfg2", 512)
    rng = np.random.default_rng(9)
    Tr = rng.integers(1, 300, mo.M).astype(np.int32)
    mo2 = gen.Motions(mo.waypoints, Tr, 0)
    gs = mrv.Scene(sc)
    wp, T = mrv.to_device(mo2)
    check_motval(sc, mo2, gs.motval(wp, T), tag="_ragged")
    check_ffc(sc, mo2, gs.ffc(wp, T), tag="_ragged")


def test_ffc_range_error():
    sc, mo = gen.make("cfg4", 4)
    gs = mrv.Scene(sc)
    wp, _ = mrv.to_device(mo)
    with pytest.raises(mrv.MrvError) as e:
        gs.ffc(wp, (1 << 32) // 66 + 1)
    assert e.value.status == mrv.MRV_ERANGE


def test_knot_limit_refused():
    """K above MRV_MAX_KNOTS (2^20; the interpolation's exact-quotient bound) is refused
    before any launch; K = 2^20 itself runs."""
    import torch
    sc, _ = gen.make("cfg1", 4)
    gs = mrv.Scene(sc)
    for K, ok in [((1 << 20) + 1, False), (1 << 20, True)]:
        wp = torch.zeros((1, 2, K, 3), dtype=torch.float32, device="cuda")
        if ok:
            assert int(gs.motval(wp, 8, mrv.CHECK_ENV).item()) in (0, 1)
        else:
            with pytest.raises(mrv.MrvError) as e:
                gs.motval(wp, 8, mrv.CHECK_ENV)
            assert e.value.status == mrv.MRV_EUNSUPPORTED


def test_counters_and_effort():
    sc, mo, gs, wp, T = data("cfg2")
    cnt = torch.zeros(mrv.NUM_COUNTERS, dtype=torch.int64, device="cuda")
    eff = torch.zeros(mo.M, dtype=torch.int32, device="cuda")
    v = gs.motval(wp, T, mrv.CHECK_ENV | mrv.DIAG_NO_EARLY_EXIT, counters=cnt, effort=eff)
    c = cnt.cpu().numpy()
    assert c[0] == mo.total_states()                    # every state evaluated once
    assert c[1] == 4 * c[0] and c[2] == 28 * c[0]
    nb = (mo.T_array() + 7) // 8
    assert np.array_equal(eff.cpu().numpy(), nb)
    assert torch.equal(v.cpu(), gs.motval(wp, T).cpu())


def test_bounds_checked_build_runs_clean(tmp_path):
    """compute-sanitizer is closed on the GPU pool; instead a -DMRV_DEBUG_BOUNDS build
    traps on any out-of-range queue / table / smem index.  Run every entry point with it
    in a subprocess (a trap fails the subprocess, not this test process)."""
    import subprocess
    import sys
    from paper_2604_23960_b200 import build
    lib = str(tmp_path / "libmrv_debug.so")
    subprocess.check_call([build.NVCC] + [f for f in build.FLAGS if f not in ("-Xptxas", "-v")] +
                          ["-DMRV_DEBUG_BOUNDS", "-o", lib] + build.SRCS)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "tools", "sanitize_run.py")],
                       env=dict(os.environ, MRV_LIB_PATH=lib), capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "MRV_CHECK failed" not in r.stdout + r.stderr, r.stdout[-2000:] + r.stderr[-2000:]


# ------------------------------------------------------------------ f1: self-collision
@pytest.mark.parametrize("flags", [mrv.CHECK_SELF, mrv.CHECK_ENV | mrv.CHECK_SELF])
def test_self_collision_parity(flags):
    sc, mo, gs, wp, T = data("cfg2")
    g = gs.motval(wp, T, flags)
    v, amb, d = oracle.motval(sc, mo, check_env=bool(flags & mrv.CHECK_ENV), check_self=True)
    gn = g.cpu().numpy()
    assert np.array_equal(gn[~amb], v[~amb])
    REPORT[f"self_{flags}"] = {"M": int(mo.M), "ambiguous": int(amb.sum()), "valid_frac": float(v.mean())}
    for extra in (mrv.ORDER_HIERARCHICAL, mrv.PACK_LINEAR, mrv.DIAG_NO_EARLY_EXIT, mrv.DIAG_NO_BROADPHASE):
        assert torch.equal(gs.motval(wp, T, flags | extra), g), extra
    # self pairs never change FFC
    assert torch.equal(gs.ffc(wp, T, mrv.CHECK_SELF), gs.ffc(wp, T))


def test_self_collision_fold_closed_form():
    import math
    from test_oracle_pins import _fold_arm
    sc = scene([_fold_arm([[0, 2]]), ball(0.1)])
    wp = np.zeros((1, 2, 2, 7), np.float32)
    wp[0, 0, 1, :3] = [0.0, math.pi, 0.0]
    wp[0, 1, :, :] = pose([50.0, 50.0, 0.0])
    for T in (9, 33, 100):
        mo = gen.Motions(wp, None, T)
        gs, v, k = run_small(sc, mo, mrv.CHECK_SELF)
        assert v[0] == 0 and k[0] == mrv.NO_CONFLICT
        gs, v, k = run_small(sc, mo, mrv.CHECK_ENV)
        assert v[0] == 1
    wp2 = wp.copy()
    wp2[0, 0, 1, 1] = 2.0          # never folds past sqrt(2 + 2 cos 2) = 1.08 > 0.6
    gs, v, k = run_small(sc, gen.Motions(wp2, None, 33), mrv.CHECK_SELF)
    assert v[0] == 1


@pytest.mark.parametrize("arm", [0, 1, 2, 3])
def test_self_collision_single_arm_parity(arm):
    """One cfg2 arm alone (no robot-robot pairs): about half of the random motions
    self-collide, so the flags are discriminative."""
    sc2, mo2 = gen.make("cfg2", 2048)
    sc = gen.Scene([sc2.robots[arm]], sc2.obs_spheres, sc2.obs_boxes)
    mo = gen.Motions(np.ascontiguousarray(mo2.waypoints[:, arm:arm + 1]), mo2.n_timesteps, 0)
    gs = mrv.Scene(sc)
    wp, T = mrv.to_device(mo)
    for flags, env in ((mrv.CHECK_SELF, False), (mrv.CHECK_SELF | mrv.CHECK_ENV, True)):
        g = gs.motval(wp, T, flags).cpu().numpy()
        v, amb, d = oracle.motval(sc, mo, check_env=env, check_self=True)
        assert np.array_equal(g[~amb], v[~amb])
        assert 0.05 < v.mean() < 0.95 or env
        REPORT[f"self_arm{arm}_{flags}"] = {"valid_frac": float(v.mean()), "ambiguous": int(amb.sum())}


# ------------------------------------------------------------------ f4: time-split long horizons
@pytest.mark.parametrize("parts", [2, 3, 8])
def test_time_split_min_equals_full(parts):
    """Splitting T into disjoint windows (one per device in a multi-GPU time split) and
    reducing with MIN (FFC keys) / AND (MotVal flags) reproduces the full query."""
    from paper_2604_23960_b200 import dist as D
    sc, mo, gs, wp, T = data("cfg4", 384)
    full_k = mrv.keys_u32(gs.ffc(wp, T))
    full_v = gs.motval(wp, T).cpu().numpy()
    keys = np.full(mo.M, 0xFFFFFFFF, np.uint64)
    valid = np.ones(mo.M, np.uint8)
    for r in range(parts):
        t0, t1 = D.time_window(mo.fixed_timesteps, r, parts)
        keys = np.minimum(keys, mrv.keys_u32(gs.ffc(wp, T, t_begin=t0, t_end=t1)).astype(np.uint64))
        valid &= gs.motval(wp, T, t_begin=t0, t_end=t1).cpu().numpy()
        # a window's conflicts lie inside it
        kw = mrv.keys_u32(gs.ffc(wp, T, t_begin=t0, t_end=t1))
        tw = kw[kw != mrv.NO_CONFLICT] // sc.n_pairs
        assert ((tw >= t0) & (tw < t1)).all()
    assert np.array_equal(keys.astype(np.uint32), full_k)
    assert np.array_equal(valid, full_v)


def test_single_long_motion_many_warps():
    """One path set with a 100k-timestep horizon: its batches are spread over many warps
    (n_slices, atomicMin + skip rule) and the key equals the single-warp answer."""
    sc, mo = gen.make("cfg4", 2)
    wp = np.repeat(mo.waypoints[:1], 1, axis=0).copy()
    gs = mrv.Scene(sc)
    wpd = torch.from_numpy(np.ascontiguousarray(wp)).cuda()
    T = 100_000 // sc.n_pairs * sc.n_pairs // 66 * 60   # T * P < 2^32
    k_auto = mrv.keys_u32(gs.ffc(wpd, T))
    k_one = mrv.keys_u32(gs.ffc(wpd, T, n_slices=1))
    k_many = mrv.keys_u32(gs.ffc(wpd, T, n_slices=97))
    assert k_auto[0] == k_one[0] == k_many[0]
    ok, lo, hi, a = oracle.ffc(sc, gen.Motions(wp, None, T))
    if not a[0]:
        assert k_one[0] == ok[0]


# ------------------------------------------------------------------ f3: per-robot path lengths
def test_stay_at_goal_golden():
    sc = scene([ball(1.0), ball(1.0)])
    wp = np.asarray([[[pose([0, 0, 0]), pose([4, 0, 0])], [pose([10, 0, 0]), pose([0, 0, 0])]]], np.float32)
    mo = gen.Motions(wp, None, 0, np.array([[5, 11]], np.int32))
    gs, v, k = run_small(sc, mo)
    assert v[0] == 0 and gs.decode(k[0]) == (5, 0, 1)


@pytest.mark.parametrize("cfg", ["cfg2", "cfg4"])
def test_per_robot_lengths_parity(cfg):
    sc, mo0 = gen.make(cfg, 256)
    rng = np.random.default_rng(17)
    hi = 150 if cfg == "cfg2" else 1000
    rt = rng.integers(1, hi, size=(mo0.M, sc.n_robots)).astype(np.int32)
    mo = gen.Motions(mo0.waypoints, None, 0, rt)
    gs = mrv.Scene(sc)
    wp, T = mrv.to_device(mo)
    assert T.dim() == 2
    check_motval(sc, mo, gs.motval(wp, T, mrv.CHECK_ENV), check_env=True, tag=f"_rt_{cfg}")
    check_ffc(sc, mo, gs.ffc(wp, T), tag=f"_rt_{cfg}")
    # SpheresFK past a robot's own end = its goal pose
    m = torch.arange(32, dtype=torch.int64, device="cuda")
    t = torch.from_numpy((mo.T_array()[:32] - 1).astype(np.int32)).cuda()
    xyz = gs.fk_states(wp, T, m, t).cpu().numpy()
    for q in range(32):
        assert np.max(np.abs(xyz[q] - oracle.centres_at(sc, mo, q, int(mo.T_array()[q] - 1)))) <= 1e-5


# ------------------------------------------------------------------ f2: PP-ST-RRT MotVal variant
def _rank(i, j, n):
    return i * n - i * (i + 1) // 2 + (j - i - 1)


@pytest.mark.parametrize("focus,partners", [(2, (0, 1)), (0, (3,)), (3, (0, 1, 2))])
def test_focus_partner_variant(focus, partners):
    """Outer loop = the focus robot only (its obstacle + self checks), inner loop = its
    higher-priority partners only; every other robot is ignored.  Expected values come
    from the oracle's per-state tables restricted to those checks."""
    sc, mo, gs, wp, T = data("cfg2", 256)
    n = sc.n_robots
    flags = mrv.CHECK_ENV | mrv.CHECK_SELF
    g = gs.motval(wp, T, flags, focus=focus, partners=partners).cpu().numpy()
    gk = mrv.keys_u32(gs.ffc(wp, T, focus=focus, partners=partners))
    P = n * (n - 1) // 2
    cols = [_rank(min(focus, j), max(focus, j), n) for j in partners]
    checked = 0
    for m in range(mo.M):
        eh, es, ph, ps = oracle.state_tables(sc, mo, m, check_env=True, check_self=True)
        sep = np.minimum(es[:, focus], ps[:, cols].min(axis=1))
        hit = eh[:, focus] | ph[:, cols].any(axis=1)
        definite = (sep <= -oracle.BAND).any()
        amb = not definite and ((sep > -oracle.BAND) & (sep < oracle.BAND)).any()
        if not amb:
            assert g[m] == (0 if hit.any() else 1), m
            checked += 1
        # FFC restricted to the focus pairs
        keys = [t * P + c for t in range(ph.shape[0]) for c in sorted(cols) if ph[t, c]]
        pseps = ps[:, cols]
        if not ((pseps > -oracle.BAND) & (pseps < oracle.BAND)).any():
            assert gk[m] == (min(keys) if keys else mrv.NO_CONFLICT), m
    assert checked > 200
    # ignoring robots changes nothing for the included ones: the all-robot query is stricter
    assert (g >= gs.motval(wp, T, flags).cpu().numpy()).all()


def test_cuda_graph_capture_replay_arc_loop():
    """MotVal / FFC launches are stream-ordered and capturable: an ARC-style loop of
    repeated FFC calls on edited paths replays one CUDA graph."""
    import time
    sc, mo, gs, wp, T = data("cfg4", 64)
    wpe = wp.clone()
    out_k = torch.empty(mo.M, dtype=torch.int32, device="cuda")
    out_v = torch.empty(mo.M, dtype=torch.uint8, device="cuda")
    gs.ffc(wpe, T, out=out_k)
    gs.motval(wpe, T, out=out_v)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        gs.ffc(wpe, T, out=out_k)
        gs.motval(wpe, T, out=out_v)
    rng = torch.Generator(device="cuda").manual_seed(0)
    for it in range(4):
        # "replan" a window of one robot's path in every path set, then re-query
        wpe[:, 5, 3:6, :3] += 0.3 * torch.randn(mo.M, 3, 3, device="cuda", generator=rng)
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(out_k, gs.ffc(wpe, T))
        assert torch.equal(out_v, gs.motval(wpe, T))
    # host latency of a small call, direct vs graph (reported, not asserted)
    t0 = time.perf_counter()
    for _ in range(50):
        gs.ffc(wpe, T, out=out_k)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    for _ in range(50):
        g.replay()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    REPORT["arc_loop_64_pathsets_us_per_call"] = {"direct_ffc": 1e6 * (t1 - t0) / 50, "graph_ffc_motval": 1e6 * (t2 - t1) / 50}


@pytest.mark.parametrize("cfg,M,chunk", [("cfg5", 5000, 1024), ("cfg2", None, 700), ("cfg3", 3000, 0)])
def test_host_batch_pipeline_equals_device_calls(cfg, M, chunk):
    """mrv_run_host_batch (host inputs, chunks growing x4, copy/compute overlap through two
    staging buffers, each query's chunks alternating between two streams) gives
    bit-identical MotVal flags and FFC keys to the device-input calls, with both queries or
    one, device or pinned-host outputs, including a ragged last chunk, many chunks reusing
    the staging buffers and per-motion T from host memory."""
    import torch
    sc, mo = gen.make(cfg, M)
    gs = mrv.Scene(sc)
    wp, T = mrv.to_device(mo)
    ref_v = gs.motval(wp, T, mrv.CHECK_ENV).cpu()
    ref_k = gs.ffc(wp, T).cpu()
    wp_h = torch.from_numpy(np.ascontiguousarray(mo.waypoints)).pin_memory()
    T_h = T if isinstance(T, int) else T.cpu().pin_memory()
    for rep in range(2):   # the second call reuses the staging buffers
        v = torch.full((mo.M,), 7, dtype=torch.uint8, device="cuda")
        k = torch.full((mo.M,), 7, dtype=torch.int32, device="cuda")
        gs.run_host(wp_h, T_h, mrv.CHECK_ENV, v, 0, k, chunk=chunk)
        assert torch.equal(v.cpu(), ref_v), f"{cfg} MotVal rep {rep}"
        assert torch.equal(k.cpu(), ref_k), f"{cfg} FFC rep {rep}"
    only = torch.full((mo.M,), 7, dtype=torch.int32, device="cuda")
    gs.run_host(wp_h, T_h, 0, None, 0, only, chunk=chunk)   # FFC only
    assert torch.equal(only.cpu(), ref_k)
    only_v = torch.full((mo.M,), 7, dtype=torch.uint8, device="cuda")
    gs.run_host(wp_h, T_h, mrv.CHECK_ENV, only_v, 0, None, chunk=chunk)   # MotVal only
    assert torch.equal(only_v.cpu(), ref_v)
    # outputs in pinned host memory (each chunk's results copied back as its kernel ends),
    # also mixed with a device output; pageable host outputs are refused
    for rep in range(2):
        hv = torch.full((mo.M,), 7, dtype=torch.uint8).pin_memory()
        hk = torch.full((mo.M,), 7, dtype=torch.int32).pin_memory()
        gs.run_host(wp_h, T_h, mrv.CHECK_ENV, hv, 0, hk, chunk=chunk)
        torch.cuda.synchronize()
        assert torch.equal(hv, ref_v) and torch.equal(hk, ref_k), f"{cfg} host outputs rep {rep}"
    hk = torch.full((mo.M,), 7, dtype=torch.int32).pin_memory()
    dv = torch.full((mo.M,), 7, dtype=torch.uint8, device="cuda")
    gs.run_host(wp_h, T_h, mrv.CHECK_ENV, dv, 0, hk, chunk=chunk)
    torch.cuda.synchronize()
    assert torch.equal(dv.cpu(), ref_v) and torch.equal(hk, ref_k)
    with pytest.raises(mrv.MrvError) as e:
        gs.run_host(wp_h, T_h, mrv.CHECK_ENV, torch.zeros(mo.M, dtype=torch.uint8), 0, None, chunk=chunk)
    assert e.value.status == mrv.MRV_EINVAL


@pytest.mark.parametrize("parts", [2, 5])
def test_fused_motval_time_windows_and_widths(parts):
    """cfg2 (4 fast-DH arms, per-motion T) takes MotVal's fused FK + obstacle path: time
    windows reduced with AND, and every batch width / slice count, reproduce the full
    query bit for bit."""
    from paper_2604_23960_b200 import dist as D
    sc, mo, gs, wp, T = data("cfg2", 1024)
    full_v = gs.motval(wp, T).cpu().numpy()
    Tmax = int(mo.T_array().max())
    valid = np.ones(mo.M, np.uint8)
    for r in range(parts):
        t0, t1 = D.time_window(Tmax, r, parts)
        valid &= gs.motval(wp, T, t_begin=t0, t_end=t1).cpu().numpy()
    assert np.array_equal(valid, full_v)
    for W in (4, 8):
        for ns in (1, 3):
            v = gs.motval(wp, T, states_per_batch=W, n_slices=ns).cpu().numpy()
            assert np.array_equal(v, full_v), (W, ns)


def _long_chain(seed, dof=16, heavy_link=5, heavy=40):
    """A dof-joint planar-ish revolute chain (DH-form origins, a = 0.12 m, alternating
    alpha = +-pi/2), 4 spheres per link and `heavy` spheres on one link (more than one
    collision group of kMaxGroupSpheres = 32)."""
    rng = np.random.default_rng(seed)
    origins, sph, link = [], [], []
    for j in range(dof):
        if j == 0:
            origins.append(gen._affine(np.eye(3), np.zeros(3)))
        else:
            s = 1.0 if j % 2 else -1.0
            rx = np.array([[1.0, 0.0, 0.0], [0.0, 0.0, -s], [0.0, s, 0.0]])
            origins.append(gen._affine(rx, np.array([0.12, 0.0, 0.0])))
        n = heavy if j == heavy_link else 4
        for k in range(n):
            sph.append([(k + 0.5) / n * 0.12, rng.uniform(-0.01, 0.01), 0.0, rng.uniform(0.02, 0.04)])
            link.append(j)
    return gen.Robot(kind=gen.CHAIN, dof=dof, sphere_link=np.asarray(link, np.int32), sphere=gen._f32(sph),
                     joint_origin=gen._f32(origins), joint_type=np.zeros(dof, np.int32), base=None)


@pytest.mark.parametrize("case", ["64_bodies", "16dof_chains"])
def test_maximum_sizes_parity(case):
    """ABI limits: MRV_MAX_ROBOTS = 64 robots (2016 robot pairs, FK over several warp
    rounds), and MRV_MAX_DOF = 16 chains with a link carrying more spheres than one
    collision group holds; MotVal and FFC against the oracle."""
    rng = np.random.default_rng(7 if case == "64_bodies" else 8)
    if case == "64_bodies":
        robots = [ball(float(rng.uniform(0.15, 0.3))) for _ in range(64)]
        obs = np.concatenate([rng.uniform(0, 6, (6, 3)), rng.uniform(0.2, 0.5, (6, 1))], axis=1)
        c = rng.uniform(0, 6, (4, 3))
        h = rng.uniform(0.1, 0.4, (4, 3))
        sc = scene(robots, obs, np.concatenate([c - h, c + h], axis=1))
        M, K, T = 24, 3, 30
        pos = rng.uniform(0, 6, (M, 64, K, 3))
        q = np.zeros((M, 64, K, 4))
        q[..., 0] = 1.0
        wp = np.concatenate([pos, q], axis=-1).astype(np.float32)
    else:
        chains = [_long_chain(s) for s in (1, 2)]
        chains[1].base = gen._f32(gen._affine(np.eye(3), np.array([0.9, 0.0, 0.0])))
        sc = scene(chains + [ball(0.2)], np.array([[0.5, 0.8, 0.3, 0.2]], np.float32),
                   np.array([[0.2, -1.0, -0.2, 0.5, -0.6, 0.4]], np.float32))
        M, K, T = 48, 2, 40
        wp = np.zeros((M, 3, K, 16), np.float32)
        wp[:, :2, :, :] = rng.uniform(-1.5, 1.5, (M, 2, K, 16))
        wp[:, 2, :, :3] = rng.uniform(-0.5, 1.5, (M, K, 3))
        wp[:, 2, :, 3] = 1.0
    mo = motions(wp, T)
    gs = mrv.Scene(sc)
    wpd, Td = mrv.to_device(mo)
    check_motval(sc, mo, gs.motval(wpd, Td, mrv.CHECK_ENV), tag=f"_max_{case}")
    check_ffc(sc, mo, gs.ffc(wpd, Td), tag=f"_max_{case}")


def test_general_chains_prismatic_se2_se3_mixed_parity():
    """General joint origins, prismatic joints, a rotated base, and SE(2) + SE(3) bodies
    in one scene: SpheresFK within 1e-5 m, MotVal and FFC against the oracle."""
    rng = np.random.default_rng(31)
    se2 = gen.Robot(kind=gen.SE2, dof=3, sphere_link=np.zeros(3, np.int32),
                    sphere=gen._f32([[0.1, 0.0, 0.2, 0.08], [-0.1, 0.05, 0.2, 0.06], [0.0, -0.1, 0.25, 0.07]]))
    robots = [general_chain(rng, 9, (0.0, 0.0, 0.3)), general_chain(rng, 5, (1.3, 0.2, 0.3)), se2, ball(0.15)]
    obs = np.array([[0.9, 1.2, 0.4, 0.1], [-0.8, -1.1, 0.2, 0.15]], np.float32)
    sc = scene(robots, obs, np.array([[1.0, -1.3, 0.0, 1.2, -1.1, 0.3]], np.float32))
    M, K, T = 64, 3, 33
    wp = np.zeros((M, 4, K, 9), np.float32)
    wp[:, 0, :, :9] = rng.uniform(-1.5, 1.5, (M, K, 9))
    wp[:, 1, :, :5] = rng.uniform(-1.5, 1.5, (M, K, 5))
    wp[:, 2, :, :2] = rng.uniform(-2.0, 2.5, (M, K, 2))
    wp[:, 2, :, 2] = rng.uniform(-np.pi, np.pi, (M, K))
    for k in range(1, K):   # SE(2) theta pre-unwrapped (reading c.7)
        d = wp[:, 2, k, 2] - wp[:, 2, k - 1, 2]
        wp[:, 2, k, 2] -= (2 * np.pi * np.round(d / (2 * np.pi))).astype(np.float32)
    wp[:, 3, :, :3] = rng.uniform(-2.0, 2.5, (M, K, 3))
    q = rng.normal(size=(M, K, 4))
    q /= np.linalg.norm(q, axis=-1, keepdims=True)
    for k in range(1, K):
        q[:, k] *= np.sign(np.sum(q[:, k] * q[:, k - 1], axis=-1, keepdims=True) + 1e-30)
    wp[:, 3, :, 3:7] = q
    mo = motions(wp, T)
    gs = mrv.Scene(sc)
    wpd, Td = mrv.to_device(mo)
    import torch
    mq = torch.arange(M, dtype=torch.int64, device="cuda").repeat_interleave(3)
    tq = torch.tensor([0, 16, 29] * M, dtype=torch.int32, device="cuda")
    xyz = gs.fk_states(wpd, Td, mq, tq).cpu().numpy()
    err = max(np.max(np.abs(xyz[i] - oracle.centres_at(sc, mo, int(mq[i]), int(tq[i])))) for i in range(len(mq)))
    REPORT["fk_general_mixed"] = {"max_abs_err_m": float(err), "queries": int(len(mq))}
    assert err <= 1e-5
    check_motval(sc, mo, gs.motval(wpd, Td, mrv.CHECK_ENV), tag="_general_mixed")
    check_motval(sc, mo, gs.motval(wpd, Td, 0), check_env=False, tag="_general_mixed_noenv")
    check_ffc(sc, mo, gs.ffc(wpd, Td), tag="_general_mixed")


@pytest.mark.parametrize("flags", [mrv.CHECK_ENV, mrv.CHECK_ENV | mrv.DIAG_NO_EARLY_EXIT, mrv.CHECK_ENV | mrv.ORDER_HIERARCHICAL])
def test_dense_obstacles_queue_overflow_parity(flags):
    """cfg2's arms among 600 small clustered boxes and spheres: grid cells list dozens of
    obstacles, so the obstacle queue overflows and is flushed in the middle of the fused
    FK walk (and of the separate pass under the hierarchical order); results must match
    the oracle and not depend on the obstacle order."""
    rng = np.random.default_rng(41)
    sc0 = gen.scene_cfg2()
    lo, hi = np.array([0.9, -0.25, 0.7]), np.array([1.3, 0.25, 1.1])   # one dense cluster at the edge of reach
    c = rng.uniform(lo, hi, (400, 3))
    h = rng.uniform(0.003, 0.01, (400, 3))
    boxes = np.concatenate([c - h, c + h], axis=1).astype(np.float32)
    sp = np.concatenate([rng.uniform(lo, hi, (200, 3)), rng.uniform(0.003, 0.01, (200, 1))], axis=1).astype(np.float32)
    sc = gen.Scene(sc0.robots, sp, boxes)
    _, mo = gen.make("cfg2", 1024)
    gs = mrv.Scene(sc)
    wp, T = mrv.to_device(mo)
    g = gs.motval(wp, T, flags)
    v, _ = check_motval(sc, mo, g, tag=f"_dense_{flags}")
    v_free, _, _ = oracle.motval(gen.Scene(sc0.robots, np.zeros((0, 4), np.float32), np.zeros((0, 6), np.float32)), mo,
                              check_env=False)
    assert 0 < v.sum() < v_free.sum()   # the cluster invalidates some, not all, robot-robot-free motions
    perm = rng.permutation(len(boxes))
    sc_p = gen.Scene(sc0.robots, sp[::-1].copy(), boxes[perm])
    gp = mrv.Scene(sc_p).motval(wp, T, flags)
    assert torch_equal(g, gp)


def torch_equal(a, b):
    import torch
    return bool(torch.equal(a, b))


@pytest.mark.parametrize("K", [60, 120])
def test_many_knots_smem_and_global_waypoints(K):
    """Knot-dense paths for the four cfg2 arms: K = 60 keeps a motion's waypoint block
    in shared memory (fused MotVal path), K = 120 (4 x 120 x 7 floats > 8 KB) reads the
    waypoints from global memory (general path); both against the oracle."""
    rng = np.random.default_rng(50 + K)
    sc = gen.scene_cfg2()
    M, T = 96, 4 * K + 7
    steps = rng.uniform(-0.08, 0.08, (M, 4, K, 7))
    wp = np.clip(np.cumsum(steps, axis=2) + rng.uniform(-2.0, 2.0, (M, 4, 1, 7)), -2.9, 2.9).astype(np.float32)
    mo = motions(wp, T)
    gs = mrv.Scene(sc)
    wpd, Td = mrv.to_device(mo)
    check_motval(sc, mo, gs.motval(wpd, Td, mrv.CHECK_ENV), tag=f"_K{K}")
    check_ffc(sc, mo, gs.ffc(wpd, Td), tag=f"_K{K}")


def test_lean_instance_equals_general_path():
    """cfg5-class batches with production options run the lean W = 8 instance (launch
    options folded to constants, fixed-offset tables); an explicit whole-horizon time
    window (t_end = T, same semantics) forces the general instance: bit-identical."""
    sc, mo = gen.make("cfg5", 16384)
    gs = mrv.Scene(sc)
    wp, T = mrv.to_device(mo)
    import torch
    assert torch.equal(gs.motval(wp, T, mrv.CHECK_ENV), gs.motval(wp, T, mrv.CHECK_ENV, t_end=T))
    assert torch.equal(gs.ffc(wp, T), gs.ffc(wp, T, t_end=T))


@pytest.mark.parametrize("base_scale,radius_scale,y_off,prismatic",
                         [(0.0, 4.0, 0.0, False), (1.5, 1.0, 0.0, False), (1.0, 1.0, 0.02, False),
                          (1.0, 1.0, 0.0, True)])
def test_tiled_level1_dense_and_pruned(base_scale, radius_scale, y_off, prismatic):
    """The tiled level 1 (rr_stage_tile: lane (robot, state) tests its arm's 3 supergroups
    against the next arm's and the diagonal arm's) on cfg5's arms with
    (a) every base at the origin and 4x sphere radii: nearly all 54 supergroup pairs
    overlap at every state, so a batch's survivors overflow the 160-entry queue and take
    the three-pass path; (b) bases pushed out 1.5x: the static reach pruning drops
    supergroup pairs, which the per-role masks must carry.  Bit-identical to the segment
    walk (MRV_DIAG_NO_BROADPHASE), lean == general instance, and in parity with the oracle.  (c) spheres moved off the
    link x axes (the generic placement in level 2's neighbours: capsule prefilter, narrow
    phase) and (d) one arm with a prismatic joint (no fast-DH walk, generic level-2 bounds)
    keep the tiled level 1 on the general-scene paths."""
    import dataclasses
    sc0, mo = gen.make("cfg5", 6144)
    robots = []
    for i, r in enumerate(sc0.robots):
        b = r.base.copy()
        b[3] *= base_scale
        b[7] *= base_scale
        sp = r.sphere.copy()
        sp[:, 3] *= radius_scale
        sp[::2, 1] += y_off
        jt = r.joint_type.copy()
        if prismatic and i == 0:
            jt[3] = 1
        robots.append(dataclasses.replace(r, base=b, sphere=sp, joint_type=jt))
    sc = gen.Scene(robots, sc0.obs_spheres, sc0.obs_boxes)
    gs = mrv.Scene(sc)
    wp, T = mrv.to_device(mo)
    g = gs.ffc(wp, T)
    assert torch.equal(g, gs.ffc(wp, T, t_end=T))   # t_end = T: the general instance (full frames), same semantics
    assert torch.equal(g, gs.ffc(wp, T, mrv.DIAG_NO_BROADPHASE))   # the segment walk over every supergroup pair
    tag = f"_tile_{base_scale}_{radius_scale}_{y_off}_{int(prismatic)}"
    k, _ = check_ffc(sc, mo, g, tag=tag)
    assert 0 < int((k != oracle.NONE).sum()) < (mo.M if base_scale else mo.M + 1)
    # MotVal (the tiled level 1 under spread packing and in Alg. 1's loop) against the segment
    # walk over every supergroup pair (MRV_DIAG_NO_BROADPHASE)
    for f in (mrv.CHECK_ENV, 0):
        v = gs.motval(wp, T, f)
        assert torch.equal(v, gs.motval(wp, T, f | mrv.PACK_SEQUENTIAL))
        assert torch.equal(v, gs.motval(wp, T, f | mrv.DIAG_NO_BROADPHASE))
        assert torch.equal(v, gs.motval(wp, T, f | mrv.DIAG_NO_EARLY_EXIT))
    check_motval(sc, mo, v, check_env=False, tag=tag)


@pytest.mark.parametrize("M,T,K", [(5000, 128, 2), (12000, 128, 2), (6000, 1, 2), (6000, 2, 3), (6000, 37, 4),
                                   (12000, 300, 2)])
def test_spread_packing_equals_sequential(M, T, K):
    """Spread packing (run_spread: up to 8 motions per warp batch, golden-ratio timestep
    order, reading c.28) against Alg. 1's own batch loop (MRV_PACK_SEQUENTIAL) on
    cfg5's team: bit-identical over mixes of valid and invalid motions (valid ones are
    drawn from a larger pool and repeated, so warps drain with lanes shared between the
    survivors), T = 1, 2, odd, > 128, K > 2; M = 5000 runs the general instance, 12000 the
    lean one; plus oracle parity on a sample."""
    rng = np.random.default_rng(M + 7 * T + K)
    sc, pool = gen.make("cfg5", 4 * M)
    wp0 = pool.waypoints
    if K > 2:   # extra knots: interpolate start -> goal and jitter the interior ones
        a = np.linspace(0.0, 1.0, K, dtype=np.float32)[None, None, :, None]
        wp0 = wp0[:, :, :1] * (1 - a) + wp0[:, :, 1:2] * a
        wp0[:, :, 1:-1] += rng.normal(0.0, 0.05, wp0[:, :, 1:-1].shape).astype(np.float32)
    big = motions(wp0, T)
    gs = mrv.Scene(sc)
    wpb, Tb = mrv.to_device(big)
    v = gs.motval(wpb, Tb, mrv.CHECK_ENV | mrv.PACK_SEQUENTIAL).cpu().numpy()
    good, bad = np.nonzero(v == 1)[0], np.nonzero(v == 0)[0]
    if good.size and bad.size:
        pick = np.concatenate([rng.choice(good, M // 2), rng.choice(bad, M - M // 2, replace=False)])
    else:   # (T = 1: every motion is its valid start state)
        pick = rng.choice(good if good.size else bad, M, replace=False)
    rng.shuffle(pick)
    mo = big.subset(pick)
    wp, Tt = mrv.to_device(mo)
    a = gs.motval(wp, Tt, mrv.CHECK_ENV)
    b = gs.motval(wp, Tt, mrv.CHECK_ENV | mrv.PACK_SEQUENTIAL)
    assert torch.equal(a, b)
    assert 0.2 < float(a.float().mean()) < 0.8 or not (good.size and bad.size)
    cnt = torch.zeros(mrv.NUM_COUNTERS, dtype=torch.int64, device="cuda")
    assert torch.equal(gs.motval(wp, Tt, mrv.CHECK_ENV, counters=cnt), a)   # the counting instance
    idx = np.sort(rng.choice(M, 256, replace=False))
    check_motval(sc, mo, a, idx=idx, tag=f"_spread_{M}_{T}_{K}")


def test_spread_packing_per_motion_T():
    """Spread packing with per-motion T in device memory (each motion's own golden-ratio
    step, computed on the device): cfg2's ragged-T batch tiled to 12,288 motions, and
    random T in [1, 300] on cfg5's team, equal to Alg. 1's batch loop and to the oracle on
    a sample; a T < 1 leaves its motion valid and raises MRV_DEVERR_TIMESTEPS."""
    sc2, mo2 = gen.make("cfg2")
    rng = np.random.default_rng(29)
    tiled = gen.Motions(np.ascontiguousarray(np.tile(mo2.waypoints, (3, 1, 1, 1))),
                        np.ascontiguousarray(np.tile(mo2.n_timesteps, 3)), 0)
    sc5, mo5 = gen.make("cfg5", 8000)
    rand_T = gen.Motions(mo5.waypoints, rng.integers(1, 301, mo5.M).astype(np.int32), 0)
    for tag, sc, mo in (("cfg2x3", sc2, tiled), ("cfg5_randT", sc5, rand_T)):
        gs = mrv.Scene(sc)
        wp, T = mrv.to_device(mo)
        a = gs.motval(wp, T, mrv.CHECK_ENV)
        assert torch.equal(a, gs.motval(wp, T, mrv.CHECK_ENV | mrv.PACK_SEQUENTIAL)), tag
        idx = np.sort(rng.choice(mo.M, 200, replace=False))
        check_motval(sc, mo, a, idx=idx, tag=f"_spread_{tag}")
        gs.device_status()
        bad = T.clone()
        bad[11] = 0
        g = gs.motval(wp, bad, mrv.CHECK_ENV)
        assert int(g[11]) == 1 and gs.device_status() == mrv.DEVERR_TIMESTEPS
        keep = torch.arange(mo.M, device="cuda") != 11
        assert torch.equal(g[keep], a[keep])


@pytest.mark.parametrize("case", ["cfg3", "mixed"])
def test_spread_packing_general_path(case):
    """Spread packing on teams the fused walk does not cover -- cfg3's eight SE(3) bodies,
    and a random mix of DH arms, general chains, SE(2) and SE(3) bodies -- where the batch
    runs the separate FK, obstacle and robot-robot stages: equal to Alg. 1's batch loop and
    to the oracle on a sample, with and without obstacle checks."""
    from helpers import random_motions, random_scene
    rng = np.random.default_rng(41)
    if case == "cfg3":
        sc, mo = gen.make("cfg3", 12000)
    else:
        while True:
            sc = random_scene(rng)
            if sc.n_robots >= 3:
                break
        mo = random_motions(rng, sc, 6000)
    gs = mrv.Scene(sc)
    wp, T = mrv.to_device(mo)
    for flags in (mrv.CHECK_ENV, 0):
        a = gs.motval(wp, T, flags)
        assert torch.equal(a, gs.motval(wp, T, flags | mrv.PACK_SEQUENTIAL)), (case, flags)
        idx = np.sort(rng.choice(mo.M, 150, replace=False))
        check_motval(sc, mo, a, check_env=bool(flags), idx=idx, tag=f"_spread_general_{case}_{flags}")


@pytest.mark.parametrize("seed", [21, 22, 23])
def test_dh_first_link_folded_into_base(seed):
    """Fast-DH arms whose link 0 is itself a DH step Tz(d) Tx(a) Rx(alpha) on bases turned
    about z: the kernels fold that step into the base on the host (dhbase) and walk joint 0
    as Rz(q_0) alone, and centre the group bounds on the links' x axes.  MotVal (fused walk,
    spread packing; the hierarchical order's separate FK stage; Alg. 1's loop) and FFC
    (robot_fk_dh) against the oracle, which composes the 4x4 transforms as given."""
    from helpers import random_dh_team
    rng = np.random.default_rng(seed)
    n = int(rng.integers(3, 5))
    sc = random_dh_team(rng, n, 7, first_link_dh=True, rotated_bases=True)
    M, T = 6000, int(rng.integers(40, 130))
    wp = rng.uniform(-np.pi, np.pi, (M, n, 2, 7)).astype(np.float32) * np.float32(0.4)
    mo = motions(wp, T)
    gs = mrv.Scene(sc)
    wpd, Td = mrv.to_device(mo)
    a = gs.motval(wpd, Td, mrv.CHECK_ENV)
    assert torch.equal(a, gs.motval(wpd, Td, mrv.CHECK_ENV | mrv.PACK_SEQUENTIAL))
    assert torch.equal(a, gs.motval(wpd, Td, mrv.CHECK_ENV | mrv.ORDER_HIERARCHICAL))
    idx = np.sort(rng.choice(M, 150, replace=False))
    check_motval(sc, mo, a, idx=idx, tag=f"_dhfold_{seed}")
    check_ffc(sc, mo, gs.ffc(wpd, Td), idx=idx, tag=f"_dhfold_{seed}")
    q = torch.arange(16, dtype=torch.int64, device="cuda")
    xyz = gs.fk_states(wpd, Td, q, torch.full((16,), T // 3, dtype=torch.int32, device="cuda")).cpu().numpy()
    for i in range(16):
        assert np.max(np.abs(xyz[i] - oracle.centres_at(sc, mo, i, T // 3))) <= 1e-5


@pytest.mark.parametrize("seed", [11, 12, 13, 14])
def test_spread_packing_random_teams(seed):
    """Spread packing on random teams of 3-4 DH arms (same dof, bases ~1 m apart, random
    obstacles, valid and invalid motions; the general instance with p.spread): equal to Alg. 1's batch loop, and to
    the oracle on a sample."""
    from helpers import random_dh_team
    rng = np.random.default_rng(seed)
    n, dof = int(rng.integers(3, 5)), int(rng.integers(3, 8))
    sc = random_dh_team(rng, n, dof)
    M, K, T = 6000, int(rng.integers(2, 4)), int(rng.integers(20, 160))
    wp = rng.uniform(-np.pi, np.pi, (M, n, K, dof)).astype(np.float32) * np.float32(rng.uniform(0.1, 0.6))
    mo = motions(wp, T)
    gs = mrv.Scene(sc)
    wpd, Td = mrv.to_device(mo)
    a = gs.motval(wpd, Td, mrv.CHECK_ENV)
    assert torch.equal(a, gs.motval(wpd, Td, mrv.CHECK_ENV | mrv.PACK_SEQUENTIAL))
    idx = np.sort(rng.choice(M, 128, replace=False))
    check_motval(sc, mo, a, idx=idx, tag=f"_spread_random_{seed}")


def _rod(n=16, r=0.05, half=0.3):
    """An SE(3) body carrying n equal spheres along its local x axis (one capsule-shaped group)."""
    xs = np.linspace(-half, half, n)
    return gen.Robot(kind=gen.SE3, dof=7, sphere_link=np.zeros(n, np.int32),
                     sphere=gen._f32([[x, 0.0, 0.0, r] for x in xs]))


def test_capsule_prefilter_near_contact_parity():
    """The narrow phase's capsule prefilter (a cull) on its hard cases: rods
    of densely packed equal spheres held within +-3 mm of contact -- near-parallel
    (rotation <= 2 mrad), exactly collinear end to end (degenerate closest-point system),
    crossing -- plus a single-sphere body (degenerate capsule).  MotVal and FFC equal the
    oracle outside the ambiguity band, hits and misses both occur, and the counters show
    the prefilter ran and rejected group pairs."""
    from scipy.spatial.transform import Rotation
    rng = np.random.default_rng(77)
    robots = [_rod(), _rod(), _rod(), ball(0.05)]
    sc = scene(robots)
    M, K, T = 4096, 2, 8
    wp = np.zeros((M, 4, K, 7), np.float32)
    ident = np.array([1.0, 0.0, 0.0, 0.0])

    def quat(rotvec):
        x, y, z, w = Rotation.from_rotvec(rotvec).as_quat()
        return np.array([w, x, y, z])

    far = [(0.0, 0.0, 5.0), (0.0, 5.0, 0.0), (5.0, 0.0, 0.0)]
    for m in range(M):
        case = m % 4   # one near-contact pair per motion, the other bodies far away
        q = [pose(far[0], ident), pose(far[1], ident), pose(far[2], ident)]
        if case == 0:     # rod 1 near-parallel beside rod 0
            phi = rng.uniform(0, 2 * np.pi)
            d = 0.1 + rng.uniform(-3e-3, 3e-3)
            ax = rng.normal(size=3)
            ax /= np.linalg.norm(ax)
            q[0] = pose((rng.uniform(-0.4, 0.4), d * np.cos(phi), d * np.sin(phi)), quat(ax * rng.uniform(0.0, 2e-3)))
        elif case == 1:   # rod 2 collinear, end to end with rod 0 (den = 0)
            q[1] = pose((0.7 + rng.uniform(-3e-3, 3e-3), 0.0, 0.0), ident)
        elif case == 2:   # rod 2 crossing rod 0 at right angles, just below it
            q[1] = pose((rng.uniform(-0.25, 0.25), rng.uniform(-0.01, 0.01), -0.1 - rng.uniform(-3e-3, 3e-3)),
                        quat(np.array([0.0, 0.0, np.pi / 2])))
        else:             # single-sphere body just off rod 0's side (degenerate capsule)
            q[2] = pose((rng.choice([-0.3, -0.28, -0.26, 0.0, 0.3]), 0.0, -0.1 - rng.uniform(-3e-3, 3e-3)), ident)
        for k in range(K):   # nearly static: the knots differ by <= 0.2 mm
            wp[m, 0, k] = pose((0.0, 0.0, 0.0), ident)
            for r in range(3):
                wp[m, r + 1, k] = np.asarray(q[r], np.float32)
                wp[m, r + 1, k, :3] += rng.uniform(-1e-4, 1e-4, 3).astype(np.float32) * k
    mo = motions(wp, T)
    gs = mrv.Scene(sc)
    wpd, Td = mrv.to_device(mo)
    import torch
    cnt = torch.zeros(mrv.NUM_COUNTERS, dtype=torch.int64, device="cuda")
    keys = gs.ffc(wpd, Td, counters=cnt)
    c = dict(zip(mrv.COUNTER_NAMES, cnt.cpu().tolist()))
    k, amb = check_ffc(sc, mo, keys, tag="_capsule_near_contact")
    v, _ = check_motval(sc, mo, gs.motval(wpd, Td, 0), check_env=False, tag="_capsule_near_contact")
    none = float((k == oracle.NONE).mean())
    REPORT["capsule_near_contact"] = {"counters": c, "conflict_free_frac": none}
    assert 0.05 < none < 0.95 and 0.05 < float(v.mean()) < 0.95
    assert c["rr_capsule"] > 0 and c["rr_narrow"] < c["rr_capsule"] * 16 * 16


@pytest.mark.parametrize("seed", list(range(101, 117)))
def test_random_scenes_all_paths_parity(seed):
    """Randomised scenes over every robot kind, group size, obstacle mix, K, T, flag set
    (obstacles, self-collision, hierarchical / linear orders) and launch knob (batch width,
    warps per motion): MotVal and FFC against the oracle outside the ambiguity band,
    SpheresFK centres within 1e-5 m."""
    rng = np.random.default_rng(seed)
    for case in range(4):
        sc = random_scene(rng)
        mo = random_motions(rng, sc, 48)
        gs = mrv.Scene(sc)
        wpd, Td = mrv.to_device(mo)
        spb = int(rng.choice([0, 4, 8, 16, 32]))
        sl = int(rng.choice([0, 1, 3]))
        for flags in (mrv.CHECK_ENV, mrv.CHECK_ENV | mrv.CHECK_SELF, mrv.CHECK_ENV | mrv.ORDER_HIERARCHICAL,
                      mrv.CHECK_ENV | mrv.PACK_LINEAR, 0):
            env = (flags & mrv.CHECK_ENV) != 0
            g = gs.motval(wpd, Td, flags, states_per_batch=spb, n_slices=sl)
            v, amb, _ = oracle.motval(sc, mo, check_env=env, check_self=bool(flags & mrv.CHECK_SELF))
            gv = g.cpu().numpy()
            bad = np.nonzero((gv != v) & ~amb)[0]
            assert bad.size == 0, (seed, case, flags, spb, sl, bad[:5])
        check_ffc(sc, mo, gs.ffc(wpd, Td, states_per_batch=spb, n_slices=sl), tag=f"_random_{seed}_{case}")
        import torch
        T = mo.fixed_timesteps
        mq = torch.tensor(rng.integers(0, 48, 16), dtype=torch.int64, device="cuda")
        tq = torch.tensor(rng.integers(0, T, 16), dtype=torch.int32, device="cuda")
        xyz = gs.fk_states(wpd, Td, mq, tq).cpu().numpy()
        err = max(np.max(np.abs(xyz[i] - oracle.centres_at(sc, mo, int(mq[i]), int(tq[i])))) for i in range(16))
        assert err <= 1e-5, (seed, case, err)


def test_counting_launch_equals_production_cfg5():
    """bench.py's roofline counts the work of an untimed counting launch (the COUNT kernel
    instance); on the bench's own batch it must return exactly the production launch's
    results (so it evaluates the same states), and its counters must be self-consistent."""
    sc, mo, gs, wp, T = data("cfg5", 65536)
    for q in ("motval", "ffc"):
        cnt = torch.zeros(mrv.NUM_COUNTERS, dtype=torch.int64, device="cuda")
        if q == "motval":
            a = gs.motval(wp, T, mrv.CHECK_ENV)
            b = gs.motval(wp, T, mrv.CHECK_ENV, counters=cnt)
        else:
            a = gs.ffc(wp, T)
            b = gs.ffc(wp, T, counters=cnt)
        assert torch.equal(a, b), q
        c = dict(zip(mrv.COUNTER_NAMES, cnt.cpu().tolist()))
        assert c["robot_states"] == 4 * c["states"] and c["joints"] == 28 * c["states"], (q, c)
        assert 0 < c["states"] <= mo.total_states(), (q, c)
