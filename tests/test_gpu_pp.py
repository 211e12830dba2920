"""GPU parity of the PP-ST-RRT MotVal variant with shared fixed partner paths (SURVEY §8
f2; "the outer loop ... is replaced with only the current robot and the
inner loop ... iterates over only higher priority robots"): the partner table built once
by mrv_pp_build_table, candidates checked by mrv_pp_motval_batch, against the fp64
oracle's orc_pp_motval_batch on the same seeded inputs (bit-exact outside the 1e-4 m
ambiguity band), plus result-neutrality of every strategy / diagnostic flag and launch knob."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from helpers import ball, pose, scene  # noqa: E402
from paper_2604_23960_b200 import gen, mrv  # noqa: E402
from parity_report import REPORT  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2604_23960_b200 import build
    build.build()
    yield


_cache = {}


def pp_data(M=4096):
    if M not in _cache:
        sc, paths, cand, t0 = gen.make_pp(M)
        gs = mrv.Scene(sc)
        pw, pT = mrv.to_device(paths)
        table = gs.pp_table(pw, pT, gen.PP_PARTNERS, gen.PP_HORIZON)
        cw, cT = mrv.to_device(cand)
        _cache[M] = (sc, paths, cand, t0, gs, table, cw, cT, torch.from_numpy(t0).cuda())
    return _cache[M]


def check_pp(sc, paths, cand, t0, g, partners, horizon, tag, check_env=True, check_self=False, focus=gen.PP_FOCUS):
    v, amb, d = oracle.pp_motval(sc, focus, partners, cand, t0, paths, horizon, check_env=check_env,
                                 check_self=check_self)
    gv = g.cpu().numpy() if hasattr(g, "cpu") else np.asarray(g)
    bad = np.nonzero((gv != v) & ~amb)[0]
    REPORT[f"pp{tag}"] = {"compared_motions": int(cand.M), "exact_compared": int((~amb).sum()),
                          "ambiguous_motions": int(amb.sum()), "mismatch": int(bad.size), "valid_frac": float(v.mean())}
    assert bad.size == 0, f"PP mismatches at {bad[:10]}: gpu {gv[bad[:5]]} oracle {v[bad[:5]]}"
    return v


@pytest.mark.parametrize("flags", [mrv.CHECK_ENV, 0, mrv.CHECK_ENV | mrv.CHECK_SELF, mrv.CHECK_SELF])
def test_pp_parity(flags):
    sc, paths, cand, t0, gs, table, cw, cT, t0d = pp_data()
    g = gs.pp_motval(cw, cT, t0d, gen.PP_FOCUS, gen.PP_PARTNERS, table, gen.PP_HORIZON, flags)
    v = check_pp(sc, paths, cand, t0, g, gen.PP_PARTNERS, gen.PP_HORIZON, f"_{flags}",
                 check_env=bool(flags & mrv.CHECK_ENV), check_self=bool(flags & mrv.CHECK_SELF))
    assert 0.02 < v.mean() < 0.98


def test_pp_flags_widths_slices_bit_identical():
    sc, paths, cand, t0, gs, table, cw, cT, t0d = pp_data()
    ref = gs.pp_motval(cw, cT, t0d, gen.PP_FOCUS, gen.PP_PARTNERS, table, gen.PP_HORIZON, mrv.CHECK_ENV)
    for f in (mrv.ORDER_HIERARCHICAL, mrv.PACK_LINEAR, mrv.DIAG_NO_EARLY_EXIT, mrv.DIAG_NO_BROADPHASE,
              mrv.ORDER_HIERARCHICAL | mrv.PACK_LINEAR):
        g = gs.pp_motval(cw, cT, t0d, gen.PP_FOCUS, gen.PP_PARTNERS, table, gen.PP_HORIZON, mrv.CHECK_ENV | f)
        assert torch.equal(g, ref), f
    for W in (4, 8, 16, 32):
        g = gs.pp_motval(cw, cT, t0d, gen.PP_FOCUS, gen.PP_PARTNERS, table, gen.PP_HORIZON, mrv.CHECK_ENV,
                         states_per_batch=W)
        assert torch.equal(g, ref), W
    for ns in (2, 5):
        g = gs.pp_motval(cw, cT, t0d, gen.PP_FOCUS, gen.PP_PARTNERS, table, gen.PP_HORIZON, mrv.CHECK_ENV,
                         n_slices=ns)
        assert torch.equal(g, ref), ns
    cnt = torch.zeros(mrv.NUM_COUNTERS, dtype=torch.int64, device="cuda")
    g = gs.pp_motval(cw, cT, t0d, gen.PP_FOCUS, gen.PP_PARTNERS, table, gen.PP_HORIZON, mrv.CHECK_ENV, counters=cnt)
    assert torch.equal(g, ref)
    c = dict(zip(mrv.COUNTER_NAMES, cnt.cpu().tolist()))
    assert c["table_bytes"] >= 16 * 9 * c["states"] and c["robot_states"] == c["states"], c   # FK of the focus only
    REPORT["pp_counters"] = c


def test_pp_partner_subsets_and_horizon_clamp():
    """A table built for all three partners serves any subset; a horizon shorter than the
    candidates' windows holds the partners at the last row (oracle: min(t0 + t, H - 1))."""
    sc, paths, cand, t0, gs, table, cw, cT, t0d = pp_data(2048)
    for partners in ((1,), (0, 2), ()):
        g = gs.pp_motval(cw, cT, t0d, gen.PP_FOCUS, partners, table, gen.PP_HORIZON, mrv.CHECK_ENV)
        check_pp(sc, paths, cand, t0, g, partners, gen.PP_HORIZON, f"_partners_{len(partners)}_{sum(partners)}")
    H = 1500   # windows starting after 1500 - 128 are clamped; those beyond H see only the last row
    short = gs.pp_table(*mrv.to_device(paths), gen.PP_PARTNERS, H)
    g = gs.pp_motval(cw, cT, t0d, gen.PP_FOCUS, gen.PP_PARTNERS, short, H, mrv.CHECK_ENV)
    check_pp(sc, paths, cand, t0, g, gen.PP_PARTNERS, H, "_horizon1500")


def test_pp_closed_form_start_times():
    """The oracle pin's closed form on the GPU: a partner ball moving x = t_abs, a parked
    focus ball at x = 50 for T = 10: invalid iff 41 <= t_start <= 50."""
    sc = scene([ball(0.5), ball(0.5)])
    paths = gen.Motions(np.asarray([[[pose([0, 0, 0]), pose([100, 0, 0])], [pose([0, 0, 0])] * 2]], np.float32),
                        None, 0, np.array([[101, 1]], np.int32))
    gs = mrv.Scene(sc)
    table = gs.pp_table(*mrv.to_device(paths), [0], 101)
    starts = np.arange(0, 91, dtype=np.int32)
    cw = torch.from_numpy(np.tile(np.asarray([[[pose([50, 0, 0])]]], np.float32), (starts.size, 1, 1, 1))).cuda()
    g = gs.pp_motval(cw, 10, torch.from_numpy(starts).cuda(), 1, [0], table, 101, 0).cpu().numpy()
    assert np.array_equal(g.astype(bool), ~((starts >= 41) & (starts <= 50)))


def test_pp_argument_checks():
    sc, paths, cand, t0, gs, table, cw, cT, t0d = pp_data(2048)
    for bad in (dict(focus=4), dict(focus=-1), dict(horizon=0)):
        kw = dict(focus=gen.PP_FOCUS, horizon=gen.PP_HORIZON)
        kw.update(bad)
        with pytest.raises(mrv.MrvError) as e:
            gs.pp_motval(cw, cT, t0d, kw["focus"], gen.PP_PARTNERS, table, kw["horizon"], mrv.CHECK_ENV)
        assert e.value.status == mrv.MRV_EINVAL
    with pytest.raises(mrv.MrvError) as e:   # MRV_FOCUS is implied, not a flag of this call
        gs.pp_motval(cw, cT, t0d, gen.PP_FOCUS, gen.PP_PARTNERS, table, gen.PP_HORIZON, mrv.FOCUS)
    assert e.value.status == mrv.MRV_EINVAL
    # a negative start time (device-resident: checked by the kernel) -> valid + status bit
    gs.device_status()
    neg = t0d.clone()
    neg[5] = -3
    ref = gs.pp_motval(cw, cT, t0d, gen.PP_FOCUS, gen.PP_PARTNERS, table, gen.PP_HORIZON, mrv.CHECK_ENV)
    g = gs.pp_motval(cw, cT, neg, gen.PP_FOCUS, gen.PP_PARTNERS, table, gen.PP_HORIZON, mrv.CHECK_ENV)
    assert int(g[5]) == 1 and gs.device_status() == mrv.DEVERR_START
    keep = torch.arange(cw.shape[0], device="cuda") != 5
    assert torch.equal(g[keep], ref[keep])


@pytest.mark.parametrize("seed", [301, 302, 303, 304])
def test_pp_random_scenes(seed):
    """Random scenes of every robot kind (DH-form and general chains with prismatic joints
    and self pairs, SE(2), SE(3) bodies with 1-40 spheres), random focus robot and partner
    set, fixed paths of random lengths (stay at goal), candidates with random K, T and start
    times (some past the horizon): the table path against the oracle's PP variant, for
    obstacle / self / plain checks and several batch widths."""
    from helpers import random_motions, random_scene
    rng = np.random.default_rng(seed)
    for case in range(3):
        sc = random_scene(rng)
        n = sc.n_robots
        focus = int(rng.integers(0, n))
        partners = [r for r in range(n) if r != focus and rng.uniform() < 0.7]
        H = int(rng.integers(8, 200))
        pm = random_motions(rng, sc, 1)   # one motion of every robot: the fixed paths
        lens = rng.integers(1, H + 1, n).astype(np.int32)[None]
        paths = gen.Motions(pm.waypoints, None, 0, lens)
        cm = random_motions(rng, sc, 64)
        cand = gen.Motions(np.ascontiguousarray(cm.waypoints[:, focus:focus + 1]), None, cm.fixed_timesteps)
        t0 = rng.integers(0, H + 20, 64).astype(np.int32)
        gs = mrv.Scene(sc)
        table = gs.pp_table(*mrv.to_device(paths), partners, H)
        cw, cT = mrv.to_device(cand)
        t0d = torch.from_numpy(t0).cuda()
        for flags in (mrv.CHECK_ENV, mrv.CHECK_ENV | mrv.CHECK_SELF, 0):
            spb = int(rng.choice([0, 8, 16, 32]))
            g = gs.pp_motval(cw, cT, t0d, focus, partners, table, H, flags, states_per_batch=spb)
            check_pp(sc, paths, cand, t0, g, partners, H, f"_random_{seed}_{case}_{flags}",
                     check_env=bool(flags & mrv.CHECK_ENV), check_self=bool(flags & mrv.CHECK_SELF), focus=focus)


def test_pp_lean_instance_equals_general():
    """pp5-class launches with the production options run the lean W = 32 PP instance
    (options folded to constants); two slices per candidate, the counting instance and an
    explicit whole-horizon window force the general one: bit-identical, and the lean
    results match the oracle on a sample."""
    sc, paths, cand, t0, gs, table, cw, cT, t0d = pp_data(65536)
    args = (cw, cT, t0d, gen.PP_FOCUS, gen.PP_PARTNERS, table, gen.PP_HORIZON, mrv.CHECK_ENV)
    lean = gs.pp_motval(*args)
    assert torch.equal(lean, gs.pp_motval(*args, n_slices=2))
    cnt = torch.zeros(mrv.NUM_COUNTERS, dtype=torch.int64, device="cuda")
    assert torch.equal(lean, gs.pp_motval(*args, counters=cnt))
    rng = np.random.default_rng(5)
    idx = np.sort(rng.choice(cand.M, 400, replace=False))
    check_pp(sc, paths, cand.subset(idx), t0[idx], lean.cpu().numpy()[idx], gen.PP_PARTNERS, gen.PP_HORIZON,
             "_lean_sample")


def test_pp_full_size_sampled():
    """pp5 at its full 2^20 candidates in the bench's launch configuration (the W = 32
    instance, one warp per candidate, the fused focus walk); 2,002 sampled candidates against
    the oracle one by one."""
    sc, paths, cand, t0 = gen.make_pp()
    gs = mrv.Scene(sc)
    table = gs.pp_table(*mrv.to_device(paths), gen.PP_PARTNERS, gen.PP_HORIZON)
    cw, cT = mrv.to_device(cand)
    g = gs.pp_motval(cw, cT, torch.from_numpy(t0).cuda(), gen.PP_FOCUS, gen.PP_PARTNERS, table, gen.PP_HORIZON,
                     mrv.CHECK_ENV).cpu().numpy()
    rng = np.random.default_rng(55)
    idx = np.concatenate([np.sort(rng.choice(cand.M, 2000, replace=False)), [0, cand.M - 1]])
    v = check_pp(sc, paths, cand.subset(idx), t0[idx], g[idx], gen.PP_PARTNERS, gen.PP_HORIZON, "_full_sampled")
    REPORT["pp_full"] = {"M": int(cand.M), "sampled": int(idx.size), "valid_frac_gpu": float(g.mean()),
                                 "valid_frac_oracle_sample": float(v.mean())}
    gs.check_device()
