"""GPU tests of the contracts round 2 closed:

  * device-resident T that the launch cannot check (T < 1, FFC T * P >= 2^32 - 1) raises
    a bit in the scene's device status word and leaves that motion at valid / no conflict;
  * mrv_run_host_batch range-checks its host T array and validates both queries before
    anything is enqueued (outputs untouched on a synchronous error);
  * interpolation with (T - 1)(K - 1) >= 2^32 (64-bit knot arithmetic) against the oracle;
  * MRV_DIAG_NO_BROADPHASE disables every cull (grid, static reach pruning, capsules):
    the counters show the dense work and the results stay bit-identical;
  * MotVal scenes whose obstacle tables do not fit shared memory (tail read from global);
  * a race stress: warps per CTA, batch width and slice count randomised on dense scenes,
    outputs bit-identical.
Each compares the CUDA path (through the C ABI) with the fp64 oracle or with itself."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from helpers import motions  # noqa: E402
from paper_2604_23960_b200 import gen, mrv  # noqa: E402
from test_gpu_parity import check_ffc, check_motval  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2604_23960_b200 import build
    build.build()
    yield


# ------------------------------------------------------------------ device status word
def test_device_T_out_of_range_sets_status():
    sc, mo = gen.make("cfg4", 8)          # P = 66
    gs = mrv.Scene(sc)
    assert gs.device_status() == 0
    wp, _ = mrv.to_device(mo)
    T = np.full(8, 1000, np.int32)
    T[3] = (1 << 32) // 66 + 1           # t * P overflows uint32
    Td = torch.from_numpy(T).cuda()
    k = mrv.keys_u32(gs.ffc(wp, Td))
    assert k[3] == mrv.NO_CONFLICT
    assert gs.device_status() == mrv.DEVERR_RANGE
    assert gs.device_status() == 0      # cleared by the read
    good = np.array([0, 1, 2, 4, 5, 6, 7])
    check_ffc(sc, mo.subset(good), k[good], tag="_dev_range_rest")
    # MotVal has no key: the long T is legal there (no status bit)
    gs.motval(wp, torch.from_numpy(np.full(8, 50, np.int32)).cuda(), 0)
    assert gs.device_status() == 0
    T[3] = 1000
    T[5] = 0                              # T < 1
    Td = torch.from_numpy(T).cuda()
    v = gs.motval(wp, Td, 0).cpu().numpy()
    assert v[5] == 1 and gs.device_status() == mrv.DEVERR_TIMESTEPS
    assert mrv.keys_u32(gs.ffc(wp, Td))[5] == mrv.NO_CONFLICT
    with pytest.raises(mrv.MrvError) as e:
        gs.check_device()
    assert e.value.status == mrv.MRV_EINVAL
    # per-robot lengths: one robot with T = 0
    RT = np.full((8, sc.n_robots), 700, np.int32)
    RT[2, 7] = 0
    gs.ffc(wp, torch.from_numpy(RT).cuda())
    assert gs.device_status() == mrv.DEVERR_TIMESTEPS


def test_host_batch_checks_T_before_enqueue():
    sc, mo = gen.make("cfg2", 256)
    gs = mrv.Scene(sc)
    wp = torch.from_numpy(np.ascontiguousarray(mo.waypoints)).pin_memory()
    T = torch.from_numpy(np.ascontiguousarray(mo.n_timesteps)).pin_memory()
    out_v = torch.full((mo.M,), 7, dtype=torch.uint8, device="cuda")
    out_k = torch.full((mo.M,), 7, dtype=torch.int32, device="cuda")
    bad = T.clone()
    bad[100] = 0
    with pytest.raises(mrv.MrvError) as e:
        gs.run_host(wp, bad.pin_memory(), mrv.CHECK_ENV, out_v, 0, out_k)
    assert e.value.status == mrv.MRV_EINVAL
    bad = T.clone()
    bad[17] = (1 << 32) // 6 + 1          # FFC key overflow (P = 6)
    with pytest.raises(mrv.MrvError) as e:
        gs.run_host(wp, bad.pin_memory(), mrv.CHECK_ENV, out_v, 0, out_k)
    assert e.value.status == mrv.MRV_ERANGE
    with pytest.raises(mrv.MrvError) as e:   # MRV_FOCUS without launch options fails the dry run
        gs.run_host(wp, T, mrv.CHECK_ENV | mrv.FOCUS, out_v, 0, out_k)
    assert e.value.status == mrv.MRV_EINVAL
    torch.cuda.synchronize()
    assert (out_v == 7).all() and (out_k == 7).all()   # nothing was enqueued
    gs.run_host(wp, T, mrv.CHECK_ENV, out_v, 0, out_k)
    wpd, Td = mrv.to_device(mo)
    assert torch.equal(out_v, gs.motval(wpd, Td)) and torch.equal(out_k, gs.ffc(wpd, Td))


# ------------------------------------------------------------------ 64-bit knot arithmetic
def test_interpolation_beyond_2_32_knot_products():
    """K = 2^17 + 1 knots over T = 40,000 timesteps: t (K - 1) exceeds 2^32, so the
    interpolation takes the exact 64-bit quotient; MotVal / FFC / SpheresFK against the
    oracle (which divides in int64)."""
    rng = np.random.default_rng(64)
    sc, _ = gen.make("cfg1", 4)
    K, T = (1 << 17) + 1, 40000
    assert (T - 1) * (K - 1) >= 1 << 32
    wp = np.zeros((2, 2, K, 3), np.float32)
    for m in range(2):
        for r in range(2):
            xy = np.cumsum(rng.uniform(-0.01, 0.01, (K, 2)), axis=0) + rng.uniform(0.5, 3.5, 2)
            wp[m, r, :, :2] = np.clip(xy, 0.0, 4.0)
            wp[m, r, :, 2] = np.cumsum(rng.uniform(-0.02, 0.02, K))
    mo = motions(wp, T)
    gs = mrv.Scene(sc)
    wpd, Td = mrv.to_device(mo)
    check_motval(sc, mo, gs.motval(wpd, Td, mrv.CHECK_ENV), tag="_K2e17")
    check_motval(sc, mo, gs.motval(wpd, Td, 0), check_env=False, tag="_K2e17_noenv")
    check_ffc(sc, mo, gs.ffc(wpd, Td), tag="_K2e17")
    tq = np.array([0, 1, 12345, 30517, 39998, 39999], np.int32)
    mq = np.array([0, 1, 0, 1, 0, 1], np.int64)
    xyz = gs.fk_states(wpd, Td, torch.from_numpy(mq).cuda(), torch.from_numpy(tq).cuda()).cpu().numpy()
    for i in range(len(tq)):
        assert np.max(np.abs(xyz[i] - oracle.centres_at(sc, mo, int(mq[i]), int(tq[i])))) <= 1e-5


# ------------------------------------------------------------------ the diagnostic disables every cull
def test_no_broadphase_disables_every_cull():
    """Under MRV_DIAG_NO_BROADPHASE + NO_EARLY_EXIT on cfg2 every state tests every
    (group, obstacle) pair (no grid), every supergroup pair of every robot pair (no static
    reach pruning: 6 pairs x 3 x 3) and no capsule; results bit-identical to production."""
    sc, mo = gen.make("cfg2", 512)
    gs = mrv.Scene(sc)
    wp, T = mrv.to_device(mo)
    S = int(mo.total_states())
    for q in ("motval", "ffc"):
        c0 = torch.zeros(mrv.NUM_COUNTERS, dtype=torch.int64, device="cuda")
        c1 = torch.zeros(mrv.NUM_COUNTERS, dtype=torch.int64, device="cuda")
        if q == "motval":
            a = gs.motval(wp, T, mrv.CHECK_ENV | mrv.DIAG_NO_EARLY_EXIT, counters=c0)
            b = gs.motval(wp, T, mrv.CHECK_ENV | mrv.DIAG_NO_EARLY_EXIT | mrv.DIAG_NO_BROADPHASE, counters=c1)
        else:
            a = gs.ffc(wp, T, mrv.DIAG_NO_EARLY_EXIT, counters=c0)
            b = gs.ffc(wp, T, mrv.DIAG_NO_EARLY_EXIT | mrv.DIAG_NO_BROADPHASE, counters=c1)
        assert torch.equal(a, b), q
        c0 = dict(zip(mrv.COUNTER_NAMES, c0.cpu().tolist()))
        c1 = dict(zip(mrv.COUNTER_NAMES, c1.cpu().tolist()))
        assert c1["states"] == c0["states"] == S
        assert c1["rr_super"] == S * 6 * 9, (q, c1)
        assert c1["rr_capsule"] == 0 and c0["rr_capsule"] > 0
        assert c1["rr_broad"] == S * 6 * 7 * 7, (q, c1)   # every group pair of every supergroup pair
        if q == "motval":
            assert c1["env_broad"] == S * 28 * 32, c1      # 28 groups x 32 boxes, no grid
            assert c0["env_broad"] < c1["env_broad"] // 10


# ------------------------------------------------------------------ obstacle tables in global memory
def test_many_obstacles_tail_in_global_memory():
    """8,000 small boxes and 2,000 sphere obstacles (320 KB of obstacle records: more than a
    CTA's shared memory): MotVal reads the tail tables from global memory; parity with the
    oracle, and bit-identity with the diagnostic that tests every obstacle."""
    rng = np.random.default_rng(8000)
    sc0 = gen.scene_cfg2()
    c = rng.uniform([-1.8, -1.8, 0.0], [1.8, 1.8, 1.6], (8000, 3))
    h = rng.uniform(0.004, 0.02, (8000, 3))
    boxes = np.concatenate([c - h, c + h], axis=1).astype(np.float32)
    sp = np.concatenate([rng.uniform([-1.8, -1.8, 0.0], [1.8, 1.8, 1.6], (2000, 3)),
                         rng.uniform(0.004, 0.02, (2000, 1))], axis=1).astype(np.float32)
    sc = gen.Scene(sc0.robots, sp, boxes)
    _, mo = gen.make("cfg2", 48)
    mo = gen.Motions(mo.waypoints, np.minimum(mo.n_timesteps, 40).astype(np.int32), 0)
    gs = mrv.Scene(sc)
    wp, T = mrv.to_device(mo)
    g = gs.motval(wp, T, mrv.CHECK_ENV)
    check_motval(sc, mo, g, tag="_10k_obstacles")
    assert torch.equal(g, gs.motval(wp, T, mrv.CHECK_ENV | mrv.DIAG_NO_BROADPHASE))
    assert torch.equal(g, gs.motval(wp, T, mrv.CHECK_ENV | mrv.ORDER_HIERARCHICAL))


# ------------------------------------------------------------------ race stress
@pytest.mark.parametrize("cfg,M", [("cfg5", 6000), ("cfg5", 12000), ("cfg3", 12000)])
def test_race_stress_spread_packing(cfg, M):
    """Spread packing (8 motions per warp batch, slots refilled mid-batch-loop, per-lane
    waypoint slots) under randomised warps per CTA: bit-identical to Alg. 1's batch loop
    (cfg5 M = 6000: the general instance; 12000: the lean one; cfg3: the separate FK /
    obstacle / robot-robot stages)."""
    rng = np.random.default_rng(M)
    sc, mo = gen.make(cfg, M)
    gs = mrv.Scene(sc)
    wp, T = mrv.to_device(mo)
    ref = gs.motval(wp, T, mrv.CHECK_ENV | mrv.PACK_SEQUENTIAL)
    assert torch.equal(gs.motval(wp, T, mrv.CHECK_ENV), ref)
    for wpc in rng.integers(1, 17, 8):
        try:
            v = gs.motval(wp, T, mrv.CHECK_ENV, warps_per_cta=int(wpc))
        except mrv.MrvError as e:
            assert e.status == mrv.MRV_EUNSUPPORTED
        else:
            assert torch.equal(v, ref), int(wpc)


@pytest.mark.parametrize("cfg", ["cfg2", "cfg3"])
def test_race_stress_random_launch_shapes(cfg):
    """compute-sanitizer's racecheck is unavailable on the pool: instead the same batch is
    run under randomised warps per CTA (1..16/18), batch widths and slice counts, on a
    dense scene where queues overflow and warps share motions; every output must be
    bit-identical (a missing __syncwarp or a cross-warp smem overlap shows up as a
    difference under some launch shape)."""
    rng = np.random.default_rng(7 if cfg == "cfg2" else 8)
    sc, mo = gen.make(cfg, 1024)
    gs = mrv.Scene(sc)
    wp, T = mrv.to_device(mo)
    ref_v = gs.motval(wp, T, mrv.CHECK_ENV)
    ref_k = gs.ffc(wp, T)
    for _ in range(24):
        wpc = int(rng.integers(1, 17))
        spb = int(rng.choice([0, 4, 8, 16, 32]))
        ns = int(rng.choice([0, 1, 2, 5]))
        flags = int(rng.choice([mrv.CHECK_ENV, mrv.CHECK_ENV | mrv.ORDER_HIERARCHICAL,
                                mrv.CHECK_ENV | mrv.DIAG_NO_EARLY_EXIT]))
        try:
            v = gs.motval(wp, T, flags, warps_per_cta=wpc, states_per_batch=spb, n_slices=ns)
        except mrv.MrvError as e:      # that many warps of this width do not fit one CTA
            assert e.status == mrv.MRV_EUNSUPPORTED
        else:
            assert torch.equal(v, ref_v), (wpc, spb, ns, flags)
        wpc_f = int(rng.integers(1, 19))
        try:
            k = gs.ffc(wp, T, warps_per_cta=wpc_f, states_per_batch=spb, n_slices=ns)
        except mrv.MrvError as e:
            assert e.status == mrv.MRV_EUNSUPPORTED
        else:
            assert torch.equal(k, ref_k), (wpc_f, spb, ns)


def test_c_example_runs():
    """examples/mrv_example.c on the GPU: a plain-C program creates a scene, runs MotVal and
    FFC on device buffers it allocated itself and decodes the keys (closed-form expected
    results: first conflicts at t = 5, one valid motion)."""
    import subprocess
    from paper_2604_23960_b200 import build
    exe = build.build_example()
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and "example: ok" in r.stdout, r.stdout + r.stderr


def test_compact_frames_warps_per_cta():
    """FFC's lean instance on cfg5 stores compact link frames (6 words per link and state)
    and may run up to 20 warps per CTA: the same keys at every CTA size; full-frame launches
    (the general instance: an explicit time window) refuse more than 18 warps."""
    sc, mo = gen.make("cfg5", 6144)
    gs = mrv.Scene(sc)
    wp, T = mrv.to_device(mo)
    ref = gs.ffc(wp, T)
    assert torch.equal(ref, gs.ffc(wp, T, t_end=T))
    for wpc in (1, 7, 18, 19, 20):
        assert torch.equal(gs.ffc(wp, T, warps_per_cta=wpc), ref), wpc
    for wpc in (19, 20):
        with pytest.raises(mrv.MrvError) as e:
            gs.ffc(wp, T, warps_per_cta=wpc, t_end=T)
        assert e.value.status == mrv.MRV_EUNSUPPORTED
    with pytest.raises(mrv.MrvError) as e:
        gs.ffc(wp, T, warps_per_cta=21)
    assert e.value.status == mrv.MRV_EINVAL
