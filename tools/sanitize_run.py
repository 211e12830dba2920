"""Small exercise of every entry point / flag / launch knob for compute-sanitizer runs."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2604_23960_b200 import gen, mrv  # noqa: E402

for cfg, M in (("cfg1", 64), ("cfg2", 96), ("cfg3", 48), ("cfg4", 8)):
    sc, mo = gen.make(cfg, M)
    gs = mrv.Scene(sc)
    wp, T = mrv.to_device(mo)
    for f in (mrv.CHECK_ENV, mrv.CHECK_ENV | mrv.ORDER_HIERARCHICAL, mrv.CHECK_ENV | mrv.PACK_LINEAR,
              mrv.CHECK_ENV | mrv.DIAG_NO_EARLY_EXIT, mrv.CHECK_ENV | mrv.DIAG_NO_BROADPHASE, 0):
        gs.motval(wp, T, f)
    for W in (4, 8, 16):
        for ns in (0, 3):
            gs.motval(wp, T, mrv.CHECK_ENV, states_per_batch=W, n_slices=ns)
            gs.ffc(wp, T, 0, states_per_batch=W, n_slices=ns)
    gs.ffc(wp, T, mrv.DIAG_NO_BROADPHASE)
    cnt = torch.zeros(mrv.NUM_COUNTERS, dtype=torch.int64, device="cuda")
    eff = torch.zeros(mo.M, dtype=torch.int32, device="cuda")
    gs.ffc(wp, T, counters=cnt, effort=eff)
    q = torch.arange(min(16, mo.M), dtype=torch.int64, device="cuda")
    gs.fk_states(wp, T, q, torch.zeros_like(q, dtype=torch.int32))
    # host-input pipeline (two chunks), time windows, the PP-ST-RRT variant, self-collision
    wp_h = torch.from_numpy(np.ascontiguousarray(mo.waypoints)).pin_memory()
    T_h = T if isinstance(T, int) else T.cpu().pin_memory()
    v = torch.empty(mo.M, dtype=torch.uint8, device="cuda")
    k = torch.empty(mo.M, dtype=torch.int32, device="cuda")
    gs.run_host(wp_h, T_h, mrv.CHECK_ENV, v, 0, k, chunk=max(1, mo.M // 2))
    gs.motval(wp, T, mrv.CHECK_ENV, t_begin=3, t_end=40)
    gs.ffc(wp, T, 0, t_begin=3, t_end=40)
    if sc.n_robots > 2:
        gs.motval(wp, T, mrv.CHECK_ENV, focus=1, partners=(0, 2))
        gs.ffc(wp, T, 0, focus=1, partners=(0, 2))
    gs.motval(wp, T, mrv.CHECK_ENV | mrv.CHECK_SELF)
    torch.cuda.synchronize()
    print(cfg, "ok", flush=True)

# a dense obstacle cluster: obstacle-queue overflow inside the fused FK walk
rng = np.random.default_rng(0)
sc0 = gen.scene_cfg2()
c = rng.uniform([0.9, -0.25, 0.7], [1.3, 0.25, 1.1], (500, 3))
boxes = np.concatenate([c - 0.01, c + 0.01], axis=1).astype(np.float32)
scd = gen.Scene(sc0.robots, np.zeros((0, 4), np.float32), boxes)
_, mo = gen.make("cfg2", 256)
gs = mrv.Scene(scd)
wp, T = mrv.to_device(mo)
for f in (mrv.CHECK_ENV, mrv.CHECK_ENV | mrv.DIAG_NO_EARLY_EXIT, mrv.CHECK_ENV | mrv.ORDER_HIERARCHICAL):
    gs.motval(wp, T, f)
torch.cuda.synchronize()
print("dense ok", flush=True)

# randomised scenes (the parity suite's generator, tests/helpers.py): every robot kind,
# group size, flag set and launch knob
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import helpers  # noqa: E402

rng = np.random.default_rng(7)
for case in range(12):
    sc = helpers.random_scene(rng)
    mo = helpers.random_motions(rng, sc, 32)
    gs = mrv.Scene(sc)
    wp, T = mrv.to_device(mo)
    for W in (0, 4, 16, 32):
        for f in (mrv.CHECK_ENV | mrv.CHECK_SELF, mrv.CHECK_ENV | mrv.ORDER_HIERARCHICAL | mrv.PACK_LINEAR,
                  mrv.CHECK_ENV | mrv.DIAG_NO_BROADPHASE):
            gs.motval(wp, T, f, states_per_batch=W, n_slices=2 if W == 16 else 0)
        gs.ffc(wp, T, 0, states_per_batch=W)
        gs.ffc(wp, T, mrv.DIAG_NO_BROADPHASE, states_per_batch=W)
    torch.cuda.synchronize()
print("random ok", flush=True)

# round 2: the PP-ST-RRT table path (every flag, width, slice count; partner subsets, a short
# horizon), the global-tail instance (thousands of obstacles), device-resident T errors,
# random warps per CTA
sc, paths, cand, t0 = gen.make_pp(512)
gs = mrv.Scene(sc)
pw, pT = mrv.to_device(paths)
cw, cT = mrv.to_device(cand)
t0d = torch.from_numpy(t0).cuda()
for H in (gen.PP_HORIZON, 700):
    table = gs.pp_table(pw, pT, gen.PP_PARTNERS, H)
    for f in (mrv.CHECK_ENV, 0, mrv.CHECK_ENV | mrv.CHECK_SELF, mrv.CHECK_ENV | mrv.ORDER_HIERARCHICAL,
              mrv.CHECK_ENV | mrv.DIAG_NO_EARLY_EXIT, mrv.CHECK_ENV | mrv.DIAG_NO_BROADPHASE):
        for W in (0, 8, 32):
            gs.pp_motval(cw, cT, t0d, gen.PP_FOCUS, gen.PP_PARTNERS, table, H, f, states_per_batch=W,
                         n_slices=2 if W == 8 else 0)
    gs.pp_motval(cw, cT, t0d, gen.PP_FOCUS, (1,), table, H, mrv.CHECK_ENV)
torch.cuda.synchronize()
print("pp ok", flush=True)
rng = np.random.default_rng(9)
c = rng.uniform([-1.8, -1.8, 0.0], [1.8, 1.8, 1.6], (9000, 3))
scg = gen.Scene(gen.scene_cfg2().robots, np.zeros((0, 4), np.float32),
                np.concatenate([c - 0.01, c + 0.01], axis=1).astype(np.float32))
_, mo = gen.make("cfg2", 64)
gs = mrv.Scene(scg)
wp, T = mrv.to_device(mo)
for f in (mrv.CHECK_ENV, mrv.CHECK_ENV | mrv.ORDER_HIERARCHICAL, mrv.CHECK_ENV | mrv.DIAG_NO_BROADPHASE):
    gs.motval(wp, T, f)
bad = T.clone()
bad[3] = 0
gs.motval(wp, bad, mrv.CHECK_ENV)
gs.ffc(wp, bad)
assert gs.device_status() == mrv.DEVERR_TIMESTEPS
for wpc in (1, 5, 11):
    gs.motval(wp, T, mrv.CHECK_ENV, warps_per_cta=wpc)
torch.cuda.synchronize()
print("tail / status / shapes ok", flush=True)

# MotVal spread packing (up to 8 motions per warp batch): the general instance (6000
# motions), the lean one (12000), the counting instance, and the lean global-tail scene
for M in (6000, 12000):
    sc, mo = gen.make("cfg5", M)
    gs = mrv.Scene(sc)
    wp, T = mrv.to_device(mo)
    gs.motval(wp, T, mrv.CHECK_ENV)
    gs.motval(wp, T, mrv.CHECK_ENV, counters=torch.zeros(mrv.NUM_COUNTERS, dtype=torch.int64, device="cuda"))
    gs.motval(wp, T, mrv.CHECK_ENV, warps_per_cta=7)
sc3, mo3 = gen.make("cfg3", 12000)   # the general (non-fused) stages under spread packing
gs3 = mrv.Scene(sc3)
wp3, T3 = mrv.to_device(mo3)
gs3.motval(wp3, T3, mrv.CHECK_ENV)
gs3.motval(wp3, T3, 0)
_, mo = gen.make("cfg5", 12000)
gs = mrv.Scene(scg)
wp, T = mrv.to_device(mo)
gs.motval(wp, T, mrv.CHECK_ENV)
torch.cuda.synchronize()
print("spread ok", flush=True)

# FFC's lean instance with the tiled level 1 (rr_stage_tile): cfg5 (12000 motions) and the
# same arms with every base at the origin and 4x radii (the queue-overflow passes)
import dataclasses  # noqa: E402
sc, mo = gen.make("cfg5", 12000)
robots = []
for r in sc.robots:
    b = r.base.copy()
    b[3] = b[7] = 0.0
    sp = r.sphere.copy()
    sp[:, 3] *= 4.0
    robots.append(dataclasses.replace(r, base=b, sphere=sp))
wp, T = mrv.to_device(mo)
for s in (sc, gen.Scene(robots, sc.obs_spheres, sc.obs_boxes)):
    gs = mrv.Scene(s)
    gs.ffc(wp, T)
    gs.ffc(wp, T, warps_per_cta=5)
torch.cuda.synchronize()
print("tiled level 1 ok", flush=True)
