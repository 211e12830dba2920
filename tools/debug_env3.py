import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle
from paper_2604_23960_b200 import gen, mrv
sc, mo = gen.make("cfg2", 4096)
m, t, r, box = 3939, 22, 3, 27
T = mo.T_array()[m]; u = np.float32(t / (T - 1))
q = (mo.waypoints[m, :, 0] + u * (mo.waypoints[m, :, 1] - mo.waypoints[m, :, 0])).astype(np.float32)
scene = gen.Scene([sc.robots[r]], sc.obs_spheres, sc.obs_boxes[box:box+1])
gs = mrv.Scene(scene)
wp = torch.from_numpy(np.ascontiguousarray(q[None, r:r+1, None, :])).cuda()
for TT in (1, 2, 3, 8, 9, 40):
    for f in (mrv.CHECK_ENV, mrv.CHECK_ENV | mrv.DIAG_NO_BROADPHASE | mrv.DIAG_NO_EARLY_EXIT):
        c = torch.zeros(8, dtype=torch.int64, device="cuda")
        v = gs.motval(wp, TT, f, counters=c, states_per_batch=8).item()
        print("T", TT, "flags", f, "valid", v, dict(zip(mrv.COUNTER_NAMES, c.cpu().tolist())))
# slot dependence: K=8 knots, T=8 -> t = knot; only knot j at the colliding pose, others far away
far = q[r].copy(); far[0] += 2.5
for j in range(8):
    w = np.stack([q[r] if k == j else far for k in range(8)])[None, None]
    wpj = torch.from_numpy(np.ascontiguousarray(w)).cuda()
    mj = gen.Motions(w.astype(np.float32), None, 8)
    print("slot", j, "oracle valid", oracle.motval(scene, mj)[0][0], "gpu rake", gs.motval(wpj, 8, mrv.CHECK_ENV, states_per_batch=8).item(),
          "gpu linear", gs.motval(wpj, 8, mrv.CHECK_ENV | mrv.PACK_LINEAR, states_per_batch=8).item())
