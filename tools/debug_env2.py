import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle
from paper_2604_23960_b200 import gen, mrv
sc, mo = gen.make("cfg2", 4096)
def qat(m, t):
    T = mo.T_array()[m]; u = np.float32(t / (T - 1))
    w0, w1 = mo.waypoints[m, :, 0], mo.waypoints[m, :, 1]
    return (w0 + u * (w1 - w0)).astype(np.float32)
for (m, t, r, box) in [(3939, 22, 3, 27), (16, 11, 3, 27), (19, 70, 1, 4), (40, 1, 1, 13), (98, 35, 0, 16)]:
    q = qat(m, t)
    print("case", m, t, "oracle", oracle.config_eval(sc, q[None])[1][0])
    for nm, scene, qq in [("full", sc, q), ("robot_only", gen.Scene([sc.robots[r]], sc.obs_spheres, sc.obs_boxes), q[r:r+1]),
                          ("robot+box", gen.Scene([sc.robots[r]], sc.obs_spheres, sc.obs_boxes[box:box+1]), q[r:r+1])]:
        gs = mrv.Scene(scene)
        wp = torch.from_numpy(np.ascontiguousarray(qq[None, :, None, :])).cuda()
        res = []
        for W in (4, 8, 16, 32):
            for f in (mrv.CHECK_ENV, mrv.CHECK_ENV | mrv.DIAG_NO_BROADPHASE):
                res.append(int(gs.motval(wp, 1, f, states_per_batch=W).item()))
        # replicate state 40 times as a T=40 motion (K=1)
        res2 = int(gs.motval(wp, 40, mrv.CHECK_ENV).item())
        print("  ", nm, "oracle", int(oracle.config_eval(scene, qq[None])[1][0]), "gpu valid W4..32 x (bp,nobp):", res, "T40:", res2)
