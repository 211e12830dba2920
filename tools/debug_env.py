import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle
from paper_2604_23960_b200 import gen, mrv
sc, mo = gen.make("cfg2", 4096)
gs = mrv.Scene(sc); wp, T = mrv.to_device(mo)
v, amb, d = oracle.motval(sc, mo)
g = gs.motval(wp, T, mrv.CHECK_ENV | mrv.DIAG_NO_BROADPHASE).cpu().numpy()
gb = gs.motval(wp, T, mrv.CHECK_ENV).cpu().numpy()
bad = np.nonzero((g != v) & ~amb)[0]
badb = np.nonzero((gb != v) & ~amb)[0]
print("nobp bad", bad.tolist(), "bp bad", len(badb))
boxes = sc.obs_boxes.astype(np.float64)
offs = np.cumsum([0] + [r.n_spheres for r in sc.robots])
for m in list(bad[:4]) + list(badb[:6]):
    m = int(m)
    eh, es, ph, ps = oracle.state_tables(sc, mo, m)
    ts = np.nonzero(eh.any(1))[0]
    print("motion", m, "T", mo.T_array()[m], "env-hit t", ts[:10].tolist(), "rr-hit", np.nonzero(ph.any(1))[0][:5].tolist())
    for t in ts[:3]:
        xyz = gs.fk_states(wp, T, torch.tensor([m], dtype=torch.int64).cuda(), torch.tensor([t], dtype=torch.int32).cuda()).cpu().numpy()[0]
        ref = oracle.centres_at(sc, mo, m, int(t))
        for r in range(4):
            if not eh[t, r]: continue
            rb = sc.robots[r]
            for k in range(rb.n_spheres):
                c = ref[offs[r] + k]; rad = float(rb.sphere[k, 3])
                e = np.maximum(np.maximum(boxes[:, :3] - c, 0), c - boxes[:, 3:])
                dd = np.sqrt((e ** 2).sum(1)) - rad
                for bi in np.nonzero(dd < 0)[0]:
                    cg = xyz[offs[r] + k].astype(np.float32)
                    e32 = np.maximum(np.maximum(sc.obs_boxes[bi, :3] - cg, 0), cg - sc.obs_boxes[bi, 3:])
                    print(f"  t={t} r={r} k={k} link={rb.sphere_link[k]} box={bi} sep={dd[bi]:.5f} gpu_fp32_hit={(e32**2).sum() < np.float32(rad)**2} centre={c.round(4).tolist()} box={sc.obs_boxes[bi].round(3).tolist()}")
