"""Diagnostics for GPU-vs-oracle mismatches (test infrastructure; lives under tests/ because
only tests/, smoke() and bench.py's cpu_baseline leg may call oracle/).

  python tests/scripts/debug_parity.py [cfg] [M]
"""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import oracle
from paper_2604_23960_b200 import gen, mrv
cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
M = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
sc, mo = gen.make(cfg, M)
gs = mrv.Scene(sc)
wp, T = mrv.to_device(mo)
out = {}
for env in (1, 0):
    v, amb, d = oracle.motval(sc, mo, check_env=bool(env))
    for extra, name in ((0, "bp"), (mrv.DIAG_NO_BROADPHASE, "nobp"), (mrv.DIAG_NO_EARLY_EXIT, "noexit"),
                        (mrv.PACK_LINEAR, "linear")):
        g = gs.motval(wp, T, (mrv.CHECK_ENV if env else 0) | extra).cpu().numpy()
        out[f"env{env}_{name}"] = {"gpu1_or0": int(((g == 1) & (v == 0) & ~amb).sum()),
                                   "gpu0_or1": int(((g == 0) & (v == 1) & ~amb).sum()),
                                   "first": np.nonzero((g != v) & ~amb)[0][:5].tolist()}
k, lo, hi, a = oracle.ffc(sc, mo)
gk = mrv.keys_u32(gs.ffc(wp, T))
gk2 = mrv.keys_u32(gs.ffc(wp, T, mrv.DIAG_NO_BROADPHASE))
out["ffc"] = {"mism": int(((gk != k) & ~a).sum()), "mism_nobp": int(((gk2 != k) & ~a).sum()),
              "first": [(int(m), int(gk[m]), int(k[m])) for m in np.nonzero((gk != k) & ~a)[0][:8]]}
print(json.dumps(out, indent=1))
