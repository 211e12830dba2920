"""Work counters of one MotVal and one FFC launch (MRV_CNT_*), per evaluated composite state.

  python tools/counters.py [cfg5] [motions]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_23960_b200 import gen, mrv  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
M = int(sys.argv[2]) if len(sys.argv) > 2 else 65536
sc, mo = gen.make(cfg, M)
gs = mrv.Scene(sc)
wp, T = mrv.to_device(mo)
for q in ("motval", "motval-sequential", "ffc"):
    c = torch.zeros(mrv.NUM_COUNTERS, dtype=torch.int64, device="cuda")
    if q == "motval":
        gs.motval(wp, T, mrv.CHECK_ENV, counters=c)
    elif q == "motval-sequential":   # Alg. 1's own batch loop (no spread packing)
        gs.motval(wp, T, mrv.CHECK_ENV | mrv.PACK_SEQUENTIAL, counters=c)
    else:
        gs.ffc(wp, T, counters=c)
    c = c.cpu().tolist()
    st = max(c[0], 1)
    print(f"{cfg} {q}: " + ", ".join(f"{n}={v / st:.2f}" for n, v in zip(mrv.COUNTER_NAMES, c)) +
          f"  (states={c[0]}, {c[0] / mo.M:.2f} per motion)")
