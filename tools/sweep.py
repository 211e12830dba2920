"""Time MotVal / FFC kernels for a few launch knobs (CUDA events, L2 flushed between runs)."""
import sys, os, json, itertools
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2604_23960_b200 import gen, mrv
cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
M = int(sys.argv[2]) if len(sys.argv) > 2 else 262144
sc, mo = gen.make(cfg, M)
gs = mrv.Scene(sc); wp, T = mrv.to_device(mo)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
def timeit(fn, reps=3):
    fn(); torch.cuda.synchronize(); ts = []
    for _ in range(reps):
        flush.zero_(); a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    return min(ts)
ref_v = gs.motval(wp, T).clone(); ref_k = gs.ffc(wp, T).clone()
for W in (4, 8, 16):
    for name, f in (("combined", mrv.CHECK_ENV), ("hier", mrv.CHECK_ENV | mrv.ORDER_HIERARCHICAL), ("noexit", mrv.CHECK_ENV | mrv.DIAG_NO_EARLY_EXIT)):
        try:
            t = timeit(lambda: gs.motval(wp, T, f, states_per_batch=W))
            ok = torch.equal(gs.motval(wp, T, f, states_per_batch=W), ref_v)
            print(f"motval W={W:2d} {name:9s} {t:8.3f} ms ok={ok}", flush=True)
        except Exception as e: print("motval", W, name, e)
    for name, f in (("ffc", 0), ("noexit", mrv.DIAG_NO_EARLY_EXIT)):
        try:
            t = timeit(lambda: gs.ffc(wp, T, f, states_per_batch=W))
            ok = torch.equal(gs.ffc(wp, T, f, states_per_batch=W), ref_k)
            print(f"ffc    W={W:2d} {name:9s} {t:8.3f} ms ok={ok}", flush=True)
        except Exception as e: print("ffc", W, name, e)
