"""End-to-end host pipeline vs device-only timing for several chunk sizes (cfg5)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2604_23960_b200 import gen, mrv
sc, mo = gen.make("cfg5")
gs = mrv.Scene(sc)
wp_h = torch.from_numpy(np.ascontiguousarray(mo.waypoints)).pin_memory()
wp = wp_h.cuda()
v = torch.empty(mo.M, dtype=torch.uint8, device="cuda"); k = torch.empty(mo.M, dtype=torch.int32, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
def t(fn, reps=3):
    fn(); torch.cuda.synchronize(); ts=[]
    for _ in range(reps):
        flush.zero_(); a=torch.cuda.Event(enable_timing=True); b=torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    return min(ts)
print("device", t(lambda: (gs.motval(wp, 128, mrv.CHECK_ENV, out=v), gs.ffc(wp, 128, out=k))))
print("copy+device", t(lambda: (wp.copy_(wp_h, non_blocking=True), gs.motval(wp, 128, mrv.CHECK_ENV, out=v), gs.ffc(wp, 128, out=k))))
print("h2d only", t(lambda: wp.copy_(wp_h, non_blocking=True)))
for c in (32768, 65536, 131072, 262144, 524288, 1048576, 2097152):
    print("host chunk", c, t(lambda: gs.run_host(wp_h, 128, mrv.CHECK_ENV, v, 0, k, chunk=c)))
hv = torch.empty(mo.M, dtype=torch.uint8).pin_memory(); hk = torch.empty(mo.M, dtype=torch.int32).pin_memory()
for c in (524288, 1048576, 2097152):
    print("host chunk, host outputs", c, t(lambda: gs.run_host(wp_h, 128, mrv.CHECK_ENV, hv, 0, hk, chunk=c)))
for c in (65536, 262144):
    def dev_chunks():
        for c0 in range(0, mo.M, c):
            gs.motval(wp[c0:c0+c], 128, mrv.CHECK_ENV, out=v[c0:c0+c]); gs.ffc(wp[c0:c0+c], 128, out=k[c0:c0+c])
    print("device chunked", c, t(dev_chunks))
