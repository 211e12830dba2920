"""MotVal kernel time vs batch size on cfg5 (spread packing vs Alg. 1 batch loop): the fixed
(tail) part of a launch.  python tools/motval_size_scan.py"""
import sys; sys.path.insert(0,'.')
import torch
from paper_2604_23960_b200 import gen, mrv
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for M in (1 << 18, 1 << 19, 1 << 20, 1 << 21):
    sc, mo = gen.make("cfg5", M)
    gs = mrv.Scene(sc); wp, T = mrv.to_device(mo)
    res = []
    for f in (mrv.CHECK_ENV, mrv.CHECK_ENV | mrv.PACK_SEQUENTIAL):
        for _ in range(2): gs.motval(wp, T, f)
        ts = []
        for _ in range(5):
            flush.zero_(); a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            a.record(); gs.motval(wp, T, f); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
        res.append(sorted(ts)[2])
    print(M, "spread %.3f ms  sequential %.3f ms" % tuple(res), flush=True)
    del wp, T, gs
