"""Kernel time vs batch size on cfg5 -- MotVal (spread packing and Alg. 1's batch loop) and
FFC -- to separate a launch's fixed (ramp / tail) part from its per-motion part.

  python tools/motval_size_scan.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_23960_b200 import gen, mrv  # noqa: E402

flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def timed(fn, reps=5):
    for _ in range(2):
        fn()
    ts = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return sorted(ts)[len(ts) // 2]


for M in (1 << 17, 1 << 18, 1 << 19, 1 << 20, 1 << 21):
    sc, mo = gen.make("cfg5", M)
    gs = mrv.Scene(sc)
    wp, T = mrv.to_device(mo)
    sp = timed(lambda: gs.motval(wp, T, mrv.CHECK_ENV))
    sq = timed(lambda: gs.motval(wp, T, mrv.CHECK_ENV | mrv.PACK_SEQUENTIAL))
    ff = timed(lambda: gs.ffc(wp, T))
    print(f"{M} motval spread {sp:.3f} ms  sequential {sq:.3f} ms  ffc {ff:.3f} ms", flush=True)
    del wp, T, gs
