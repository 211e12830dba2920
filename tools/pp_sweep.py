"""PP-ST-RRT variant: kernel time of mrv_pp_motval_batch vs batch width W on the pp5
workload (and the replicated-waypoint MRV_FOCUS path at its default W), CUDA events,
L2 flushed.  python tools/pp_sweep.py [motions]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2604_23960_b200 import gen, mrv  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
sc, paths, cand, t0 = gen.make_pp(M)
gs = mrv.Scene(sc)
pw, pT = mrv.to_device(paths)
table = gs.pp_table(pw, pT, gen.PP_PARTNERS, gen.PP_HORIZON)
cw, cT = mrv.to_device(cand)
t0d = torch.from_numpy(t0).cuda()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def timed(fn, reps=3):
    ts = []
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return min(ts)


ref = gs.pp_motval(cw, cT, t0d, gen.PP_FOCUS, gen.PP_PARTNERS, table, gen.PP_HORIZON, mrv.CHECK_ENV, states_per_batch=8)
for W in (8, 16, 32):
    for order in (0, mrv.ORDER_HIERARCHICAL):
        out = gs.pp_motval(cw, cT, t0d, gen.PP_FOCUS, gen.PP_PARTNERS, table, gen.PP_HORIZON, mrv.CHECK_ENV | order,
                           states_per_batch=W)
        assert torch.equal(out, ref)
        cnt = torch.zeros(mrv.NUM_COUNTERS, dtype=torch.int64, device="cuda")
        gs.pp_motval(cw, cT, t0d, gen.PP_FOCUS, gen.PP_PARTNERS, table, gen.PP_HORIZON, mrv.CHECK_ENV | order,
                     states_per_batch=W, counters=cnt)
        ms = timed(lambda: gs.pp_motval(cw, cT, t0d, gen.PP_FOCUS, gen.PP_PARTNERS, table, gen.PP_HORIZON,
                                        mrv.CHECK_ENV | order, states_per_batch=W))
        c = dict(zip(mrv.COUNTER_NAMES, cnt.cpu().tolist()))
        print(f"pp W={W} order={order}: {ms:.2f} ms, states {c['states'] / M:.1f}/motion, "
              f"rr_super {c['rr_super'] / max(1, c['states']):.1f}/state, table {c['table_bytes'] / max(1, c['states']):.0f} B/state",
              flush=True)
print("valid", ref.float().mean().item())
