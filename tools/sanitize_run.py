"""Small exercise of every entry point / flag / launch knob for compute-sanitizer runs."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2604_23960_b200 import gen, mrv  # noqa: E402

for cfg, M in (("cfg1", 64), ("cfg2", 96), ("cfg3", 48), ("cfg4", 8)):
    sc, mo = gen.make(cfg, M)
    gs = mrv.Scene(sc)
    wp, T = mrv.to_device(mo)
    for f in (mrv.CHECK_ENV, mrv.CHECK_ENV | mrv.ORDER_HIERARCHICAL, mrv.CHECK_ENV | mrv.PACK_LINEAR,
              mrv.CHECK_ENV | mrv.DIAG_NO_EARLY_EXIT, mrv.CHECK_ENV | mrv.DIAG_NO_BROADPHASE, 0):
        gs.motval(wp, T, f)
    for W in (4, 8, 16):
        for ns in (0, 3):
            gs.motval(wp, T, mrv.CHECK_ENV, states_per_batch=W, n_slices=ns)
            gs.ffc(wp, T, 0, states_per_batch=W, n_slices=ns)
    gs.ffc(wp, T, mrv.DIAG_NO_BROADPHASE)
    cnt = torch.zeros(mrv.NUM_COUNTERS, dtype=torch.int64, device="cuda")
    eff = torch.zeros(mo.M, dtype=torch.int32, device="cuda")
    gs.ffc(wp, T, counters=cnt, effort=eff)
    q = torch.arange(min(16, mo.M), dtype=torch.int64, device="cuda")
    gs.fk_states(wp, T, q, torch.zeros_like(q, dtype=torch.int32))
    torch.cuda.synchronize()
    print(cfg, "ok", flush=True)
