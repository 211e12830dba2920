"""Print the launch configuration (instance, warps per CTA, shared memory, spread packing)
each query shape gets on a cfg5 and a pp5 slice: run with MRV_LAUNCH_LOG=1.

  MRV_LAUNCH_LOG=1 python tools/launch_log.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_23960_b200 import gen, mrv  # noqa: E402

sc, mo = gen.make("cfg5", 65536)
gs = mrv.Scene(sc)
wp, T = mrv.to_device(mo)
gs.motval(wp, T, mrv.CHECK_ENV)
gs.motval(wp, T, mrv.CHECK_ENV | mrv.PACK_SEQUENTIAL)
gs.ffc(wp, T)
psc, paths, cand, t0 = gen.make_pp(65536)
pgs = mrv.Scene(psc)
table = pgs.pp_table(*mrv.to_device(paths), gen.PP_PARTNERS, gen.PP_HORIZON)
cw, cT = mrv.to_device(cand)
t0d = torch.from_numpy(t0).cuda()
for f in (mrv.CHECK_ENV, mrv.CHECK_ENV | mrv.PACK_SEQUENTIAL):
    pgs.pp_motval(cw, cT, t0d, gen.PP_FOCUS, gen.PP_PARTNERS, table, gen.PP_HORIZON, f)
torch.cuda.synchronize()
