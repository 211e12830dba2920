import sys, os
sys.path.insert(0, "/root/repo")
import torch
from paper_2604_23960_b200 import gen, mrv
cfg = sys.argv[1]
sc, mo = gen.make(cfg)
gs = mrv.Scene(sc)
wp, T = mrv.to_device(mo)
for _ in range(3): gs.ffc(wp, T)
torch.cuda.synchronize()
