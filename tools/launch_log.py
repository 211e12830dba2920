import sys; sys.path.insert(0,'.')
import torch
from paper_2604_23960_b200 import gen, mrv
sc, mo = gen.make("cfg5", 65536)
gs = mrv.Scene(sc); wp, T = mrv.to_device(mo)
gs.motval(wp, T, mrv.CHECK_ENV); gs.motval(wp, T, mrv.CHECK_ENV | mrv.PACK_SEQUENTIAL); gs.ffc(wp, T)
torch.cuda.synchronize()
