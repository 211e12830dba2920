"""Write ``paper_2604_23960_b200/pools/<name>_accepted.npz``: the indices of the
candidate composite states (seeded streams in ``gen.candidate_block``) that the
ORACLE classifies as definitely free, i.e. min signed separation >= +1e-4 m over
all robot-obstacle and robot-robot sphere pairs (reading c.25: endpoints of
random motions are valid composite states, as planner edges are; the band is
BASELINE.json's 1e-4 m so acceptance never hinges on fp rounding).

Test infrastructure: this script calls only ``oracle/`` (plus the generator that
produces its inputs).  Usage: ``python oracle/make_pools.py [cfg2 cfg3 cfg5]``.
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import oracle  # noqa: E402
from paper_2604_23960_b200 import gen  # noqa: E402

SCENES = {"cfg2": gen.scene_cfg2, "cfg3": gen.scene_cfg3}


def make(name: str) -> str:
    stream, scene_name, count = gen.POOLS[name]
    scene = SCENES[scene_name]()
    acc = []
    b = 0
    while sum(a.size for a in acc) < count:
        q = gen.candidate_block(stream, b)
        ms, _ = oracle.config_eval(scene, q, check_env=True)
        acc.append(np.nonzero(ms >= oracle.BAND)[0].astype(np.int64) + b * gen.BLOCK)
        b += 1
        print(f"{name}: block {b}, accepted {sum(a.size for a in acc)}/{count}", flush=True)
    acc = np.concatenate(acc)[:count].astype(np.uint32)
    os.makedirs(gen.POOL_DIR, exist_ok=True)
    path = gen.pool_path(name)
    np.savez_compressed(path, accepted=acc, stream=np.array(stream), band=np.float64(oracle.BAND))
    return path


if __name__ == "__main__":
    for n in (sys.argv[1:] or list(gen.POOLS)):
        print(make(n))
