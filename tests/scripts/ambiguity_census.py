"""Ambiguity census (BASELINE.json north_star: "states whose oracle minimum signed sphere
separation is within 1e-4 m of zero ... are counted and reported"; SURVEY §8(c) "Counts
reported").  Full-scan fp64 oracle classification of the motion sets the GPU parity tests
compare, per config:

  * ambiguous states: states whose minimum signed separation over the query's pairs
    (robot-obstacle if check_env, and robot-robot) lies in (-1e-4, +1e-4) m -- every state of
    every motion, not only the prefix up to the first definite hit;
  * ambiguous motions (MotVal: no definite hit and >= 1 ambiguous state) and ambiguous FFC
    results (a (t, pair) at or before the answer inside the band) -- the cases the parity
    tests do not compare bit-exactly;
  * the exact-comparable counts.

Oracle only (no GPU).  Usage: python tests/scripts/ambiguity_census.py [out.json]
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
from paper_2604_23960_b200 import gen  # noqa: E402

# (config, motions compared by the GPU parity tests: a prefix, or a seeded sample of the
# full-size batch exactly as tests/test_gpu_parity.py draws it)
SETS = [
    ("cfg1", "all 256", lambda mo: np.arange(mo.M)),
    ("cfg2", "all 4096", lambda mo: np.arange(mo.M)),
    ("cfg3", "first 4096 (test_motval_parity)", lambda mo: np.arange(4096)),
    ("cfg3", "2002 sampled of 65,536 (test_full_size_cfg3_sampled_parity)",
     lambda mo: np.concatenate([np.sort(np.random.default_rng(3).choice(mo.M, 2000, replace=False)), [0, mo.M - 1]])),
    ("cfg4", "first 384 (test_ffc_parity)", lambda mo: np.arange(384)),
    ("cfg4", "256 sampled of 16,384 (test_cfg4_full_size_sampled)",
     lambda mo: np.sort(np.random.default_rng(6).choice(mo.M, 256, replace=False))),
    ("cfg5", "first 8192 (test_motval_parity)", lambda mo: np.arange(8192)),
    ("cfg5", "3002 sampled of 1,048,576 (test_full_size_cfg5_sampled_parity)",
     lambda mo: np.concatenate([np.sort(np.random.default_rng(5).choice(mo.M, 3000, replace=False)), [0, mo.M - 1]])),
]
QUERIES = {"cfg1": ("motval", "ffc"), "cfg2": ("motval", "ffc"), "cfg3": ("motval", "ffc"), "cfg4": ("ffc",),
           "cfg5": ("motval", "ffc")}


def census(cfg, what, pick, cache):
    if cfg not in cache:
        cache[cfg] = gen.make(cfg)
    sc, mo = cache[cfg]
    sub = mo.subset(pick(mo))
    rec = {"config": cfg, "motions": what, "M": int(sub.M), "composite_states": int(sub.T_array().sum()),
           "band_m": oracle.BAND}
    t0 = time.time()
    if "motval" in QUERIES[cfg]:
        v, amb, d, na, ns = oracle.motval_counts(sc, sub, check_env=True, full_scan=True)
        rec["motval"] = {"ambiguous_states": int(na.sum()), "classified_states": int(ns.sum()),
                         "ambiguous_motions": int(amb.sum()), "exact_comparable_motions": int((~amb).sum()),
                         "definite_hit_motions": int(d.sum()), "valid_motions": int(v.sum())}
    k, lo, hi, a, fa, fs = oracle.ffc_counts(sc, sub, full_scan=True)
    rec["ffc"] = {"ambiguous_states": int(fa.sum()), "classified_states": int(fs.sum()),
                  "ambiguous_results": int(a.sum()), "exact_comparable_results": int((~a).sum()),
                  "conflict_free": int((k == oracle.NONE).sum())}
    rec["oracle_s"] = round(time.time() - t0, 1)
    rec["threads"] = oracle.threads()
    return rec


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "ambiguity_census_r2.json")
    cache, recs = {}, []
    for cfg, what, pick in SETS:
        r = census(cfg, what, pick, cache)
        print(json.dumps(r), flush=True)
        recs.append(r)
    with open(out, "w") as f:
        json.dump({"what": __doc__.strip().splitlines()[0], "sets": recs}, f, indent=1)
    print(out)


if __name__ == "__main__":
    main()
