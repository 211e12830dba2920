"""Fig. 7-shaped MotVal ablation on B200.

For teams of 2/4/8/16 synthetic 7-DOF arms in two facing rows, with and without box
obstacles, 1000 random motions each: the four MotVal strategies (combined /
hierarchical ordering x rake / linear packing; self-collision is
part of the robot-obstacle check) -- validation effort (share of the
CC work a full evaluation would do that was done before early termination, from the
kernel's work counters) and kernel time, plus the valid fraction.  Writes
profiles/<name>_fig7_ablation.{json,md}.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2604_23960_b200 import gen, mrv  # noqa: E402

STRATS = {"combined-linear": mrv.PACK_LINEAR, "combined-rake": 0,
          "hierarchical-linear": mrv.ORDER_HIERARCHICAL | mrv.PACK_LINEAR, "hierarchical-rake": mrv.ORDER_HIERARCHICAL}


def cc_work(c):
    # CC calls = broad + narrow tests of every kind (obstacles, self pairs, robot pairs)
    return sum(c[k] for k in ("env_broad", "env_narrow", "self_broad", "rr_super", "rr_broad", "rr_narrow"))


def run(name="r1", M=1000, reps=5):
    rows = []
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for n in (2, 4, 8, 16):
        for obst in (True, False):
            sc = gen.scene_arm_team(n, obst)
            mo = gen.motions_arm_team(n, M)
            gs = mrv.Scene(sc)
            wp, T = mrv.to_device(mo)
            base = mrv.CHECK_SELF | (mrv.CHECK_ENV if obst else 0)
            ref = None
            for sname, sf in STRATS.items():
                f = base | sf
                full = torch.zeros(mrv.NUM_COUNTERS, dtype=torch.int64, device="cuda")
                gs.motval(wp, T, f | mrv.DIAG_NO_EARLY_EXIT, counters=full)
                cnt = torch.zeros(mrv.NUM_COUNTERS, dtype=torch.int64, device="cuda")
                v = gs.motval(wp, T, f, counters=cnt)
                if ref is None:
                    ref = v.clone()
                assert torch.equal(v, ref), "strategies must agree"
                cf = dict(zip(mrv.COUNTER_NAMES, full.cpu().tolist()))
                ce = dict(zip(mrv.COUNTER_NAMES, cnt.cpu().tolist()))
                ts = []
                for _ in range(reps):
                    flush.zero_()
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record()
                    gs.motval(wp, T, f)
                    b.record()
                    torch.cuda.synchronize()
                    ts.append(a.elapsed_time(b))
                rows.append({"robots": n, "obstacles": obst, "strategy": sname,
                             "effort_pct": 100.0 * cc_work(ce) / max(1, cc_work(cf)),
                             "states_pct": 100.0 * ce["states"] / max(1, cf["states"]),
                             "ms": float(np.median(ts)), "valid_frac": float(ref.float().mean().item()),
                             "motions": M, "composite_states": mo.total_states()})
                print(json.dumps(rows[-1]), flush=True)
    out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles")
    os.makedirs(out, exist_ok=True)
    json.dump(rows, open(os.path.join(out, f"{name}_fig7_ablation.json"), "w"), indent=1)
    lines = [f"# Fig. 7-shaped MotVal ablation on one B200 ({name})", "",
             "Synthetic 7-DOF arm teams in two facing rows, 1000 random motions each (no endpoint rejection), "
             "self-collision checked with the robot-obstacle test (PAPER.md:240), W = 8 states per batch. "
             "effort = CC tests done before early termination / CC tests of a full evaluation "
             "(kernel work counters); ms = median MotVal kernel time (CUDA events, L2 flushed).", "",
             "| robots | obstacles | valid | " + " | ".join(f"{s} effort % / ms" for s in STRATS) + " |",
             "|---|---|---|" + "---|" * len(STRATS)]
    for n in (2, 4, 8, 16):
        for obst in (True, False):
            rs = {r["strategy"]: r for r in rows if r["robots"] == n and r["obstacles"] == obst}
            lines.append(f"| {n} | {'yes' if obst else 'no'} | {rs['combined-rake']['valid_frac']:.3f} | " +
                         " | ".join(f"{rs[s]['effort_pct']:.2f} / {rs[s]['ms']:.3f}" for s in STRATS) + " |")
    open(os.path.join(out, f"{name}_fig7_ablation.md"), "w").write("\n".join(lines) + "\n")


if __name__ == "__main__":
    run(*(sys.argv[1:2] or ["r1"]))
