"""A/B timing of libmrv builds (experiments only): for each .so, time MotVal and FFC on a
config with CUDA events (L2 flushed before each rep) and check the outputs are identical
to the first build's.

  python tools/ab.py cfg5 exp/base.so exp/new.so [...]      (runs each lib in a subprocess)
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(cfg, M, out_prefix):
    sys.path.insert(0, ROOT)
    import numpy as np
    import torch
    from paper_2604_23960_b200 import gen, mrv
    sc, mo = gen.make(cfg, M)
    gs = mrv.Scene(sc)
    wp, T = mrv.to_device(mo)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    res = {}

    def timeit(fn, reps=5):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            flush.zero_()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        return min(ts), sorted(ts)[len(ts) // 2]

    extra = getattr(mrv, os.environ["AB_FLAG"]) if os.environ.get("AB_FLAG") else 0   # e.g. DIAG_NO_EARLY_EXIT
    for q in ("motval", "ffc"):
        f = (lambda: gs.motval(wp, T, mrv.CHECK_ENV | extra)) if q == "motval" else (lambda: gs.ffc(wp, T, extra))
        mn, md = timeit(f)
        out = f().cpu().numpy()
        np.save(f"{out_prefix}_{q}.npy", out)
        res[q] = {"min_ms": mn, "median_ms": md}
    print(json.dumps(res))


def main():
    if sys.argv[1] == "--child":
        child(sys.argv[2], int(sys.argv[3]) if sys.argv[3] != "0" else None, sys.argv[4])
        return
    cfg = sys.argv[1]
    M = os.environ.get("AB_MOTIONS", "0")
    libs = sys.argv[2:]
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    import numpy as np
    ref = None
    for i, lib in enumerate(libs):
        env = dict(os.environ, MRV_LIB_PATH=os.path.abspath(lib))
        pref = f"/tmp/ab_{i}"
        r = subprocess.run([sys.executable, __file__, "--child", cfg, M, pref], env=env, capture_output=True, text=True)
        if r.returncode != 0:
            print(f"{lib}: FAILED\n{r.stderr[-2000:]}")
            continue
        res = json.loads(r.stdout.strip().splitlines()[-1])
        same = {}
        for q in ("motval", "ffc"):
            o = np.load(f"{pref}_{q}.npy")
            if ref is None:
                same[q] = True
            else:
                same[q] = bool(np.array_equal(o, ref[q]))
        if ref is None:
            ref = {q: np.load(f"{pref}_{q}.npy") for q in ("motval", "ffc")}
        print(f"{lib:28s} motval {res['motval']['min_ms']:8.3f} ms (med {res['motval']['median_ms']:8.3f}) "
              f"same={same['motval']}   ffc {res['ffc']['min_ms']:8.3f} ms (med {res['ffc']['median_ms']:8.3f}) "
              f"same={same['ffc']}", flush=True)


if __name__ == "__main__":
    main()
