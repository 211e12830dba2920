"""ARC-style repeated FFC latency: one planner
iteration calls FFC on a handful of path sets, edits a path, calls again.  Measures the
device time per call with CUDA events for B path sets of cfg4 (12 robots x 1000
timesteps), direct launches vs one captured CUDA graph replayed, and the horizon split
over many warps (n_slices) that makes a single path set fast.

  python tools/arc_loop.py > profiles/<tag>_arc_loop.json
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_23960_b200 import gen, mrv  # noqa: E402


def main():
    sc, mo = gen.make("cfg4", 1024)
    gs = mrv.Scene(sc)
    wp_all, T = mrv.to_device(mo)
    out = {"workload": "cfg4 path sets (12 robots, 10 knots, 1000 timesteps), FFC", "rows": []}
    for B in (1, 8, 64, 1024):
        wp = wp_all[:B].contiguous()
        key = torch.empty(B, dtype=torch.int32, device="cuda")
        stream = torch.cuda.Stream()
        with torch.cuda.stream(stream):
            for _ in range(5):
                gs.ffc(wp, T, out=key, stream=stream)
        torch.cuda.synchronize()
        reps = 200 if B <= 64 else 20
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            a.record(stream)
            for _ in range(reps):
                gs.ffc(wp, T, out=key, stream=stream)
            b.record(stream)
        torch.cuda.synchronize()
        direct = a.elapsed_time(b) * 1e3 / reps
        one = None
        if B == 1:   # the same path set on a single warp (no horizon split)
            with torch.cuda.stream(stream):
                a.record(stream)
                for _ in range(reps):
                    gs.ffc(wp, T, out=key, stream=stream, n_slices=1)
                b.record(stream)
            torch.cuda.synchronize()
            one = a.elapsed_time(b) * 1e3 / reps
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            gs.ffc(wp, T, out=key, stream=torch.cuda.current_stream())
        g.replay()
        torch.cuda.synchronize()
        a.record()
        for _ in range(reps):
            g.replay()
        b.record()
        torch.cuda.synchronize()
        graph = a.elapsed_time(b) * 1e3 / reps
        out["rows"].append({"path_sets": B, "us_per_call_direct": direct, "us_per_call_graph": graph,
                            "us_single_warp": one, "path_sets_per_s": B / (graph * 1e-6)})
    print(json.dumps(out))


if __name__ == "__main__":
    main()
