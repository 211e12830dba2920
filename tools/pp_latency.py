"""PP-ST-RRT call latency: a prioritized planner validates
a few candidate edges of the robot being planned per tree extension, against the same fixed
higher-priority paths.  Device time per mrv_pp_motval_batch call for B candidates of pp5
(the partner table built once), direct launches vs a captured CUDA graph, and the table
rebuild a new priority level costs.

  python tools/pp_latency.py > profiles/<tag>_pp_latency.json
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_23960_b200 import gen, mrv  # noqa: E402


def timed(fn, reps, stream):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        for _ in range(3):
            fn()
        a.record(stream)
        for _ in range(reps):
            fn()
        b.record(stream)
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3 / reps


def main():
    sc, paths, cand, t0 = gen.make_pp(65536)
    gs = mrv.Scene(sc)
    pw, pT = mrv.to_device(paths)
    table = gs.pp_table(pw, pT, gen.PP_PARTNERS, gen.PP_HORIZON)
    cw_all, T = mrv.to_device(cand)
    t0_all = torch.from_numpy(t0).cuda()
    stream = torch.cuda.Stream()
    out = {"workload": "pp5 candidates (arm 3 of the cfg2 scene vs the fixed paths of arms 0-2, T = 128)", "rows": []}
    out["table_rebuild_us"] = timed(lambda: gs.pp_table(pw, pT, gen.PP_PARTNERS, gen.PP_HORIZON), 50, stream)
    for B in (1, 16, 256, 4096, 65536):
        cw, t0d = cw_all[:B].contiguous(), t0_all[:B].contiguous()
        res = torch.empty(B, dtype=torch.uint8, device="cuda")
        reps = 200 if B <= 4096 else 20
        direct = timed(lambda: gs.pp_motval(cw, T, t0d, gen.PP_FOCUS, gen.PP_PARTNERS, table, gen.PP_HORIZON,
                                            mrv.CHECK_ENV, out=res, stream=stream), reps, stream)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            gs.pp_motval(cw, T, t0d, gen.PP_FOCUS, gen.PP_PARTNERS, table, gen.PP_HORIZON, mrv.CHECK_ENV, out=res,
                         stream=torch.cuda.current_stream())
        graph = timed(g.replay, reps, torch.cuda.current_stream())
        out["rows"].append({"candidates": B, "us_per_call_direct": direct, "us_per_call_graph": graph,
                            "candidates_per_s": B / (min(direct, graph) * 1e-6)})
    print(json.dumps(out))


if __name__ == "__main__":
    main()
