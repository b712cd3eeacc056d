"""Kernel timeline of one sweep evaluation (CUPTI via the torch profiler):
which chain kernels run while the batched precorrection is in flight.
    python tools/sweep_timeline.py [--excitations 8] [--batched]"""
import argparse
import json
import os
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--excitations", type=int, default=8)
    ap.add_argument("--batched", action="store_true", help="one-shift multi-RHS batch instead of a sweep")
    args = ap.parse_args()
    import numpy as np
    import torch
    from torch.profiler import ProfilerActivity, profile
    import bench
    import paper_2312_02376_b200 as fp
    from paper_2312_02376_b200.workloads import c5_kshift
    E = args.excitations
    w, pos, q, cfg, box, prm = bench.problem_objects(fp, 5, e=0)
    rng = np.random.default_rng(3)
    Q = torch.from_numpy(rng.standard_normal((E, q.size)) + 1j * rng.standard_normal((E, q.size))).cuda()
    U = torch.empty_like(Q)
    s = torch.cuda.current_stream().cuda_stream
    if args.batched:
        plan = fp.build_plan(cfg, box, fp.SourcePointSet(pos, q), fp.ObserverPointSet(pos), prm, device=0)
        run = lambda: plan.native.evaluate_into(Q.data_ptr(), U.data_ptr(), E, fp._native.ALL, s)
    else:
        sw = fp.build_sweep_plan(cfg, box, fp.SourcePointSet(pos, q), fp.ObserverPointSet(pos), prm, 0,
                                 [c5_kshift(e)[0] for e in range(E)], device=0)
        run = lambda: sw.evaluate_into(Q.data_ptr(), U.data_ptr(), s)
    run()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        run()
        torch.cuda.synchronize()
    path = os.path.join(tempfile.mkdtemp(), "trace.json")
    prof.export_chrome_trace(path)
    ks = [e for e in json.load(open(path))["traceEvents"] if e.get("cat") == "kernel"]
    ks.sort(key=lambda e: e["ts"])
    t0 = ks[0]["ts"]
    for e in ks:
        name = e["name"].split("(")[0].replace("void ", "")[:40]
        print(f"stream {e['args'].get('stream', '?'):>4} {e['ts'] - t0:10.1f} -> {e['ts'] + e['dur'] - t0:10.1f} "
              f"({e['dur']:8.1f}) {name}")


if __name__ == "__main__":
    main()
