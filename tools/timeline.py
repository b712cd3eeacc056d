"""Per-kernel device timeline of a few evaluations of a bench config, from the
torch profiler's CUDA activity trace (CUPTI, process-wide, so it sees the
library's kernels on the plan's streams).  Run with FFTPIM_NO_GRAPHS=1 so the
kernels are launched individually.  Prints, for the last evaluation, each
kernel's stream, start and end relative to the evaluation's first kernel.

    FFTPIM_NO_GRAPHS=1 python tools/timeline.py --config 2
"""
import argparse
import json
import os
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--evals", type=int, default=5)
    args = ap.parse_args()
    import torch
    from torch.profiler import ProfilerActivity, profile
    import bench
    import paper_2312_02376_b200 as fp
    from paper_2312_02376_b200 import _native as nat

    w, pos, q, cfg, box, prm = bench.problem_objects(fp, args.config, e=0)
    plan = fp.build_plan(cfg, box, fp.SourcePointSet(pos, q), fp.ObserverPointSet(pos), prm, device=0)
    stream = torch.cuda.current_stream()
    q_dev = torch.from_numpy(q).cuda()
    u_dev = torch.empty(w.n_points, dtype=torch.complex128, device="cuda")

    def ev():
        plan.native.evaluate_into(q_dev.data_ptr(), u_dev.data_ptr(), 1, nat.ALL, stream.cuda_stream)

    for _ in range(5):
        ev()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(args.evals):
            ev()
            torch.cuda.synchronize()
    path = os.path.join(tempfile.mkdtemp(), "trace.json")
    prof.export_chrome_trace(path)
    tr = json.load(open(path))
    ks = [e for e in tr["traceEvents"] if e.get("cat") == "kernel"]
    ks.sort(key=lambda e: e["ts"])
    # split into evaluations at the permutation kernel
    evals, cur = [], []
    for e in ks:
        if "k_permute_q" in e["name"] and cur:
            evals.append(cur)
            cur = []
        cur.append(e)
    evals.append(cur)
    last = evals[-1]
    t0 = min(e["ts"] for e in last)
    t1 = max(e["ts"] + e["dur"] for e in last)
    print(f"{w.name}: evaluation span {t1 - t0:.1f} us over {len(last)} kernels")
    for e in last:
        name = e["name"].split("(")[0].replace("void ", "")[:44]
        print(f"  stream {e['args'].get('stream', '?'):>4}  {e['ts'] - t0:8.1f} -> {e['ts'] + e['dur'] - t0:8.1f}"
              f"  ({e['dur']:6.1f})  {name}")


if __name__ == "__main__":
    main()
