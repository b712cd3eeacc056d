"""Schedule probe: device time of one graph-replayed evaluation for each `parts`
subset (NEAR, FAR, ALL) of a bench config.  Diagnostic only (not a bench line).

    python tools/parts_probe.py --config 2 --steps 50
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--steps", type=int, default=50)
    args = ap.parse_args()
    import torch
    import bench
    import paper_2312_02376_b200 as fp
    from paper_2312_02376_b200 import _native as nat

    w, pos, q, cfg, box, prm = bench.problem_objects(fp, args.config, e=0)
    plan = fp.build_plan(cfg, box, fp.SourcePointSet(pos, q), fp.ObserverPointSet(pos), prm, device=0)
    stream = torch.cuda.current_stream()
    q_dev = torch.from_numpy(q).cuda()
    u_dev = torch.empty(w.n_points, dtype=torch.complex128, device="cuda")
    for name, parts in (("near", nat.NEAR), ("far", nat.FAR), ("all", nat.ALL)):
        for _ in range(5):
            plan.native.evaluate_into(q_dev.data_ptr(), u_dev.data_ptr(), 1, parts, stream.cuda_stream)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            plan.native.evaluate_into(q_dev.data_ptr(), u_dev.data_ptr(), 1, parts, stream.cuda_stream)
        e1.record(stream)
        torch.cuda.synchronize()
        print(f"{w.name} parts={name:4s} {e0.elapsed_time(e1) / args.steps * 1e3:8.1f} us")


if __name__ == "__main__":
    main()
