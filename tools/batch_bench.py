"""Multi-RHS throughput of one plan: B charge vectors per evaluate call, device
resident, CUDA events; compares the batched precorrection (B >= 8) with B
single evaluations.   python tools/batch_bench.py --config 2 --batch 64"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    import numpy as np
    import torch
    import bench
    import paper_2312_02376_b200 as fp
    w, pos, q, cfg, box, prm = bench.problem_objects(fp, args.config, e=0)
    plan = fp.build_plan(cfg, box, fp.SourcePointSet(pos, q), fp.ObserverPointSet(pos), prm, device=0)
    rng = np.random.default_rng(1)
    Q = torch.from_numpy(rng.standard_normal((args.batch, q.size)) + 1j * rng.standard_normal((args.batch, q.size))).cuda()
    U = torch.empty((args.batch, w.n_points), dtype=torch.complex128, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    nat = plan.native

    def batched():
        nat.evaluate_into(Q.data_ptr(), U.data_ptr(), args.batch, fp._native.ALL, s)

    q1 = torch.empty_like(Q[0])
    u1 = torch.empty_like(U[0])

    def singles():   # one graph replay per vector (fixed buffers, device copies in and out)
        for b in range(args.batch):
            q1.copy_(Q[b])
            nat.evaluate_into(q1.data_ptr(), u1.data_ptr(), 1, fp._native.ALL, s)
            U[b].copy_(u1)

    out = {"config": w.name, "batch": args.batch}
    for name, fn in (("batched", batched), ("singles", singles)):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.reps
        out[name] = {"ms_per_call": ms, "points_per_s": args.batch * w.n_points / (ms * 1e-3)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
