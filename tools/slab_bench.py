"""Slab-decomposed GN Hessian matvec (config 5a: 4096^2, nt=32, H2 beta=1e-4) over NCCL.

  python -m torch.distributed.run --nnodes=1 --nproc-per-node N --master-addr 127.0.0.1 \\
      --master-port 29512 tools/slab_bench.py [--size 4096] [--nt 32] [--steps 5]

Every rank builds its slab of the per-iterate invariants (SlabHessian.build: distributed
setup; --setup replicated slices the single-device operator instead), and times K slab
matvecs (device events, barrier on both sides, max over ranks).  Rank 0 checks the assembled
result against the single-device matvec and prints one JSON line.  With one process it runs
the same code path over a 1-rank NCCL group.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch
import torch.distributed as dist

from paper_1604_02153_b200 import api, slab, synth


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", "--n", dest="n", type=int, default=4096)
    ap.add_argument("--nt", type=int, default=32)
    ap.add_argument("--beta", type=float, default=1e-4)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--setup", default="distributed", choices=["distributed", "replicated"])
    a = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29512")
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", local))
    ctx = api.Context(local)
    n, nt = a.n, a.nt
    mT = synth.smoothed_noise(n, n, 1000)
    v1, v2 = synth.smooth_velocity(n, n, 2000)
    vt1, vt2 = synth.smooth_velocity(n, n, 3000)
    F = ctx.field
    comm = slab.DistComm()
    L = n // world
    dev = torch.device("cuda", local)
    torch.cuda.synchronize(dev)
    t_setup = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_setup[0].record()
    if a.setup == "replicated":
        H = api.HessianOperator(ctx, (F(v1), F(v2)), F(mT), F(mT), api.H2SEMI, a.beta, api.COMPRESSIBLE, nt)
        S = slab.SlabHessian.from_operator(ctx, comm, H, api.H2SEMI, a.beta)
    else:
        vs = [F(np.stack([v1[rank * L:(rank + 1) * L], v2[rank * L:(rank + 1) * L]]))]
        S = slab.SlabHessian.build(ctx, comm, vs, [F(mT[rank * L:(rank + 1) * L])], n, nt, api.H2SEMI, a.beta)
        H = None
    t_setup[1].record()
    torch.cuda.synchronize(dev)
    setup_ms = t_setup[0].elapsed_time(t_setup[1])
    vts = [F(np.stack([vt1[rank * L:(rank + 1) * L], vt2[rank * L:(rank + 1) * L]]))]
    outs = [ctx.empty(2, L, n)]
    for _ in range(a.warmup):
        S.apply(vts, outs)
    dist.barrier()
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.steps):
        S.apply(vts, outs)
    e1.record()
    dist.barrier()
    torch.cuda.synchronize(dev)
    ms = torch.tensor([e0.elapsed_time(e1) / a.steps], device=dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    # single-device reference on rank 0 (the full grid fits one B200)
    full = [torch.empty_like(outs[0]) for _ in range(world)]
    dist.all_gather(full, outs[0])
    if rank == 0:
        got = torch.cat(full, dim=1).cpu().numpy()
        if H is None:
            H = api.HessianOperator(ctx, (F(v1), F(v2)), F(mT), F(mT), api.H2SEMI, a.beta, api.COMPRESSIBLE, nt)
        vtd = (F(vt1), F(vt2))
        h1, h2 = H.apply(vtd)
        e = np.stack([h1.cpu().numpy(), h2.cpu().numpy()])
        torch.cuda.synchronize()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record()
        for _ in range(a.steps):
            H.apply(vtd)
        t1.record()
        torch.cuda.synchronize()
        print(json.dumps({"metric": f"slab-decomposed GN Hessian matvec {n}^2 nt={nt} H2 beta={a.beta}",
                          "ranks": world, "ms_per_matvec": float(ms.item()),
                          "matvecs_per_s": 1e3 / float(ms.item()),
                          "single_device_ms_per_matvec": t0.elapsed_time(t1) / a.steps,
                          "max_rel_diff_vs_single_device": float(np.abs(got - e).max() / np.abs(e).max()),
                          "slab_rows": L, "window_rows": S.geo.win_rows, "halo_rows": [S.geo.top, S.geo.bot],
                          "setup": a.setup, "setup_ms_rank0": setup_ms}))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
