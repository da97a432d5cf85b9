"""Batched independent registrations across GPUs (BASELINE configs 3 and 5b).

One process per GPU (torchrun).  The pairs are independent, so each rank takes a round-robin
shard and there is no data-path collective: rank r solves pairs r, r+W, r+2W, ...  Only the
small per-pair reports are gathered (all_gather_object) at the end.  `scaling` is weak.

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
        -m paper_1604_02153_b200.batch --n 512 --pairs 8 --nt 16
"""
from __future__ import annotations

import argparse
import json
import os
import time
from typing import Callable


def shard(n_items: int, rank: int, world: int) -> list[int]:
    """Round-robin shard of item indices for `rank` out of `world`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return list(range(rank, n_items, world))


def run_sharded(n_items: int, runner: Callable[[int], dict], rank: int = 0, world: int = 1) -> list[dict] | None:
    """Runs runner(i) for this rank's shard; returns all results ordered by item on rank 0
    (None elsewhere).  With world > 1 torch.distributed must be initialised (any backend)."""
    mine = [dict(runner(i), item=i) for i in shard(n_items, rank, world)]
    if world > 1:
        import torch.distributed as dist

        gathered = [None] * world
        dist.all_gather_object(gathered, mine)
        allres = [r for part in gathered for r in part]
    else:
        allres = mine
    if rank != 0:
        return None
    return sorted(allres, key=lambda r: r["item"])


def pair_inputs(n: int, p: int, nt: int, vmax: float = 0.3):
    """Config 3/5b pair p: smoothed-noise template (seed 1000+p), random smooth v* (2000+p);
    the reference image is m_T transported by v* with nt SL steps (computed on the device)."""
    from . import synth

    mT = synth.smoothed_noise(n, n, 1000 + p)
    v1, v2 = synth.smooth_velocity(n, n, 2000 + p, vmax)
    return mT, (v1, v2)


def registration_runner(ctx, n: int, nt: int, beta: float, norm: int, cheb_iters: int, tol_rel: float):
    from . import api

    def run(p: int) -> dict:
        mT, (v1, v2) = pair_inputs(n, p, nt)
        mR = api.Solver(ctx, (ctx.field(v1), ctx.field(v2)), nt).solve_state_final(ctx.field(mT)).cpu().numpy()
        t0 = time.perf_counter()
        w1, w2, recs, summ = api.newton_solve(ctx, mR, mT, norm, beta, api.COMPRESSIBLE, nt=nt,
                                              kind=api.PC_TWO_LEVEL, coarse_solver=api.COARSE_CHEB,
                                              cheb_iters=cheb_iters, tol_rel=tol_rel)
        return {"seconds": time.perf_counter() - t0, "newton_iterations": summ["iterations"],
                "inner_iterations": int(sum(r["innerIterations"] for r in recs)), "status": summ["status"],
                "final_grad_rel": summ["finalGradNormRel"], "final_residual_rel": summ["finalResidualRel"]}

    return run


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=512)
    ap.add_argument("--pairs", type=int, default=8)
    ap.add_argument("--nt", type=int, default=16)
    ap.add_argument("--beta", type=float, default=1e-3)
    ap.add_argument("--norm", type=int, default=2)
    ap.add_argument("--cheb", type=int, default=10)
    ap.add_argument("--tol-rel", type=float, default=1e-2)
    a = ap.parse_args()
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local))
    from . import api

    ctx = api.Context(local)
    t0 = time.perf_counter()
    res = run_sharded(a.pairs, registration_runner(ctx, a.n, a.nt, a.beta, a.norm, a.cheb, a.tol_rel), rank, world)
    wall = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([wall], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        wall = float(t.item())
    if rank == 0:
        print(json.dumps({"pairs": a.pairs, "n": a.n, "nt": a.nt, "world": world, "wall_s": wall,
                          "pairs_per_s": a.pairs / wall, "results": res}))
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
