"""Batched independent registrations across GPUs (BASELINE configs 3 and 5b).

One process per GPU (torchrun).  The pairs are independent, so each rank takes a round-robin
shard and there is no data-path collective: rank r solves pairs r, r+W, r+2W, ...  Only the
small per-pair reports are gathered (all_gather_object) at the end.  `scaling` is weak.

Within a GPU, `--batch B` solves B pairs together in lockstep (api.newton_solve_batch: every
step of the B registrations in the same kernel launches, csrc/batch.cu), and `--lanes L` runs L
solves (or batches) at once: L host threads, each with its own library context and stream,
take the rank's pairs (or batches) from a shared queue.  A solve at 256^2 launches
kernels too small to fill 148 SMs, so concurrent streams fill the device (config 5b).  The
library's per-call state is per context (plans, graphs, scratch) or thread-local, and each
newton_solve is a single C call that releases the GIL.

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
        -m paper_1604_02153_b200.batch --size 512 --pairs 8 --nt 16   (--size, not --n: torchrun rejects --n as an ambiguous abbreviation of its own options)
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


def run_lanes(items: list[int], make_runner: Callable[[int], Callable[[int], dict]], lanes: int) -> list[dict]:
    """Runs the items on `lanes` threads; lane k builds its runner once (make_runner(k), e.g.
    its own context and stream) and then takes items from a shared queue.  Results come back
    in item order, each tagged with its item; the first exception of any lane is re-raised."""
    import queue
    import threading

    if lanes < 1:
        raise ValueError("lanes must be >= 1")
    todo: queue.SimpleQueue = queue.SimpleQueue()
    for i in items:
        todo.put(i)
    results: dict[int, dict] = {}
    errors: list[BaseException] = []

    def lane(k: int):
        try:
            run = make_runner(k)
            while not errors:
                try:
                    i = todo.get_nowait()
                except queue.Empty:
                    return
                results[i] = dict(run(i), item=i, lane=k)
        except BaseException as e:  # noqa: BLE001 - handed to the caller
            errors.append(e)

    threads = [threading.Thread(target=lane, args=(k,), daemon=True) for k in range(min(lanes, max(1, len(items))))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if errors:
        raise errors[0]
    return [results[i] for i in items]


def run_sharded(n_items: int, runner: Callable[[int], dict] | None, rank: int = 0, world: int = 1,
                make_runner: Callable[[int], Callable[[int], dict]] | None = None, lanes: int = 1) -> list[dict] | None:
    """Runs this rank's shard (runner(i) in order, or on `lanes` concurrent lanes built by
    make_runner); returns all results ordered by item on rank 0 (None elsewhere).  With
    world > 1 torch.distributed must be initialised (any backend)."""
    if make_runner is not None:
        mine = run_lanes(shard(n_items, rank, world), make_runner, lanes)
    else:
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


def make_images(ctx, n: int, p: int, nt: int):
    """Host images (mR, mT) of pair p: mR is m_T transported by v* on the device."""
    from . import api

    mT, (v1, v2) = pair_inputs(n, p, nt)
    mR = api.Solver(ctx, (ctx.field(v1), ctx.field(v2)), nt).solve_state_final(ctx.field(mT)).cpu().numpy()
    return mR, mT


def registration_runner(ctx, n: int, nt: int, beta: float, norm: int, cheb_iters: int, tol_rel: float,
                        images: dict | None = None):
    """runner(p): newton_solve of pair p (images[p] = (mR, mT) when given, else made here)."""
    from . import api

    def run(p: int) -> dict:
        mR, mT = images[p] if images is not None else make_images(ctx, n, p, nt)
        t0 = time.perf_counter()
        w1, w2, recs, summ = api.newton_solve(ctx, mR, mT, norm, beta, api.COMPRESSIBLE, nt=nt,
                                              kind=api.PC_TWO_LEVEL, coarse_solver=api.COARSE_CHEB,
                                              cheb_iters=cheb_iters, tol_rel=tol_rel)
        return {"seconds": time.perf_counter() - t0, "newton_iterations": summ["iterations"],
                "inner_iterations": int(sum(r["innerIterations"] for r in recs)), "status": summ["status"],
                "final_grad_rel": summ["finalGradNormRel"], "final_residual_rel": summ["finalResidualRel"]}

    return run


def batched_runner(ctx, n: int, nt: int, beta: float, norm: int, cheb_iters: int, tol_rel: float, images: dict,
                   chunks: list[list[int]]):
    """runner(c): the pairs chunks[c] solved together in lockstep (api.newton_solve_batch: one
    launch per step for all of them, csrc/batch.cu); one result per pair under "pairs"."""
    import numpy as np

    from . import api

    def run(c: int) -> dict:
        ps = chunks[c]
        mR = np.stack([images[p][0] for p in ps])
        mT = np.stack([images[p][1] for p in ps])
        t0 = time.perf_counter()
        out = api.newton_solve_batch(ctx, mR, mT, norm, beta, api.COMPRESSIBLE, nt=nt, kind=api.PC_TWO_LEVEL,
                                     coarse_solver=api.COARSE_CHEB, cheb_iters=cheb_iters, tol_rel=tol_rel)
        dt = time.perf_counter() - t0
        res = []
        for p, (_, _, recs, summ) in zip(ps, out):
            res.append({"item": p, "seconds": dt, "batch": len(ps), "newton_iterations": summ["iterations"],
                        "inner_iterations": int(sum(r["innerIterations"] for r in recs)), "status": summ["status"],
                        "error": summ["error"], "final_grad_rel": summ["finalGradNormRel"],
                        "final_residual_rel": summ["finalResidualRel"]})
        return {"pairs": res}

    return run


def _reference_batch(a, images, rank, world):
    """The same pairs through the reference's own newtonSolve on host threads (CPU baseline of
    configs 3/5b): one single-threaded solve per thread, threads in parallel (the reference's
    solves are reentrant, proj/README.md:157-158; ctypes releases the GIL).  Images as for
    the GPU arm (m_R transported on the device, bit-compatible with the reference's)."""
    from oracle import ref

    threads = a.threads or os.cpu_count() or 1

    def make_runner(_lane):
        def run(p):
            mR, mT = images[p]
            t0 = time.perf_counter()
            _, _, rep, rs = ref.newton_solve(mR, mT, a.norm, a.beta, 0, nt=a.nt, two_level=True, cheb=True,
                                             cheb_iters=a.cheb, tol_rel=a.tol_rel)
            return {"seconds": time.perf_counter() - t0, "newton_iterations": int(rs[1]),
                    "inner_iterations": int(sum(int(q[5]) for q in rep[:int(rs[1])]))}
        return run

    t0 = time.perf_counter()
    res = run_lanes(sorted(images), make_runner, threads)
    wall = time.perf_counter() - t0
    if rank == 0:
        print(json.dumps({"impl": "reference", "pairs": len(images), "n": a.n, "nt": a.nt, "world": world,
                          "threads": threads, "wall_s": wall, "pairs_per_s": len(images) / wall, "results": res}))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", "--n", dest="n", type=int, default=512)
    ap.add_argument("--pairs", type=int, default=8)
    ap.add_argument("--nt", type=int, default=16)
    ap.add_argument("--beta", type=float, default=1e-3)
    ap.add_argument("--norm", type=int, default=2)
    ap.add_argument("--cheb", type=int, default=10)
    ap.add_argument("--tol-rel", type=float, default=1e-2)
    ap.add_argument("--lanes", type=int, default=1, help="concurrent solves per GPU (own context + stream each)")
    ap.add_argument("--batch", type=int, default=1,
                    help="pairs solved together in lockstep per solve (same kernel launches; 1 = one pair per solve)")
    ap.add_argument("--passes", type=int, default=1, help="passes over the pairs; the last one is reported")
    ap.add_argument("--impl", default="vrg", choices=["vrg", "reference"],
                    help="reference: the unmodified reference's newtonSolve (oracle/_ref) on --threads host threads")
    ap.add_argument("--threads", type=int, default=0, help="host threads of --impl reference (0: all)")
    a = ap.parse_args()
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local))
    from . import api

    # the images of this rank's pairs are made before the timed region (a registration service
    # receives them); one context + stream per lane, made up front; --passes 2 times a second
    # pass over the same pairs (plans, graphs and the block cache warm)
    main_ctx = api.Context(local)
    images = {p: make_images(main_ctx, a.n, p, a.nt) for p in shard(a.pairs, rank, world)}
    if a.impl == "reference":
        return _reference_batch(a, images, rank, world)
    ctxs = [main_ctx] + [api.Context(local, stream=torch.cuda.Stream(local)) for _ in range(1, a.lanes)]

    def make_runner(lane: int):
        return registration_runner(ctxs[lane], a.n, a.nt, a.beta, a.norm, a.cheb, a.tol_rel, images)

    mine = shard(a.pairs, rank, world)
    chunks = [mine[i:i + a.batch] for i in range(0, len(mine), max(1, a.batch))]

    def make_batched(lane: int):
        return batched_runner(ctxs[lane], a.n, a.nt, a.beta, a.norm, a.cheb, a.tol_rel, images, chunks)

    for _ in range(a.passes):
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        t0 = time.perf_counter()
        if a.batch > 1:
            part = [r for c in run_lanes(list(range(len(chunks))), make_batched, a.lanes) for r in c["pairs"]]
            if world > 1:
                gathered = [None] * world
                torch.distributed.all_gather_object(gathered, part)
                part = [r for g in gathered for r in g]
            res = sorted(part, key=lambda r: r["item"]) if rank == 0 else None
        else:
            res = run_sharded(a.pairs, None, rank, world, make_runner=make_runner, lanes=a.lanes)
        wall = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([wall], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        wall = float(t.item())
    if rank == 0:
        print(json.dumps({"pairs": a.pairs, "n": a.n, "nt": a.nt, "world": world, "lanes": a.lanes, "batch": a.batch,
                          "passes": a.passes, "wall_s": wall,
                          "pairs_per_s": a.pairs / wall, "results": res}))
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
