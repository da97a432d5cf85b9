"""Config 5a registration: 4096^2, nt=32, H2 beta=1e-4, two-level preconditioner with a
10-iteration Chebyshev coarse solve, smoothed-noise template (seed 1000) transported by a
random smooth v* (seed 2000, max|v|=0.3) -> m_R.  Time to solution through newton_solve:

  --mode single : the library's single-device solve (its own fine Hessian);
  --mode slab   : slab-decomposed over the torchrun ranks (slab.SlabFineOperator over NCCL,
                  one slab per GPU): the fine GN data term, the gradient (state, adjoint, body
                  force) and every line-search objective; the driver's vector algebra and the
                  two-level preconditioner's coarse solve run replicated on every rank.

  python tools/slab_newton.py --mode single
  python -m torch.distributed.run --nnodes=1 --nproc-per-node N --master-addr 127.0.0.1 \\
      --master-port 29513 tools/slab_newton.py --mode slab

Rank 0 prints one JSON line (iterations, Krylov iterations, wall time, the time in each slab
callback and the share of the solve outside them: the non-decomposed work).  --max-outer bounds
the run.
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

from paper_1604_02153_b200 import api, slab, synth


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", "--n", dest="n", type=int, default=4096)
    ap.add_argument("--nt", type=int, default=32)
    ap.add_argument("--beta", type=float, default=1e-4)
    ap.add_argument("--mode", default="single", choices=["single", "slab"])
    ap.add_argument("--max-outer", type=int, default=50)
    ap.add_argument("--tol-rel", type=float, default=1e-2)
    a = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    comm = None
    if a.mode == "slab":
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29513")
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", local))
        comm = slab.DistComm()
    ctx = api.Context(local)
    n, nt = a.n, a.nt
    t0 = time.perf_counter()
    mT = synth.smoothed_noise(n, n, 1000)
    v1, v2 = synth.smooth_velocity(n, n, 2000)
    mR = api.Solver(ctx, (ctx.field(v1), ctx.field(v2)), nt).solve_state_final(ctx.field(mT)).cpu().numpy()
    t_inputs = time.perf_counter() - t0
    fo = slab.SlabFineOperator(ctx, comm, mT, api.H2SEMI, a.beta, mR=mR) if comm is not None else None
    ctx.sync()
    if comm is not None:
        comm.dist.barrier()
    t0 = time.perf_counter()
    w1, w2, recs, summ = api.newton_solve(ctx, mR, mT, api.H2SEMI, a.beta, api.COMPRESSIBLE, nt=nt,
                                          kind=api.PC_TWO_LEVEL, coarse_solver=api.COARSE_CHEB, cheb_iters=10,
                                          tol_rel=a.tol_rel, max_outer=a.max_outer, fine_operator=fo)
    ctx.sync()
    wall = time.perf_counter() - t0
    if comm is not None:
        t = torch.tensor([wall], dtype=torch.float64, device=ctx.device)
        comm.dist.all_reduce(t, op=comm.dist.ReduceOp.MAX)
        wall = float(t)
    if rank == 0:
        line = {
            "workload": f"config5a registration {n}x{n} fp64, nt={nt}, H2 beta={a.beta:g}, 2L-cheb10, tolRelGrad {a.tol_rel:g}",
            "mode": a.mode, "ranks": world if comm is not None else 1,
            "time_to_solution_s": wall, "inputs_s": t_inputs,
            "status": summ["status"], "newton_iterations": summ["iterations"],
            "krylov_iterations": int(sum(r["innerIterations"] for r in recs)),
            "line_search_steps": [int(r["lineSearchSteps"]) for r in recs],
            "final_grad_norm_rel": summ["finalGradNormRel"], "final_residual_rel": summ["finalResidualRel"],
            "objective": [r["objective"] for r in recs],
            "per_iteration_s": [r["wallTimeSec"] for r in recs],
            "v_max": float(max(np.abs(w1).max(), np.abs(w2).max())),
        }
        if fo is not None:
            inside = fo.build_s + fo.apply_s + fo.gradient_s + fo.objective_s + fo.coarse_s + fo.precond_s
            line.update(slab_builds=fo.builds, slab_build_s=fo.build_s, slab_matvecs=fo.matvecs,
                        slab_data_term_s=fo.apply_s, slab_gradients=fo.gradients, slab_gradient_s=fo.gradient_s,
                        slab_objectives=fo.objectives, slab_objective_s=fo.objective_s,
                        slab_coarse_builds=fo.coarse_builds, slab_coarse_s=fo.coarse_s,
                        slab_two_level_applies=fo.precond_applies, slab_two_level_s=fo.precond_s,
                        decomposed_s=inside, non_decomposed_s=wall - inside,
                        non_decomposed_share=(wall - inside) / wall,
                        # within the outer iterations (the hooks all run inside them): excludes the
                        # once-per-solve eigenvalue estimate and the final Jacobian
                        iterations_s=sum(r["wallTimeSec"] for r in recs),
                        per_iteration_non_decomposed_share=(sum(r["wallTimeSec"] for r in recs) - inside)
                        / sum(r["wallTimeSec"] for r in recs),
                        note="non-decomposed = the driver's whole-grid vector algebra, the eigenvalue estimate "
                             "at v=0 (once per solve) and the final Jacobian (rank 0's clock)")
        print(json.dumps(line), flush=True)
    if comm is not None:
        comm.dist.destroy_process_group()


if __name__ == "__main__":
    main()
