"""CPU tests of the slab decomposition's host logic: geometry, the
periodic row-halo exchange and the distributed FFT regularisation, with world_size 2 over gloo
(DistComm) against the in-process LocalComm and against a plain 2-D FFT."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1604_02153_b200 import slab


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _field(n1, n2, seed):
    g = torch.Generator().manual_seed(seed)
    return torch.randn(2, n1, n2, generator=g, dtype=torch.float64)


def _reg_reference(v, norm, beta):
    """beta A v with one 2-D FFT per component (spectral.cpp:109-120)."""
    n1, n2 = v.shape[-2:]
    k1 = np.fft.fftfreq(n1, 1.0 / n1)
    k2 = np.arange(n2 // 2 + 1)
    k1 = np.where(np.arange(n1) <= n1 // 2, np.arange(n1), np.arange(n1) - n1)
    sym = beta * (k1[:, None] ** 2 + k2[None, :] ** 2) ** norm
    return np.stack([np.fft.irfft2(np.fft.rfft2(c) * sym, s=(n1, n2)) for c in v.numpy()])


def test_geometry():
    g = slab.SlabGeometry(4096, 4096, 8, 6)
    assert g.L == 512 and g.win_rows % 16 == 0 and g.win_rows >= g.L + 2 * 6 + 3
    assert g.top == 6 + 1 + 32 and g.bot == g.win_rows - 512 - 7 + 32
    assert g.win_base(0) == -7 and g.win_base(3) == 3 * 512 - 7
    with pytest.raises(Exception):
        slab.SlabGeometry(100, 64, 3, 2)


def test_local_exchange_periodic():
    n1, n2, G = 48, 8, 4
    full = torch.arange(n1 * n2, dtype=torch.float64).view(n1, n2)
    comm = slab.LocalComm(G)
    locs = list(full.split(n1 // G, dim=0))
    out = comm.exchange_rows(locs, 5, 20)  # bot wider than a slab: spans two neighbours
    for i, o in enumerate(out):
        rows = [(i * 12 + r) % n1 for r in range(-5, 12 + 20)]
        assert torch.equal(o, full[rows])


def test_local_fill_halos_matches_exchange():
    n1, n2, G, top, bot = 64, 6, 4, 9, 13
    full = torch.randn(n1, n2, dtype=torch.float64)
    L = n1 // G
    comm = slab.LocalComm(G)
    bufs = [torch.zeros(top + L + bot, n2, dtype=torch.float64) for _ in range(G)]
    for i in range(G):
        bufs[i][top:top + L] = full[i * L:(i + 1) * L]
    comm.fill_halos(bufs, L, top, bot)
    ref = comm.exchange_rows(list(full.split(L, dim=0)), top, bot)
    for b, r in zip(bufs, ref):
        assert torch.equal(b, r)


def test_distributed_reg_local():
    n1, n2 = 32, 24
    v = _field(n1, n2, 7)
    for G in (1, 2, 4):
        comm = slab.LocalComm(G)
        outs = slab.distributed_reg(comm, list(v.split(n1 // G, dim=-2)), n1, n2, 2, 1e-3)
        got = torch.cat(outs, dim=-2).numpy()
        ref = _reg_reference(v, 2, 1e-3)
        assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max()


def test_local_allgather_rows():
    v = _field(32, 24, 5)
    comm = slab.LocalComm(4)
    out = torch.empty_like(v)
    comm.allgather_rows(list(v.split(8, dim=-2)), out)
    assert torch.equal(out, v)


def test_row_reach():
    n1, n2 = 16, 4
    h = 2 * np.pi / n1
    x = torch.tensor(-np.pi + np.arange(n1) * h)[:, None].repeat(1, n2)
    x[3, 1] += 2.5 * h
    x[15, 0] += 1.5 * h  # wraps past +pi
    assert abs(slab.row_reach(x, n1) - 2.5) < 1e-12
    x[0, 0] = float("nan")
    assert slab.row_reach(x, n1) == float("inf")


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n1, n2 = 32, 24
        v = _field(n1, n2, 11)
        L = n1 // world
        comm = slab.DistComm()
        loc = v[:, rank * L:(rank + 1) * L].contiguous()
        ex = comm.exchange_rows([loc], 7, 9)[0]
        buf = torch.zeros(2, 7 + L + 9, n2, dtype=torch.float64)
        buf[:, 7:7 + L] = loc
        comm.fill_halos([buf[0]], L, 7, 9)
        comm.fill_halos([buf[1]], L, 7, 9)
        assert torch.equal(buf, ex)
        reg = slab.distributed_reg(comm, [loc], n1, n2, 1, 1e-2)[0]
        m = comm.allreduce_max([torch.tensor([float(rank), -float(rank)])])[0]
        gathered = torch.full_like(v, float("nan"))
        comm.allgather_rows([loc], gathered)  # SlabFineOperator's b gather
        assert torch.equal(gathered, v)
        # a NaN on one rank reaches every rank as +inf (guards and finiteness checks fail together)
        nanm = comm.allreduce_max([torch.tensor([float("nan") if rank == 1 else 0.5, 0.25])])[0]
        # the fine-operator callbacks' common verdict: one failing rank fails all
        verdicts = (comm.any_failed(rank == 1), comm.any_failed(False),
                    float(comm.allreduce_sum([torch.tensor([rank + 1.0])])[0].item()))
        # numpy copies: tensors would travel as shared-memory handles the exiting worker frees
        q.put((rank, ex.numpy().copy(), reg.numpy().copy(), m.tolist(), nanm.tolist(), verdicts))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_slab_comm():
    world = 2
    ctxm = mp.get_context("spawn")
    q = ctxm.Queue()
    port = _free_port()
    procs = [ctxm.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    n1, n2 = 32, 24
    v = _field(n1, n2, 11)
    local = slab.LocalComm(world)
    ex_ref = local.exchange_rows(list(v.split(n1 // world, dim=-2)), 7, 9)
    reg_ref = _reg_reference(v, 1, 1e-2)
    for rank, ex, reg, m, nanm, verdicts in res:
        assert nanm == [float("inf"), 0.25] and verdicts == (True, False, 3.0)
        assert np.array_equal(ex, ex_ref[rank].numpy())
        L = n1 // world
        assert np.abs(reg - reg_ref[:, rank * L:(rank + 1) * L]).max() <= 1e-12 * np.abs(reg_ref).max()
        assert m == [1.0, 0.0]


def test_local_allreduce_max_nan_and_verdict():
    comm = slab.LocalComm(3)
    m = comm.allreduce_max([torch.tensor([0.5, 1.0]), torch.tensor([float("nan"), 2.0]), torch.tensor([0.1, 3.0])])
    assert all(x.tolist() == [float("inf"), 3.0] for x in m)
    assert comm.any_failed(True) and not comm.any_failed(False)
    assert [float(x) for x in comm.allreduce_sum([torch.tensor(1.0), torch.tensor(2.0), torch.tensor(4.0)])] == [7.0] * 3
