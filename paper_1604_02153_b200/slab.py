"""Slab-decomposed GN Hessian matvec for one large grid.

The n1 x n2 grid is split along axis 1 into G slabs of L = n1/G rows, one per rank (one GPU
per process under torchrun, NCCL over NVLink).  The reference is single-process; this is the
B200 extension of `inverse::HessianOperator::apply` (src/inverse.cpp:176-233) for a grid whose
matvec should use several GPUs.  Per SL step of the incremental state / adjoint:

* the step's gather kernel (C ABI `vrg_slab_step`, the band kernel) interpolates at the
  departure points of the slab's rows from a *coefficient window* (the slab's rows plus D+1
  rows above and the rest of a 16-row multiple below, D = largest departure displacement in
  rows), applies the step epilogue and row-filters the result (rows are complete in a slab);
* the column pass needs the row-filtered field on the window plus the 32-row reach of the
  chunk-carry filter: one halo exchange of `top`/`bot` rows with the two neighbouring slabs
  (periodic ring), then `vrg_slab_cols` computes the window's coefficients, including the
  halo rows redundantly, so the gather needs no second exchange;
* the regularisation beta A vt uses a distributed 2-D FFT: row FFTs (local rows) -> all-to-all
  transpose -> column FFTs -> symbol -> inverse -> all-to-all -> inverse row FFTs;
* the blow-up guard reduces the per-row maxima of every step with a max over ranks and is
  checked in the reference's order with its messages (transport.cpp:16-20).

The per-iterate invariants (state trajectory, gradients, departure points, div v) are built
once per Newton iterate by the single-device operator and sliced per slab (`from_operator`);
the matvec, applied many times per iterate, is the decomposed hot path.

Communicators: `DistComm` (torch.distributed; NCCL on GPUs, gloo on CPU for the host-logic
tests) and `LocalComm` (G virtual slabs in one process, run phase by phase: single-device
validation of the decomposition, no concurrency between the virtual ranks).
"""
from __future__ import annotations

import ctypes as C
import math

import torch

from . import api

KIND_STORE, KIND_INC, KIND_INC0, KIND_SEED, KIND_SEED0, KIND_ADJ, KIND_ADJ_LAST, KIND_STATE = range(8)
CARRY = 32  # rows of chunk-carry reach of the column pass (2 chunks of 16)


# ------------------------------------------------------------------------------ communicators
def _nan_to_inf(t):
    return torch.nan_to_num(t, nan=float("inf")) if t.is_floating_point() else t


class LocalComm:
    """G virtual slabs in one process: exchanges are tensor copies."""

    def __init__(self, size: int):
        self.size = size
        self.ranks = list(range(size))

    def exchange_rows(self, locs, top, bot):
        """locs[i] = (..., L, n2) slab of rank i -> (..., top + L + bot, n2) with the periodic
        neighbours' rows (may span several slabs when L < top or L < bot)."""
        full = torch.cat(locs, dim=-2)
        n1 = full.shape[-2]
        L = locs[0].shape[-2]
        out = []
        for i in self.ranks:
            idx = torch.arange(i * L - top, i * L + L + bot, device=full.device) % n1
            out.append(full.index_select(-2, idx))
        return out

    def fill_halos(self, bufs, L, top, bot):
        """bufs[i] = (top + L + bot, n2) with the slab's rows at [top, top+L): fills the halo
        rows from the periodic neighbours' slab rows."""
        full = torch.cat([b[top:top + L] for b in bufs], dim=0)
        n1 = full.shape[0]
        for i in self.ranks:
            if top:
                bufs[i][:top] = full.index_select(0, torch.arange(i * L - top, i * L, device=full.device) % n1)
            if bot:
                bufs[i][top + L:] = full.index_select(
                    0, torch.arange(i * L + L, i * L + L + bot, device=full.device) % n1)

    def alltoall(self, send):
        """send[i][q] from rank i to rank q -> recv[q][i]."""
        return [[send[i][q] for i in self.ranks] for q in self.ranks]

    def allreduce_max(self, vals):
        m = torch.stack([_nan_to_inf(torch.as_tensor(v)) for v in vals]).amax(0)
        return [m for _ in self.ranks]

    def allgather_rows(self, locs, out):
        """locs[i] = (m, L, n2) slab of rank i -> out (m, n1, n2), the slabs in rank order."""
        out.copy_(torch.cat(locs, dim=-2))

    def any_failed(self, failed: bool) -> bool:
        return bool(failed)

    def allreduce_sum(self, vals):
        """Sum over the virtual ranks in rank order."""
        t = torch.as_tensor(vals[0]).clone()
        for v in vals[1:]:
            t = t + torch.as_tensor(v)
        return [t for _ in self.ranks]


class DistComm:
    """One slab per process over torch.distributed (NCCL on GPUs, gloo on CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.size = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.ranks = [self.rank]

    def exchange_rows(self, locs, top, bot):
        (loc,) = locs
        L = loc.shape[-2]
        if top > L or bot > L:
            raise api.InvalidArgument("slab halo is wider than a slab: use fewer ranks")
        d, G, r = self.dist, self.size, self.rank
        nxt, prv = (r + 1) % G, (r - 1) % G
        up = torch.empty_like(loc[..., :top, :]) if top else None
        dn = torch.empty_like(loc[..., :bot, :]) if bot else None
        reqs = []
        if G == 1:
            if top:
                up.copy_(loc[..., L - top:, :])
            if bot:
                dn.copy_(loc[..., :bot, :])
        else:
            ops = []
            if top:
                ops += [d.P2POp(d.isend, loc[..., L - top:, :].contiguous(), nxt, self.group),
                        d.P2POp(d.irecv, up, prv, self.group)]
            if bot:
                ops += [d.P2POp(d.isend, loc[..., :bot, :].contiguous(), prv, self.group),
                        d.P2POp(d.irecv, dn, nxt, self.group)]
            reqs = d.batch_isend_irecv(ops)
            for q in reqs:
                q.wait()
        parts = [p for p in (up, loc, dn) if p is not None]
        return [torch.cat(parts, dim=-2)]

    def fill_halos(self, bufs, L, top, bot):
        (b,) = bufs
        if top > L or bot > L:
            raise api.InvalidArgument("slab halo is wider than a slab: use fewer ranks")
        d, G, r = self.dist, self.size, self.rank
        mid = b[top:top + L]
        if G == 1:
            if top:
                b[:top] = mid[L - top:]
            if bot:
                b[top + L:] = mid[:bot]
            return
        nxt, prv = (r + 1) % G, (r - 1) % G
        ops = []
        if top:  # my last `top` rows are the next slab's top halo
            ops += [d.P2POp(d.isend, mid[L - top:], nxt, self.group), d.P2POp(d.irecv, b[:top], prv, self.group)]
        if bot:  # my first `bot` rows are the previous slab's bottom halo
            ops += [d.P2POp(d.isend, mid[:bot], prv, self.group), d.P2POp(d.irecv, b[top + L:], nxt, self.group)]
        for q in d.batch_isend_irecv(ops):
            q.wait()

    def alltoall(self, send):
        (chunks,) = send
        recv = [torch.empty_like(c) for c in chunks]
        d = self.dist
        if self.size == 1:
            recv[0].copy_(chunks[0])
        elif d.get_backend(self.group) == "nccl":
            d.all_to_all(recv, [c.contiguous() for c in chunks], group=self.group)
        else:  # gloo has no all_to_all: pairwise exchanges
            recv[self.rank].copy_(chunks[self.rank])
            ops = []
            for q in range(self.size):
                if q != self.rank:
                    ops += [d.P2POp(d.isend, chunks[q].contiguous(), q, self.group),
                            d.P2POp(d.irecv, recv[q], q, self.group)]
            for r in d.batch_isend_irecv(ops):
                r.wait()
        return [recv]

    def allreduce_max(self, vals):
        """Max over ranks.  NaN becomes +inf first, so a rank's non-finite value reaches every
        rank whatever the backend does with NaN under MAX.  NCCL reduces device tensors only:
        a host input (e.g. a departure reach computed on the host) travels to the rank's
        device and the result comes back to the input's device."""
        (v,) = vals
        t = _nan_to_inf(torch.as_tensor(v)).clone()
        if self.size > 1:
            home = t.device
            if self.dist.get_backend(self.group) == "nccl" and t.device.type != "cuda":
                t = t.to(torch.device("cuda", torch.cuda.current_device()))
            self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
            t = t.to(home)
        return [t]

    def allreduce_sum(self, vals):
        """Sum over ranks (device tensors under NCCL, as allreduce_max)."""
        (v,) = vals
        t = torch.as_tensor(v).clone()
        if self.size > 1:
            home = t.device
            if self.dist.get_backend(self.group) == "nccl" and t.device.type != "cuda":
                t = t.to(torch.device("cuda", torch.cuda.current_device()))
            self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)
            t = t.to(home)
        return [t]

    def any_failed(self, failed: bool) -> bool:
        """True on every rank when any rank reports a failure (the callbacks' common verdict)."""
        return bool(self.allreduce_max([torch.tensor(1.0 if failed else 0.0)])[0].item() > 0.0)

    def allgather_rows(self, locs, out):
        (loc,) = locs
        if self.size == 1:
            out.copy_(loc)
            return
        G, L = self.size, loc.shape[-2]
        for c in range(out.shape[0]):  # out[c] (n1, n2) contiguous: G row blocks in rank order
            self.dist.all_gather(list(out[c].view(G, L, -1).unbind(0)), loc[c].contiguous(), group=self.group)


# ------------------------------------------------------------------------------ geometry
class SlabGeometry:
    """Rows, window and halo sizes of the slabs (host logic, tested on CPU)."""

    def __init__(self, n1, n2, size, reach_rows):
        if n1 % size:
            raise api.InvalidArgument("slab decomposition: n1 must be a multiple of the number of ranks")
        self.n1, self.n2, self.size = n1, n2, size
        self.L = n1 // size
        self.D = int(reach_rows)
        need = self.L + 2 * self.D + 3               # rows r0-D-1 .. r0+L+D+1
        self.win_rows = (need + 15) // 16 * 16
        self.top = self.D + 1 + CARRY                # rows above the slab in the exchange
        self.bot = self.win_rows - self.L - self.D - 1 + CARRY

    def r0(self, rank):
        return rank * self.L

    def win_base(self, rank):
        """Grid row of window row 0 (may be negative: periodic)."""
        return self.r0(rank) - self.D - 1


def row_reach(x1, n1, r0=0):
    """Largest |departure - arrival| along axis 1 in cells over the rows of x1 (global row r0 +
    local row), minimum image; non-finite -> inf."""
    h = 2 * math.pi / n1
    L = x1.shape[-2]
    xa = (-math.pi + (r0 + torch.arange(L, device=x1.device, dtype=x1.dtype)) * h)[:, None]
    d = x1 - xa
    d = d - 2 * math.pi * torch.floor((d + math.pi) / (2 * math.pi))
    if not bool(torch.isfinite(d).all()):
        return float("inf")
    return float(d.abs().max()) / h


def reg_symbol_cols(n1, n2, norm, beta, c0, c1, device):
    """beta * gamma on half-spectrum columns c0..c1-1 for all rows (spectral.cpp:46-66)."""
    k1 = torch.arange(n1, device=device, dtype=torch.float64)
    k1 = torch.where(k1 <= n1 // 2, k1, k1 - n1)
    k2 = torch.arange(c0, c1, device=device, dtype=torch.float64)
    ksq = k1[:, None] ** 2 + k2[None, :] ** 2
    return beta * ksq ** int(norm)


def distributed_spectral(comm, fields, n1, n2, op):
    """Distributed 2-D FFT pipeline over slab fields: fields[i] = (m, L, n2) -> per rank the
    inverse transforms of op(spectra (m, n1, wc) of the rank's column block, k1 (n1, 1),
    k2 (1, wc), valid columns) = (m', n1, wc).  Row FFTs of the local rows, all-to-all transpose
    to column blocks, column FFTs, op, inverse column FFTs, all-to-all back, inverse row FFTs
    (torch.fft = cuFFT on the device; the inverse transforms carry the 1/N of
    fft.cpp:70-78)."""
    G = comm.size
    nc = n2 // 2 + 1
    wc = -(-nc // G)  # half-spectrum columns per rank in the transposed layout
    L = n1 // G
    send = []
    for f in fields:
        s = torch.fft.rfft(f, dim=-1)
        s = torch.nn.functional.pad(s, (0, G * wc - nc))
        send.append([s[..., q * wc:(q + 1) * wc].contiguous() for q in range(G)])
    recv = comm.alltoall(send)
    back = []
    for k, q in enumerate(comm.ranks):
        col = torch.fft.fft(torch.cat(recv[k], dim=-2), dim=-2)  # (m, n1, wc)
        c0, c1 = min(q * wc, nc), min((q + 1) * wc, nc)
        dev = col.device
        k1 = torch.arange(n1, device=dev, dtype=torch.float64)
        k1 = torch.where(k1 <= n1 // 2, k1, k1 - n1)[:, None]
        k2 = torch.arange(q * wc, (q + 1) * wc, device=dev, dtype=torch.float64)[None, :]
        out = op(col, k1, k2, c1 - c0)
        out[..., c1 - c0:] = 0
        col = torch.fft.ifft(out, dim=-2)
        back.append([col[..., r * L:(r + 1) * L, :].contiguous() for r in range(G)])
    got = comm.alltoall(back)
    return [torch.fft.irfft(torch.cat(got[k], dim=-1)[..., :nc], n=n2, dim=-1) for k in range(len(comm.ranks))]


def distributed_reg(comm, vts, n1, n2, norm, beta):
    """beta A vt (applyReg, spectral.cpp:109-120) of slab fields vts[i] = (..., L, n2)."""
    def op(f, k1, k2, _):
        return f * (beta * (k1 ** 2 + k2 ** 2) ** int(norm))
    return distributed_spectral(comm, vts, n1, n2, op)


def _nyq0(k, n):
    return torch.where(k == n // 2, torch.zeros_like(k), k)  # spectral.cpp:31-33


def distributed_gradient(comm, fields, n1, n2):
    """spectral::gradient (spectral.cpp:68-87) of slab fields (m, L, n2) -> (m, 2, L, n2)."""
    def op(f, k1, k2, _):
        d1 = 1j * _nyq0(k1, n1) * f
        d2 = 1j * _nyq0(k2, n2) * f
        return torch.stack([d1, d2], dim=-3)
    return distributed_spectral(comm, fields, n1, n2, op)


def distributed_divergence(comm, vs, n1, n2):
    """spectral::divergence (spectral.cpp:89-107) of slab vector fields (2, L, n2) -> (L, n2)."""
    def op(f, k1, k2, _):
        return 1j * _nyq0(k1, n1) * f[..., 0, :, :] + 1j * _nyq0(k2, n2) * f[..., 1, :, :]
    return distributed_spectral(comm, vs, n1, n2, op)


def _wave(n, device):
    k = torch.arange(n, device=device, dtype=torch.int64)
    return torch.where(k <= n // 2, k, k - n)  # fft.cpp:80


def distributed_resample(comm, fields, n1, n2, t1, t2):
    """spectral::resample (spectral.cpp:157-186) of slab fields (m, n1/G, n2) -> (m, t1/G, t2):
    modes |k_i| < min(n_i, t_i)/2 kept (truncation or zero padding), amplitude x t1 t2 / (n1 n2);
    the distributed 2-D FFT of distributed_spectral with the row count changing between the
    forward and the inverse column transforms."""
    G = comm.size
    ncs, nct = n2 // 2 + 1, t2 // 2 + 1
    wc = -(-nct // G)
    band1, band2 = min(n1, t1) // 2, min(n2, t2) // 2
    amp = (t1 * t2) / (n1 * n2)
    Lt = t1 // G
    take = min(ncs, nct)
    send = []
    for f in fields:
        sp = torch.fft.rfft(f, dim=-1)[..., :take]
        sp = torch.nn.functional.pad(sp, (0, G * wc - take))
        send.append([sp[..., q * wc:(q + 1) * wc].contiguous() for q in range(G)])
    recv = comm.alltoall(send)
    back = []
    for k, q in enumerate(comm.ranks):
        col = torch.fft.fft(torch.cat(recv[k], dim=-2), dim=-2)  # (m, n1, wc)
        dev = col.device
        kt = _wave(t1, dev)
        keep = kt.abs() < band1
        rows = torch.remainder(kt[keep], n1)
        out = torch.zeros(col.shape[:-2] + (t1, wc), dtype=col.dtype, device=dev)
        out[..., keep, :] = amp * col[..., rows, :]
        cidx = q * wc + torch.arange(wc, device=dev)
        out[..., :, (cidx >= band2) | (cidx >= nct)] = 0
        col = torch.fft.ifft(out, dim=-2)
        back.append([col[..., r * Lt:(r + 1) * Lt, :].contiguous() for r in range(G)])
    got = comm.alltoall(back)
    return [torch.fft.irfft(torch.cat(got[k], dim=-1)[..., :nct], n=t2, dim=-1) for k in range(len(comm.ranks))]


def distributed_cutoff_high(comm, fields, n1, n2):
    """spectral::cutoffFilter(., High) (spectral.cpp:188-203) of slab fields: the modes outside
    |k1| < n1/4 and |k2| < n2/4."""
    def op(f, k1, k2, _):
        low = (k1.abs() < n1 // 4) & (k2.abs() < n2 // 4)
        return torch.where(low, torch.zeros_like(f), f)
    return distributed_spectral(comm, fields, n1, n2, op)


def inv_half_symbol(k1, k2, norm, beta):
    """(beta gamma_reg)^(-1/2) (spectral.cpp:46-66, 121-131): gamma = |k|^(2p) by repeated
    multiplication, gamma_reg(0) = 1, then a correctly rounded square root and division."""
    ksq = k1 * k1 + k2 * k2
    gam = ksq
    for _ in range(int(norm) - 1):
        gam = gam * ksq
    gam = torch.where(gam == 0, torch.ones_like(gam), gam)
    return 1.0 / torch.sqrt(beta * gam)


def tridiag_max_eig(alpha, beta):
    """tridiagMaxEig (precond.cpp:88-117): Sturm bisection, 100 halvings."""
    m = len(alpha)
    if m == 1:
        return alpha[0]
    lo = hi = alpha[0]
    for i in range(m):
        off = (abs(beta[i - 1]) if i > 0 else 0.0) + (abs(beta[i]) if i < m - 1 else 0.0)
        lo = min(lo, alpha[i] - off)
        hi = max(hi, alpha[i] + off)

    def count_below(x):
        count, d = 0, 1.0
        for i in range(m):
            offsq = beta[i - 1] * beta[i - 1] if i > 0 else 0.0
            d = alpha[i] - x - offsq / d
            if d == 0.0:
                d = -1e-300
            if d < 0.0:
                count += 1
        return count

    for _ in range(100):
        mid = 0.5 * (lo + hi)
        if count_below(mid) >= m:
            hi = mid
        else:
            lo = mid
    return 0.5 * (lo + hi)


# ------------------------------------------------------------------------------ operator
class SlabHessian:
    """GN Hessian matvec of one grid decomposed over comm's ranks (see the module docstring)."""

    def __init__(self, ctx, comm, n1, n2, nt, norm, beta, parts, reach_rows):
        """parts[i]: dict of rank i's slab tensors: Xf, Xb (2, L, n2), G (nt+1, 2, L, n2),
        GD (nt, 2, L, n2), dv, dvd (L, n2)."""
        self.ctx, self.comm = ctx, comm
        self.n1, self.n2, self.nt, self.norm, self.beta = n1, n2, nt, norm, beta
        self.geo = SlabGeometry(n1, n2, comm.size, reach_rows)
        self.parts = parts
        g = self.geo
        dev = ctx.device
        self._alloc_windows()
        self.scr = [ctx.empty(g.L, n2) for _ in comm.ranks]
        self.vtD = [ctx.empty(2, g.L, n2) for _ in comm.ranks]
        self.b = [ctx.empty(2, g.L, n2) for _ in comm.ranks]
        self.partials = [ctx.empty(nt + 1, g.L) for _ in comm.ranks]
        self.flags = [torch.zeros(nt + 2, dtype=torch.int32, device=dev) for _ in comm.ranks]

    def _alloc_windows(self):
        g, ctx, n2 = self.geo, self.ctx, self.n2
        self.win = [ctx.empty(g.win_rows, n2 + 3) for _ in self.comm.ranks]
        self.winv = [ctx.empty(2, g.win_rows, n2 + 3) for _ in self.comm.ranks]
        # row-filtered fields live inside their halo buffers (rows [top, top+L)), so a step's
        # output needs no copy before the exchange
        self.halo = [ctx.empty(g.top + g.L + g.bot, n2) for _ in self.comm.ranks]
        self.rows = [h[g.top:g.top + g.L] for h in self.halo]

    # -- construction from the single-device operator (per-iterate invariants, sliced)
    @classmethod
    def from_operator(cls, ctx, comm, H: api.HessianOperator, norm, beta):
        n1, n2 = H.shape
        nt = H.nt
        ptrs = (C.c_void_p * 7)()
        ctx.check(ctx.lib.vrg_hess_buffers(H.h, ptrs))
        N = n1 * n2

        def view(ptr, count):
            return _DeviceView(ptr, count, ctx.device).tensor()

        G = view(ptrs[1], (nt + 1) * 2 * N).view(nt + 1, 2, n1, n2)
        GD = view(ptrs[2], nt * 2 * N).view(nt, 2, n1, n2)
        Xf = view(ptrs[3], 2 * N).view(2, n1, n2)
        Xb = view(ptrs[4], 2 * N).view(2, n1, n2)
        dv = view(ptrs[5], N).view(n1, n2)
        dvd = view(ptrs[6], N).view(n1, n2)
        L = n1 // comm.size
        parts = []
        reach = 0.0
        for i in comm.ranks:
            s = slice(i * L, (i + 1) * L)
            p = dict(Xf=Xf[:, s].clone(), Xb=Xb[:, s].clone(), G=G[:, :, s].clone(), GD=GD[:, :, s].clone(),
                     dv=dv[s].clone(), dvd=dvd[s].clone())
            reach = max(reach, row_reach(p["Xf"][0], n1, i * L), row_reach(p["Xb"][0], n1, i * L))
            parts.append(p)
        reach = float(comm.allreduce_max([torch.tensor(reach)] * len(comm.ranks))[0])
        if not math.isfinite(reach):
            raise api.InvalidArgument("evaluate: non-finite point coordinate")
        return cls(ctx, comm, n1, n2, nt, norm, beta, parts, math.ceil(reach) + 3)

    # -- distributed construction (every per-iterate invariant computed on the slabs)
    @classmethod
    def build(cls, ctx, comm, vs, mTs, n1, nt, norm, beta):
        """HessianOperator ctor (inverse.cpp:150-175) + the lazy per-velocity caches of its
        Solver (transport.cpp:91-127) on the slabs: vs[i] = (2, L, n2) velocity rows of rank i,
        mTs[i] = (L, n2) template rows.  Departure points by the Heun trace (transport.cpp:60-89,
        same rounding steps as EpiTrace), the state by slab SL steps with the guard, gradients
        and div v by the distributed FFT, (grad m)_D and (div v)_D by slab interpolation."""
        X = cls.trace(ctx, comm, vs, n1, nt, norm, beta, ("Xf", "Xb"))
        S = cls.for_points(ctx, comm, X, n1, vs[0].shape[-1], nt, norm, beta)
        ms = S.state(X["Xf"], mTs)
        S.derive(vs, X, ms)
        S.add_gd()
        return S

    @classmethod
    def trace(cls, ctx, comm, vs, n1, nt, norm, beta, dirs):
        """traceCharacteristics (transport.cpp:60-89) on the slabs for the directions in dirs
        ("Xf" forward, "Xb" backward): {name: [per-rank (2, L, n2)]}."""
        n2 = vs[0].shape[-1]
        G = comm.size
        L = n1 // G
        ht = 1.0 / nt
        h1, h2 = 2 * math.pi / n1, 2 * math.pi / n2
        vmax = float(comm.allreduce_max([v[0].abs().amax() for v in vs])[0])
        if not math.isfinite(vmax):
            raise api.InvalidArgument("transport velocity: non-finite value")
        # trace: the star and departure points move by at most ht max|v1| along axis 1
        tr = cls(ctx, comm, n1, n2, nt, norm, beta, None, math.ceil(ht * vmax / h1) + 3)
        for c in range(2):
            tr._prefilter([v[c] for v in vs], [w[c] for w in tr.winv])
        X = {}
        for sgn, name in ((1.0, "Xf"), (-1.0, "Xb")):
            if name not in dirs:
                continue
            xs = []
            for i, q in enumerate(comm.ranks):
                dev = vs[i].device
                i1 = (q * L + torch.arange(L, device=dev, dtype=torch.float64))[:, None]
                i2 = torch.arange(n2, device=dev, dtype=torch.float64)[None, :]
                c1 = (-math.pi) + h1 * i1
                c2 = (-math.pi) + h2 * i2
                star = torch.stack([c1 - (sgn * ht) * vs[i][0], c2 - (sgn * ht) * vs[i][1]])
                vstar = ctx.empty(2, L, n2)
                for c in range(2):
                    tr._step(i, KIND_STORE, tr.winv[i][c], star, [vstar[c]], ht, 0.0, tr.scr[i], tr.partials[i][0],
                             None)
                sh = sgn * 0.5 * ht
                xs.append(torch.stack([c1 - sh * (vs[i][0] + vstar[0]), c2 - sh * (vs[i][1] + vstar[1])]))
            X[name] = xs
        tr._check_window()
        return X

    @classmethod
    def for_points(cls, ctx, comm, X, n1, n2, nt, norm, beta):
        """An operator whose coefficient windows cover the departure displacement of the
        point sets in X (max over ranks)."""
        L = n1 // comm.size
        reach = max(row_reach(xs[i][0], n1, q * L) for xs in X.values() for i, q in enumerate(comm.ranks))
        reach = float(comm.allreduce_max([torch.tensor(reach)] * len(comm.ranks))[0])
        if not math.isfinite(reach):
            raise api.InvalidArgument("evaluate: non-finite point coordinate")
        return cls(ctx, comm, n1, n2, nt, norm, beta, None, math.ceil(reach) + 3)

    def state(self, Xf, mTs):
        """slState with the guard (transport.cpp:214-227): per-rank (nt+1, L, n2) trajectories."""
        ctx, comm, nt = self.ctx, self.comm, self.nt
        L, n2, ht = self.geo.L, self.n2, 1.0 / nt
        ms = [ctx.empty(nt + 1, L, n2) for _ in comm.ranks]
        for i in range(len(comm.ranks)):
            ms[i][0].copy_(mTs[i])
            self.partials[i].zero_()
            self.flags[i].zero_()
            self.partials[i][0][:L].copy_(mTs[i].abs().amax(dim=1))
            self.flags[i][0] = (~torch.isfinite(mTs[i])).any().to(self.flags[i].dtype)  # prefilter input check
        self._prefilter([m[0] for m in ms], self.win)
        for j in range(1, nt + 1):
            if j > 1:
                self._windows_from_rows()
            for i in range(len(comm.ranks)):
                self._step(i, KIND_STATE, self.win[i], Xf[i], [ms[i][j]], ht, 0.0, self.rows[i], self.partials[i][j],
                           self.flags[i][j:j + 1])
        self._check_state_guard()
        return ms

    def derive(self, vs, X, ms):
        """grad m_j, div v and (div v)_D of the state ms at velocity vs (the lazy caches of the
        GN operator and of evaluateGradient's adjoint / body force)."""
        ctx, comm, nt, n1, n2 = self.ctx, self.comm, self.nt, self.n1, self.n2
        L, ht = self.geo.L, 1.0 / nt
        grads = distributed_gradient(comm, ms, n1, n2)  # (nt+1, 2, L, n2) per rank
        dvs = distributed_divergence(comm, vs, n1, n2)
        self._prefilter(dvs, self.win)
        dvds = [ctx.empty(L, n2) for _ in comm.ranks]
        for i in range(len(comm.ranks)):
            self._step(i, KIND_STORE, self.win[i], X["Xb"][i], [dvds[i]], ht, 0.0, self.scr[i], self.partials[i][0],
                       None)
        self._check_window()
        self.parts = [dict(Xf=X["Xf"][i], Xb=X["Xb"][i], G=grads[i], dv=dvs[i], dvd=dvds[i], m=ms[i])
                      for i in range(len(comm.ranks))]

    def add_gd(self):
        """(grad m_{j-1})_D at the forward departure points: the last per-iterate invariant of
        the GN operator (inverse.cpp:177-187)."""
        ctx, comm, nt = self.ctx, self.comm, self.nt
        L, n2, ht = self.geo.L, self.n2, 1.0 / nt
        gds = [ctx.empty(nt, 2, L, n2) for _ in comm.ranks]
        for j in range(1, nt + 1):
            for c in range(2):
                self._prefilter([p["G"][j - 1][c] for p in self.parts], self.win)
                for i in range(len(comm.ranks)):
                    self._step(i, KIND_STORE, self.win[i], self.parts[i]["Xf"], [gds[i][j - 1][c]], ht, 0.0,
                               self.scr[i], self.partials[i][0], None)
        self._check_window()
        for i, p in enumerate(self.parts):
            p["GD"] = gds[i]

    def gradient(self, mRs, regs, outs):
        """evaluateGradient's adjoint and body force (inverse.cpp:130-146, SL): lambda(1) =
        -(m(1) - m_R), the adjoint solved back with the guard, b = sum_j w_j lambda_j grad m_j
        accumulated by the adjoint steps, outs[i] = beta A v + b (compressible)."""
        nt, ht = self.nt, 1.0 / self.nt
        ranks = range(len(self.comm.ranks))
        wof = lambda j: ht * (0.5 if j in (0, nt) else 1.0)  # noqa: E731
        lams = []
        for i in ranks:
            p = self.parts[i]
            lam = -1.0 * (p["m"][nt] - mRs[i])
            lams.append(lam)
            self.flags[i].zero_()
            self.partials[i].zero_()
            self.partials[i][nt][:self.geo.L].copy_(lam.abs().amax(dim=1))
            self.flags[i][nt] = (~torch.isfinite(lam)).any().to(self.flags[i].dtype)
            self.b[i][0].copy_(wof(nt) * (lam * p["G"][nt][0]))
            self.b[i][1].copy_(wof(nt) * (lam * p["G"][nt][1]))
        self._prefilter(lams, self.win)
        for j in range(nt, 0, -1):
            if j < nt:
                self._windows_from_rows()
            for i in ranks:
                p = self.parts[i]
                ops = [p["dvd"], p["dv"], p["G"][j - 1][0], p["G"][j - 1][1], self.b[i][0], self.b[i][1]]
                if j == 1:
                    ops += [regs[i][0], regs[i][1], outs[i][0], outs[i][1]]
                    self._step(i, KIND_ADJ_LAST, self.win[i], p["Xb"], ops, ht, wof(0), self.scr[i],
                               self.partials[i][0], None)
                else:
                    self._step(i, KIND_ADJ, self.win[i], p["Xb"], ops, ht, wof(j - 1), self.rows[i],
                               self.partials[i][j - 1], self.flags[i][j - 1:j])
        self._check_guard()
        return lams

    def _check_window(self):
        fl = self.comm.allreduce_max([f.to(torch.float64) for f in self.flags])[0].cpu()
        if fl[self.nt + 1] != 0:
            raise api.VrgError("slab window too small for the departure displacement")

    def _check_state_guard(self):
        """checkGuard of slState (transport.cpp:16-20, 221): ||m_j|| <= 1e3 ||m_0||, forward."""
        nt = self.nt
        mx = self.comm.allreduce_max([p.amax(dim=1) for p in self.partials])[0].cpu()
        fl = self.comm.allreduce_max([f.to(torch.float64) for f in self.flags])[0].cpu()
        if fl[nt + 1] != 0:
            raise api.VrgError("slab window too small for the departure displacement")
        threshold = 1e3 * float(mx[0])
        for j in range(1, nt + 1):
            if fl[j - 1] != 0:
                raise api.InvalidArgument("prefilter: non-finite value")
            if float(mx[j]) > threshold:
                raise api.BlowupError(f"state solve exceeded the blow-up guard at step {j}")

    # -- building blocks
    def _prefilter(self, fields, windows):
        """Coefficient windows of slab fields (per rank (L, n2)): row pass, halo exchange,
        column pass."""
        g, ctx = self.geo, self.ctx
        for i, f in enumerate(fields):
            ctx.check(ctx.lib.vrg_prefilter_rows(ctx.h, g.L, self.n2, api._p(f), api._p(self.rows[i]), None))
        self.comm.fill_halos(self.halo, g.L, g.top, g.bot)
        for i, hb in enumerate(self.halo):
            ctx.check(ctx.lib.vrg_slab_cols(ctx.h, g.win_rows, self.n2, api._p(hb), api._p(windows[i])))

    def _windows_from_rows(self):
        """Coefficient windows from the row-filtered step outputs in self.rows."""
        g, ctx = self.geo, self.ctx
        self.comm.fill_halos(self.halo, g.L, g.top, g.bot)
        for i, hb in enumerate(self.halo):
            ctx.check(ctx.lib.vrg_slab_cols(ctx.h, g.win_rows, self.n2, api._p(hb), api._p(self.win[i])))

    def _step(self, i, kind, coef, X, ops, ht, w, row_out, partial, flag):
        g, ctx = self.geo, self.ctx
        arr = (C.c_void_p * len(ops))(*[o.data_ptr() for o in ops])
        ctx.check(ctx.lib.vrg_slab_step(ctx.h, kind, self.n1, self.n2, g.L, g.win_base(self.comm.ranks[i]),
                                        g.win_rows, api._p(coef), api._p(X[0]), api._p(X[1]), arr, len(ops),
                                        ht, w, api._p(row_out), api._p(partial),
                                        C.c_void_p(flag.data_ptr()) if flag is not None else None,
                                        C.c_void_p(self.flags[i][self.nt + 1:].data_ptr())))

    def reg(self, vts):
        return distributed_reg(self.comm, vts, self.n1, self.n2, self.norm, self.beta)

    # The per-step orchestration of a slab matvec (one library call and one halo exchange per SL
    # step, from Python) is captured into one CUDA graph per (inputs, outputs) and replayed: the
    # first `capture_after` applies of a pointer set run eagerly (warming every buffer), the next
    # captures on the context's stream, later ones replay; the guard check stays on the host
    # after the replay.  `graphs = False` keeps every apply eager.  With NCCL exchanges between processes
    # (DistComm, more than one rank) the capture is opt-in (`graphs_multirank`) until it has run
    # on a multi-GPU node; in-process slabs (LocalComm) and a one-rank group capture by default.
    graphs = True
    graphs_multirank = False
    capture_after = 8  # an operator rebuilt every Newton iteration applies ~4 times: stays eager

    def apply_staged(self, vts, data_term_only=False):
        """apply() through persistent input / output slabs owned by the operator (copies of vts
        in, the result out): callers whose temporaries change address every call keep one
        pointer set, so the captured graph replays."""
        if not hasattr(self, "_stage_in"):
            g = self.geo
            self._stage_in = [self.ctx.empty(2, g.L, self.n2) for _ in self.comm.ranks]
            self._stage_out = [self.ctx.empty(2, g.L, self.n2) for _ in self.comm.ranks]
        for dst, src in zip(self._stage_in, vts):
            dst.copy_(src)
        return self.apply(self._stage_in, self._stage_out, data_term_only=data_term_only)

    def _capturable(self, vts):
        if not self.graphs or not vts[0].is_cuda:
            return False
        return isinstance(self.comm, LocalComm) or self.comm.size == 1 or self.graphs_multirank

    def apply(self, vts, outs=None, data_term_only=False):
        """vts[i] = (2, L, n2) slab of vt on rank i -> H vt slabs (or the data term b)."""
        ranks = range(len(self.comm.ranks))
        outs = outs if outs is not None else [self.ctx.empty(2, self.geo.L, self.n2) for _ in ranks]
        if not self._capturable(vts):
            self._apply_body(vts, outs, data_term_only)
        else:
            key = (tuple(t.data_ptr() for vt in vts for t in vt), tuple(o.data_ptr() for o in outs), data_term_only)
            cache = self.__dict__.setdefault("_graph_cache", {})
            entry = cache.get(key)
            if entry is None and len(cache) >= 16:  # a caller cycling through many buffers
                cache.clear()
            if entry is None or (isinstance(entry, int) and entry < self.capture_after):
                # eager until the pointer set has proved reused: a capture (its eager-speed run
                # plus the graph instantiation) pays off only over several replays (the coarse
                # level's Chebyshev loops), not for an operator rebuilt every Newton iteration
                self._apply_body(vts, outs, data_term_only)
                cache[key] = (entry or 0) + 1
            elif isinstance(entry, int):
                try:
                    graph = torch.cuda.CUDAGraph()
                    graph.capture_begin(capture_error_mode="thread_local")
                    try:
                        self._apply_body(vts, outs, data_term_only)
                    finally:
                        graph.capture_end()
                except Exception:  # noqa: BLE001 - not capturable here (e.g. the backend): stay eager
                    self.graphs = False
                    self._apply_body(vts, outs, data_term_only)
                else:
                    cache[key] = graph
                    graph.replay()
            else:
                entry.replay()
        self._check_guard()
        return outs

    def _apply_body(self, vts, outs, data_term_only):
        """The launch sequence of one slab matvec (no host synchronisation: capturable)."""
        nt, ht = self.nt, 1.0 / self.nt
        ranks = range(len(self.comm.ranks))
        regs = self.reg(vts) if not data_term_only else None
        for i in ranks:
            self.flags[i].zero_()
            self.partials[i].zero_()
        wof = lambda j: ht * (0.5 if j in (0, nt) else 1.0)  # noqa: E731
        # vt_D (2 interps)
        for c in range(2):
            self._prefilter([vt[c] for vt in vts], [wv[c] for wv in self.winv])
        for i in ranks:
            for c in range(2):
                self._step(i, KIND_STORE, self.winv[i][c], self.parts[i]["Xf"], [self.vtD[i][c]], ht, 0.0,
                           self.scr[i], self.partials[i][0], None)
        # incremental state, the last step seeding the adjoint
        for j in range(1, nt + 1):
            if j > 1:
                self._windows_from_rows()
            for i in ranks:
                p = self.parts[i]
                ops = [self.vtD[i][0], self.vtD[i][1], p["GD"][j - 1][0], p["GD"][j - 1][1], vts[i][0], vts[i][1],
                       p["G"][j][0], p["G"][j][1]]
                if j == nt:
                    kind = KIND_SEED0 if j == 1 else KIND_SEED
                    ops += [self.b[i][0], self.b[i][1]]
                    self._step(i, kind, self.win[i], p["Xf"], ops, ht, wof(nt), self.rows[i], self.partials[i][nt],
                               self.flags[i][nt:nt + 1])
                else:
                    kind = KIND_INC0 if j == 1 else KIND_INC
                    self._step(i, kind, self.win[i], p["Xf"], ops, ht, 0.0, self.rows[i], self.partials[i][0], None)
        # incremental adjoint + body force (+ beta A vt on the last step)
        for j in range(nt, 0, -1):
            self._windows_from_rows()
            for i in ranks:
                p = self.parts[i]
                ops = [p["dvd"], p["dv"], p["G"][j - 1][0], p["G"][j - 1][1], self.b[i][0], self.b[i][1]]
                if j == 1:
                    if data_term_only:
                        zero = torch.zeros_like(self.b[i])
                        ops += [zero[0], zero[1], outs[i][0], outs[i][1]]
                    else:
                        ops += [regs[i][0], regs[i][1], outs[i][0], outs[i][1]]
                    self._step(i, KIND_ADJ_LAST, self.win[i], p["Xb"], ops, ht, wof(0), self.scr[i],
                               self.partials[i][0], None)
                else:
                    self._step(i, KIND_ADJ, self.win[i], p["Xb"], ops, ht, wof(j - 1), self.rows[i],
                               self.partials[i][j - 1], self.flags[i][j - 1:j])

    def _check_guard(self):
        """transport.cpp:16-20 guard of the GN adjoint (inverse.cpp:185) over all slabs, in the
        reference's step order, and the window/finiteness flags."""
        nt = self.nt
        mx = self.comm.allreduce_max([p.amax(dim=1) for p in self.partials])[0].cpu()
        fl = self.comm.allreduce_max([f.to(torch.float64) for f in self.flags])[0].cpu()
        if fl[nt + 1] != 0:
            raise api.VrgError("slab window too small for the departure displacement")
        threshold = 1e3 * float(mx[nt])
        for s in range(1, nt + 1):
            j = nt + 1 - s
            if fl[j] != 0:
                raise api.InvalidArgument("prefilter: non-finite value")
            if float(mx[j - 1]) > threshold:
                raise api.BlowupError(f"adjoint solve exceeded the blow-up guard at step {j}")


class SlabCoarse:
    """precond::CoarseOperator (precond.cpp:163-171, 207-240) on half-grid slabs: the problem and
    the velocity restricted by distributed spectral truncation, the coarse nt from the CFL-5 rule
    (transport.cpp:44-50, maxima over ranks), a slab GN operator at the coarse velocity, and the
    pieces of the two-level CHEB preconditioner (precond.cpp:180-205, 264-289) and of the
    Chebyshev bound re-estimate (lanczosEmax, precond.cpp:120-161) on those slabs."""

    def __init__(self, ctx, comm, vs, mRs, mTs, n1, n2, norm, beta, cfl=5.0):
        self.ctx, self.comm = ctx, comm
        self.n1, self.n2, self.t1, self.t2 = n1, n2, n1 // 2, n2 // 2
        if self.t1 % comm.size:
            raise api.InvalidArgument("slab decomposition: the coarse grid's n1 must be a multiple of the ranks")
        self.norm, self.beta = norm, beta
        self.vc = distributed_resample(comm, vs, n1, n2, self.t1, self.t2)
        ims = distributed_resample(comm, [torch.stack([r, t]) for r, t in zip(mRs, mTs)], n1, n2, self.t1, self.t2)
        self.mTc = [im[1].contiguous() for im in ims]
        h1, h2 = 2 * math.pi / self.t1, 2 * math.pi / self.t2
        m1 = float(comm.allreduce_max([v[0].abs().amax() for v in self.vc])[0])
        m2 = float(comm.allreduce_max([v[1].abs().amax() for v in self.vc])[0])
        ratio = max(0.0, m1 / (cfl * h1), m2 / (cfl * h2))
        self.nt = max(2, int(math.ceil(ratio)))
        self.S = SlabHessian.build(ctx, comm, self.vc, self.mTc, self.t1, self.nt, norm, beta)

    def _dot(self, a, b):
        h = (2 * math.pi / self.t1) * (2 * math.pi / self.t2)
        return h * float(self.comm.allreduce_sum([torch.sum(x * y).reshape(1) for x, y in zip(a, b)])[0].item())

    def split(self, ss):
        """applySplitHessianOf (precond.cpp:20-26): M^{-1/2} Q M^{-1/2} s + s on coarse slabs."""
        op = lambda f, k1, k2, _: f * inv_half_symbol(k1, k2, self.norm, self.beta)  # noqa: E731
        t = distributed_spectral(self.comm, ss, self.t1, self.t2, op)
        b = self.S.apply_staged(t, data_term_only=True)
        o = distributed_spectral(self.comm, b, self.t1, self.t2, op)
        return [x + s for x, s in zip(o, ss)]

    def chebyshev(self, rhs, k, emin, emax):
        """chebyshevSolve (precond.cpp:180-205): x_0 = 0, exactly k operator applications."""
        theta, delta = 0.5 * (emax + emin), 0.5 * (emax - emin)
        sigma = theta / delta
        rho = 1.0 / sigma
        x = [torch.zeros_like(r) for r in rhs]
        r = [t.clone() for t in rhs]
        d = [(1.0 / theta) * t for t in r]
        for it in range(1, k + 1):
            if it > 1:
                rho_new = 1.0 / (2.0 * sigma - rho)
                d = [(rho_new * rho) * di + (2.0 * rho_new / delta) * ri for di, ri in zip(d, r)]
                rho = rho_new
            x = [xi + di for xi, di in zip(x, d)]
            ad = self.split(d)
            r = [ri - ai for ri, ai in zip(r, ad)]
        return x

    def two_level(self, rs, k, emin, emax):
        """applyTwoLevel (precond.cpp:264-289), CHEB(k): the low band restricted (the cutoff band
        is the restriction band), solved, prolonged, plus the high band; (z slabs, diverged)."""
        rc = distributed_resample(self.comm, rs, self.n1, self.n2, self.t1, self.t2)
        high = distributed_cutoff_high(self.comm, rs, self.n1, self.n2)
        sc = self.chebyshev(rc, k, emin, emax)
        bad = torch.tensor(float(any(not bool(torch.isfinite(x).all()) for x in sc)))
        if float(self.comm.allreduce_max([bad] * len(self.comm.ranks))[0]) > 0:
            return [r.clone() for r in rs], True
        up = distributed_resample(self.comm, sc, self.t1, self.t2, self.n1, self.n2)
        return [u + h for u, h in zip(up, high)], False

    def lanczos_emax(self, steps=30, seed=0x5EED):
        """lanczosEmax (precond.cpp:120-161) of the coarse split operator from the seeded band-limited
        probe (the library's randomBandLimitedVelocity on the whole coarse grid, sliced); returns
        (eMax, operator applications)."""
        Lc = self.t1 // self.comm.size
        probe = api.random_bandlimited_velocity(self.ctx, (self.t1, self.t2), seed)
        q = [torch.stack([probe[0][r * Lc:(r + 1) * Lc], probe[1][r * Lc:(r + 1) * Lc]]).contiguous()
             for r in self.comm.ranks]
        nq = math.sqrt(self._dot(q, q))
        if not nq > 0.0:
            return 1.0, 0
        q = [(1.0 / nq) * x for x in q]
        basis, alpha, beta, applied = [q], [], [], 0
        for j in range(steps):
            w = self.split(basis[j])
            applied += 1
            if j > 0:
                w = [wi + (-beta[j - 1]) * bi for wi, bi in zip(w, basis[j - 1])]
            a = self._dot(w, basis[j])
            alpha.append(a)
            w = [wi + (-a) * bi for wi, bi in zip(w, basis[j])]
            for qi in basis:
                c = self._dot(w, qi)
                w = [wi + (-c) * qq for wi, qq in zip(w, qi)]
            b = math.sqrt(self._dot(w, w))
            if not math.isfinite(b):
                raise api.NotSupported("slab coarse Lanczos broke down (non-finite); the power-iteration fallback "
                                       "of precond.cpp:153 is not implemented on the slabs")
            if b < 1e-12:
                break
            beta.append(b)
            basis.append([(1.0 / b) * wi for wi in w])
        return tridiag_max_eig(alpha, beta[:len(alpha) - 1]), applied


class SlabFineOperator:
    """Slab-decomposed operators for `api.newton_solve(..., fine_operator=...)` (config 5a).

    The library's Newton driver (newton.cpp:24-159, host C++) keeps the control flow and the
    whole-grid vectors (v, g, the PCG vectors); the transport-heavy parts run decomposed, each
    rank on its rows (halo exchanges and all-to-all FFT transposes inside), their slab outputs
    all-gathered back into the driver's fields:
      * build(v, nt) per outer iteration and data_term(vt) -> b per fine matvec (the
        precond::LinOp plug-in point, precond.hpp:25, C ABI vrg_set_fine_operator);
      * with mR given, also gradient(v, nt, reuse) -> g, m(1) and the objective terms
        (evaluateGradient, inverse.cpp:119-148) and objective(v, nt) per line-search trial
        (evaluateObjective, inverse.cpp:96-117), C ABI vrg_set_external_ops: the state, adjoint
        and body force of the gradient and the state of every trial are slab SL solves, and
        the Hessian's per-iterate invariants reuse the gradient's (trace, state, grad m_j, div v);
      * and, where the half grid fits the slab step, the two-level CHEB preconditioner's coarse
        level (SlabCoarse: restriction, coarse GN operator, Chebyshev, prolongation, the bound
        re-estimate) on half-grid slabs.
    What stays replicated is the vector algebra of the driver and the eigenvalue estimate at
    v = 0 made once per solve.  All ranks call the hooks in the same order because the
    driver is deterministic and sees identical data; every callback reaches a common verdict."""

    def __init__(self, ctx, comm, mT, norm, beta, mR=None):
        import numpy as np

        self.ctx, self.comm = ctx, comm
        mT = ctx.field(np.asarray(mT) if not torch.is_tensor(mT) else mT)
        self.n1, self.n2 = int(mT.shape[0]), int(mT.shape[1])
        if self.n1 % comm.size:
            raise api.InvalidArgument("slab decomposition: n1 must be a multiple of the number of ranks")
        self.norm, self.beta = int(norm), float(beta)
        self.L = self.n1 // comm.size
        self.mTs = [mT[q * self.L:(q + 1) * self.L].contiguous() for q in comm.ranks]
        self.full = mR is not None
        if self.full:
            mR = ctx.field(np.asarray(mR) if not torch.is_tensor(mR) else mR)
            self.mRs = [mR[q * self.L:(q + 1) * self.L].contiguous() for q in comm.ranks]
        self.S = None
        self.error = None
        self._stage = None       # (v, SlabHessian with the gradient's invariants) of the iterate
        self._candidate = None   # (nt, Xf, state) of the last objective call (the accepted trial)
        self.builds = self.matvecs = self.gradients = self.objectives = 0
        self.build_s = self.apply_s = self.gradient_s = self.objective_s = 0.0
        self._cb_build = api.FINE_BUILD_FN(self._build)
        self._cb_data_term = api.FINE_DATA_TERM_FN(self._data_term)
        self._cb_gradient = api.GRADIENT_FN(self._gradient)
        self._cb_objective = api.OBJECTIVE_FN(self._objective)
        self._cb_coarse_build = api.COARSE_BUILD_FN(self._coarse_build)
        self._cb_two_level = api.TWO_LEVEL_FN(self._two_level)
        self._cb_coarse_emax = api.COARSE_EMAX_FN(self._coarse_emax)
        self._cb_split = api.SPLIT_FN(self._split)
        self.coarse = None
        # the coarse level on slabs too where its rows fit the slab step (half-grid rows of a
        # multiple of 256 up to 4096, half-grid n1 divisible by the ranks); else the driver's
        # own coarse operator, replicated
        c1, c2 = self.n1 // 2, self.n2 // 2
        self.coarse_slabs = self.full and c2 % 256 == 0 and 256 <= c2 <= 4096 and c1 % comm.size == 0
        self.coarse_builds = self.precond_applies = 0
        self.coarse_s = self.precond_s = 0.0

    def callbacks(self):
        cbs = {"build": self._cb_build, "data_term": self._cb_data_term}
        if self.full:
            cbs.update(gradient=self._cb_gradient, objective=self._cb_objective, split=self._cb_split)
        if self.coarse_slabs:
            cbs.update(coarse_build=self._cb_coarse_build, two_level=self._cb_two_level,
                       coarse_emax=self._cb_coarse_emax)
        return cbs

    def _full(self, ptr, comps=2):
        N = self.n1 * self.n2
        t = _DeviceView(ptr, comps * N, self.ctx.device).tensor()
        return t.view(comps, self.n1, self.n2) if comps > 1 else t.view(self.n1, self.n2)

    def _slabs(self, f):
        L = self.L
        return [f[..., q * L:(q + 1) * L, :].contiguous() for q in self.comm.ranks]

    def _verdict(self, failed: bool) -> int:
        """Every rank returns the same status: the driver aborts on all ranks together instead
        of one rank leaving while the others wait in its next collective."""
        try:
            anyf = self.comm.any_failed(failed)
        except BaseException as e:  # the verdict itself failed: fail locally
            self.error = self.error or e
            return 1
        if anyf and self.error is None:
            self.error = RuntimeError("slab fine operator failed on another rank")
        return 1 if anyf else 0

    def _dot(self, a, b):
        """dot (field.cpp:51-57) of slab fields, summed over ranks: h1 h2 sum(a b)."""
        h = (2 * math.pi / self.n1) * (2 * math.pi / self.n2)
        part = [torch.sum(x * y).reshape(1) for x, y in zip(a, b)]
        return h * float(self.comm.allreduce_sum(part)[0].item())

    def _objective_terms(self, vs, ms, nt):
        """mismatch = 1/2 |m(1) - m_R|^2 and regTerm = 1/2 <beta A v, v> (inverse.cpp:104-108);
        returns them with beta A v."""
        resid = [m[nt] - r for m, r in zip(ms, self.mRs)]
        mismatch = 0.5 * self._dot(resid, resid)
        regs = distributed_reg(self.comm, vs, self.n1, self.n2, self.norm, self.beta)
        reg_term = 0.5 * self._dot(regs, vs)
        return mismatch, reg_term, regs

    @staticmethod
    def _scalars(ptr, mismatch, reg_term):
        out = (C.c_double * 4).from_address(ptr)
        out[0], out[1], out[2], out[3] = mismatch + reg_term, mismatch, reg_term, 0.0

    def _objective(self, _user, vptr, nt, m1ptr, scptr):
        import time

        failed, blowup = False, False
        try:
            t0 = time.perf_counter()
            vs = self._slabs(self._full(vptr))
            X = SlabHessian.trace(self.ctx, self.comm, vs, self.n1, int(nt), self.norm, self.beta, ("Xf",))
            S = SlabHessian.for_points(self.ctx, self.comm, X, self.n1, self.n2, int(nt), self.norm, self.beta)
            try:
                ms = S.state(X["Xf"], self.mTs)
            except api.BlowupError:  # common to all ranks: the guard reduces over them
                self._candidate = None
                blowup = True
            if not blowup:
                mismatch, reg_term, _ = self._objective_terms(vs, ms, int(nt))
                self._scalars(scptr, mismatch, reg_term)
                self.comm.allgather_rows([m[int(nt)].unsqueeze(0) for m in ms], self._full(m1ptr, 1).unsqueeze(0))
                self._candidate = (int(nt), X["Xf"], ms)
            self.objectives += 1
            self.objective_s += time.perf_counter() - t0
        except BaseException as e:
            self.error = e
            failed = True
        rc = self._verdict(failed)
        return rc if rc else (2 if blowup else 0)

    def _gradient(self, _user, vptr, nt, reuse, gptr, m1ptr, scptr):
        import time

        failed = False
        try:
            t0 = time.perf_counter()
            nt = int(nt)
            v = self._full(vptr)
            vs = self._slabs(v)
            if reuse and self._candidate is not None and self._candidate[0] == nt:
                _, Xf, ms = self._candidate  # the accepted trial's state (newton.cpp:54-56)
                X = dict(Xf=Xf, **SlabHessian.trace(self.ctx, self.comm, vs, self.n1, nt, self.norm, self.beta,
                                                    ("Xb",)))
                S = SlabHessian.for_points(self.ctx, self.comm, X, self.n1, self.n2, nt, self.norm, self.beta)
            else:
                X = SlabHessian.trace(self.ctx, self.comm, vs, self.n1, nt, self.norm, self.beta, ("Xf", "Xb"))
                S = SlabHessian.for_points(self.ctx, self.comm, X, self.n1, self.n2, nt, self.norm, self.beta)
                ms = S.state(X["Xf"], self.mTs)
            S.derive(vs, X, ms)
            mismatch, reg_term, regs = self._objective_terms(vs, ms, nt)
            outs = [self.ctx.empty(2, self.L, self.n2) for _ in self.comm.ranks]
            S.gradient(self.mRs, regs, outs)
            self.comm.allgather_rows(outs, self._full(gptr))
            self.comm.allgather_rows([m[nt].unsqueeze(0) for m in ms], self._full(m1ptr, 1).unsqueeze(0))
            self._scalars(scptr, mismatch, reg_term)
            self._stage = (v.clone(), nt, S)
            self._candidate = None
            self.gradients += 1
            self.gradient_s += time.perf_counter() - t0
        except BaseException as e:  # re-raised by api.newton_solve
            self.error = e
            failed = True
        return self._verdict(failed)

    def _build(self, _user, vptr, nt):
        import time

        failed = False
        try:
            t0 = time.perf_counter()
            self.S = None
            v = self._full(vptr)
            st = self._stage
            if st is not None and st[1] == int(nt) and torch.equal(st[0], v):
                S = st[2]  # the gradient's trace, state, grad m_j and div v at this iterate
                S.add_gd()
                self.S = S
            else:
                self.S = SlabHessian.build(self.ctx, self.comm, self._slabs(v), self.mTs, self.n1, int(nt),
                                           self.norm, self.beta)
            self._stage = None
            self.builds += 1
            self.build_s += time.perf_counter() - t0
        except BaseException as e:  # re-raised by api.newton_solve
            self.error = e
            failed = True
        return self._verdict(failed)

    def _coarse_build(self, _user, vptr, ntc_ptr):
        import time

        failed = False
        try:
            t0 = time.perf_counter()
            self.coarse = None
            self.coarse = SlabCoarse(self.ctx, self.comm, self._slabs(self._full(vptr)), self.mRs, self.mTs, self.n1,
                                     self.n2, self.norm, self.beta)
            ntc_ptr[0] = self.coarse.nt
            self.coarse_builds += 1
            self.coarse_s += time.perf_counter() - t0
        except BaseException as e:
            self.error = e
            failed = True
        return self._verdict(failed)

    def _two_level(self, _user, rptr, zptr, k, emin, emax):
        import time

        failed, diverged = False, False
        try:
            t0 = time.perf_counter()
            zs, diverged = self.coarse.two_level(self._slabs(self._full(rptr)), int(k), emin, emax)
            self.comm.allgather_rows(zs, self._full(zptr))
            self.precond_applies += 1
            self.precond_s += time.perf_counter() - t0
        except BaseException as e:
            self.error = e
            failed = True
        rc = self._verdict(failed)
        return rc if rc else (3 if diverged else 0)

    def _coarse_emax(self, _user, emax_ptr, applied_ptr):
        failed = False
        try:
            e, applied = self.coarse.lanczos_emax()
            emax_ptr[0] = e
            applied_ptr[0] = applied
        except BaseException as e:
            self.error = e
            failed = True
        return self._verdict(failed)

    def _split(self, _user, sptr, optr):
        """applySplitHessianOf (precond.cpp:20-26) on the slabs: t = M^{-1/2} s, the slab data term,
        o = M^{-1/2} b + s (the symbols by the distributed FFT)."""
        import time

        failed = False
        try:
            t0 = time.perf_counter()
            op = lambda f, k1, k2, _: f * inv_half_symbol(k1, k2, self.norm, self.beta)  # noqa: E731
            ss = self._slabs(self._full(sptr))
            t = distributed_spectral(self.comm, ss, self.n1, self.n2, op)
            b = self.S.apply_staged(t, data_term_only=True)
            o = distributed_spectral(self.comm, b, self.n1, self.n2, op)
            self.comm.allgather_rows([x + y for x, y in zip(o, ss)], self._full(optr))
            self.matvecs += 1
            self.apply_s += time.perf_counter() - t0
        except BaseException as e:
            self.error = e
            failed = True
        return self._verdict(failed)

    def _data_term(self, _user, vtptr, bptr):
        import time

        failed = False
        try:
            t0 = time.perf_counter()
            outs = self.S.apply_staged(self._slabs(self._full(vtptr)), data_term_only=True)
            self.comm.allgather_rows(outs, self._full(bptr))
            self.matvecs += 1
            self.apply_s += time.perf_counter() - t0
        except BaseException as e:
            self.error = e
            failed = True
        return self._verdict(failed)


class _DeviceView:
    """Zero-copy torch view of library-owned device memory (__cuda_array_interface__)."""

    def __init__(self, ptr, count, device):
        self.__cuda_array_interface__ = {"shape": (count,), "typestr": "<f8", "data": (int(ptr), False),
                                         "version": 2, "strides": None}
        self.device = device

    def tensor(self):
        return torch.as_tensor(self, device=self.device)
