#!/usr/bin/env python
"""Benchmark of the GN Hessian-matvec hot path (BASELINE config 4: 1024^2 fp64, nt=16, H2,
beta=1e-3, GN, SL) — one JSON line on rank 0.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl vrg|reference]

A step is one reduced-space GN Hessian matvec HessianOperator::apply(vtilde)
(src/inverse.cpp:229-233) at a fixed iterate, i.e. one pass of the hot path.  With N > 1
(torchrun, one process per GPU) every rank holds its own independent image pair and
iterate (batched pairs): no data-path collective, weak scaling.

`value`   : matvecs/s over all ranks, inputs resident in HBM, device-timed (CUDA events on
            the launching stream, barrier + synchronize on both sides, max over ranks): the K
            matvecs queued through vrg_hess_apply_batch (each matvec's guard checked on the
            host while the next runs); `per_call` the same with one vrg_hess_apply per matvec.
`e2e`     : the same metric through the drop-in host-buffer calls: every step's H2D of vtilde
            from pinned memory + matvec + D2H of the result inside the timed region;
            vrg_hess_apply_host_batch over the K steps (copies of neighbouring matvecs
            overlap the current one's compute), and `e2e.serial` one vrg_hess_apply_host per step.
`roofline`: dominant kernel of the matvec, algorithmic bytes / average launch time from
            per-launch CUDA events of a second (profiled) pass over the same K steps.
`cpu_baseline`: the unmodified reference (oracle/_ref) on the host cores, rank 0, N=1 only.
`--impl reference`: the reference CPU implementation on the host cores (all threads), same
            metric/config; ranks > 0 exit without work.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_GRID, NT, BETA, NORM = 1024, 16, 1e-3, 2
F_BYTES = 8 * N_GRID * N_GRID
METRIC = "GN Hessian matvecs/s at 1024^2 fp64 (nt=16, H2, SL)"
UNIT = "matvec/s"
CONFIG = {
    "workload": "config4: single GN Hessian matvec, 1024x1024 fp64, nt=16, H2 beta=1e-3, SL, compressible",
    "grid": [N_GRID, N_GRID], "nt": NT, "beta": BETA, "norm": "H2",
    "inputs": "seeded synthetic: smoothed-noise template (sigma=4 px), (1+|k|^2)^-2 random velocity max|v|=0.3",
    "l2": "per-matvec working set ~0.7 GB of cached state fields >> 126 MB L2 (inputs larger than L2)",
}


# ------------------------------------------------------------------------------ inputs
def make_problem(rank: int):
    from paper_1604_02153_b200 import synth

    mT = synth.smoothed_noise(N_GRID, N_GRID, 1000 + rank)
    v1, v2 = synth.smooth_velocity(N_GRID, N_GRID, 2000 + rank)
    vtA = synth.smooth_velocity(N_GRID, N_GRID, 3000 + rank)
    vtB = synth.smooth_velocity(N_GRID, N_GRID, 4000 + rank)
    return mT, (v1, v2), vtA, vtB


# ------------------------------------------------------------------------------ clocks
class ClockSampler:
    """SM clocks and throttle reasons sampled during the timed region: NVML polled every
    millisecond from a thread (a timed region of 20 matvecs lasts ~16 ms, shorter than one
    `nvidia-smi -lms` start-up), nvidia-smi as the fallback."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []
        self.nvml = None
        self.samples = []  # (sm_mhz, reason names)
        self.smax = None

    def start(self):
        try:
            import pynvml as N

            N.nvmlInit()
            h = N.nvmlDeviceGetHandleByIndex(self.device)
            self.smax = float(N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM))
            bits = [N.nvmlClocksEventReasonHwSlowdown, N.nvmlClocksEventReasonHwThermalSlowdown,
                    N.nvmlClocksEventReasonSwThermalSlowdown, N.nvmlClocksEventReasonSwPowerCap]
            self.nvml = (N, h, bits)
            self.stop_flag = threading.Event()

            def poll():
                while not self.stop_flag.is_set():
                    try:
                        mhz = float(N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM))
                        mask = N.nvmlDeviceGetCurrentClocksEventReasons(h)
                        self.samples.append((mhz, [nm for nm, b in zip(self.NAMES, bits) if mask & b]))
                    except Exception:  # noqa: BLE001
                        pass
                    time.sleep(0.001)

            self.t = threading.Thread(target=poll, daemon=True)
            self.t.start()
            return
        except Exception:  # noqa: BLE001 - no NVML: nvidia-smi
            self.nvml = None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.nvml is not None:
            self.stop_flag.set()
            self.t.join(timeout=1)
            sm = [m for m, _ in self.samples]
            reasons = sorted({r for _, rs in self.samples for r in rs})
            return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.smax, "reasons": reasons,
                    "samples": len(sm), "source": "nvml (1 ms polling during the timed region)"}
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for nm, val in zip(self.NAMES, parts[5:9]):
                if val.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm), "source": "nvidia-smi -lms 100"}


# ------------------------------------------------------------------------------ algorithmic bytes
# Per-launch algorithmic bytes (multiples of F = one fp64 field) of the library's kernels in
# one matvec.  Reads of the gathered coefficient field count once.
KERNEL_BYTES_F = {
    "evaluate/adjoint_bodyforce": 12,  # coef, X_D(2), dvDep, dv, G(2), b(2) in; lam, b(2) out
    "evaluate/incstate": 12,           # coef, X_D(2), vtD(2), GD(2), vt(2), G(2) in; m~ out
    "evaluate/store2": 7,              # coef(2), X_D(2) in; 2 out  (+ shared weights)
    "k_prefilter_rows": 2,
    "k_prefilter_cols": 2,
    "pointwise/adjoint_seed": 6,       # m~, G(2), b... : m~ + G(2) in, lam + b(2) out
    "evaluate/state_step": 4,
}


# Kernel classes of one matvec (vrg_hess_bench_kernel ids): name, launches per matvec at nt,
# algorithmic bytes per launch in F.  Two launch structures: the band
# path (default where the grid allows it: gather + epilogue + next row pass in one kernel,
# then the column pass) and the plain 3-kernel step.
KERNEL_CLASSES_BAND = {
    7: ("band/incstate (K6 + K1 rows)", NT - 1, 12),      # X(2) coef vtD(2) GD(2) vt(2) G(2) in; rows out
    8: ("band/adjoint_bodyforce (K5+K8 + K1 rows)", NT - 1, 12),  # X(2) coef dvD dv G(2) b(2) in; b(2) rows out
    4: ("prefilter column pass (K1 cols)", 2 * NT - 1, 2),
    1: ("evaluate/adjoint_bodyforce (K5+K8, last step)", 1, 12),
    2: ("prefilter rows+cols (K1, vt)", 2, 4),
    3: ("evaluate/store2 (K2, vt_D)", 1, 6),
    5: ("reference: field copy D2D (not in matvec)", 0, 2),
    6: ("reference: field axpy kernel (not in matvec)", 0, 3),
}
# ncu kernel-name fragments of the band-path classes (for the traffic lookup)
L2_STREAM_GBS = 10200.0  # streaming read of an 80 MB L2-resident set on B200 (tools/probe/l2probe.cu)
# ncu names of the band kernels at 1024^2 (strip blocks, evalband.cuh k_eval_strip)
NCU_NAMES = {7: "k_eval_strip<EpiIncState, 1, 128>", 8: "EpiAdjointBF, 1, 128>", 4: "k_pf_cols_reg"}
KERNEL_CLASSES_PLAIN = {
    0: ("evaluate/incstate (K6)", NT - 1, 12),
    1: ("evaluate/adjoint_bodyforce (K5+K8)", NT, 12),
    2: ("prefilter rows+cols (K1)", 2 * NT + 1, 4),
    3: ("evaluate/store2 (K2, vt_D)", 1, 6),
    4: ("prefilter cols only (K1 column pass)", 0, 2),  # included in id 2; breakdown only
    5: ("reference: field copy D2D (not in matvec)", 0, 2),
    6: ("reference: field axpy kernel (not in matvec)", 0, 3),
}


def matvec_algorithmic_bytes(nt: int = NT) -> int:
    """B_mv = (24 nt + 12) F."""
    return (24 * nt + 12) * F_BYTES


# ------------------------------------------------------------------------------ GPU arm
def run_vrg(args, rank, world, local_rank):
    import torch

    from paper_1604_02153_b200 import api

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    ctx = api.Context(local_rank)
    mT, v, vtA, vtB = make_problem(rank)
    T = lambda a: ctx.field(a)  # noqa: E731
    mT_d, v_d = T(mT), (T(v[0]), T(v[1]))
    # reference image: the template transported by the true velocity (GN does not depend on it)
    mR_d = api.Solver(ctx, v_d, NT).solve_state_final(mT_d)
    H = api.HessianOperator(ctx, v_d, mR_d, mT_d, NORM, BETA, api.COMPRESSIBLE, NT)
    vts = [ctx.empty(2, N_GRID, N_GRID) for _ in range(2)]
    vts[0][0].copy_(T(vtA[0])); vts[0][1].copy_(T(vtA[1]))
    vts[1][0].copy_(T(vtB[0])); vts[1][1].copy_(T(vtB[1]))
    out = ctx.empty(2, N_GRID, N_GRID)
    stream = ctx.stream

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize(dev)

    def timed(fn, k):
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for i in range(k):
            fn(i)
        e1.record(stream)
        barrier()
        ms = e0.elapsed_time(e1)
        if world > 1:
            t = torch.tensor([ms], device=dev)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    step = lambda i: H.apply((vts[i & 1][0], vts[i & 1][1]), out=out)  # noqa: E731
    # graph priming: the operator captures a CUDA graph on the second use of an (input, output)
    # pair, so each of the two alternating inputs is applied twice before the warm-up steps
    for i in range(4):
        step(i)
    for i in range(args.warmup):
        step(i)
    # headline: the K matvecs queued back to back through vrg_hess_apply_batch (each matvec's
    # guard checked on the host while the next one runs; same results as K apply calls)
    batch_in = [(vts[i & 1][0], vts[i & 1][1]) for i in range(args.steps)]
    batch_out = [(out[0], out[1])] * args.steps
    H.apply_batch(batch_in[:max(4, args.warmup)], batch_out[:max(4, args.warmup)])
    launches0 = ctypes_launches(ctx)
    clocks = ClockSampler(local_rank)
    clocks.start()
    ms = timed(lambda i: H.apply_batch(batch_in, batch_out) if i == 0 else None, 1)
    clk = clocks.stop()
    launches = ctypes_launches(ctx) - launches0
    value = world * args.steps / (ms / 1e3)
    # one vrg_hess_apply call per matvec (the reference API's call pattern: the guard is read
    # back before the call returns, so the device idles for one host round trip per matvec)
    ms_call = timed(step, args.steps)
    per_call = world * args.steps / (ms_call / 1e3)

    # e2e: drop-in host-buffer calls, pinned host memory, copies inside the timed region.
    # Headline: vrg_hess_apply_host_batch over the K steps (the copies of neighbouring matvecs
    # overlap the compute of the current one); also the one-call-per-step vrg_hess_apply_host.
    hin = [torch.empty(2, N_GRID, N_GRID, dtype=torch.float64, pin_memory=True) for _ in range(2)]
    hin[0].copy_(vts[0].cpu()); hin[1].copy_(vts[1].cpu())
    hout = [torch.empty(2, N_GRID, N_GRID, dtype=torch.float64, pin_memory=True) for _ in range(2)]
    batch_in = [(hin[i & 1][0], hin[i & 1][1]) for i in range(args.steps)]
    batch_out = [(hout[i & 1][0], hout[i & 1][1]) for i in range(args.steps)]
    nprime = max(4, args.warmup)  # graph capture of both device slots before the timed call
    H.apply_host_batch([(hin[i & 1][0], hin[i & 1][1]) for i in range(nprime)],
                       [(hout[i & 1][0], hout[i & 1][1]) for i in range(nprime)])
    barrier()
    t0 = time.perf_counter()
    ms_e2e = timed(lambda i: H.apply_host_batch(batch_in, batch_out) if i == 0 else None, 1)
    wall_e2e = time.perf_counter() - t0
    e2e_value = world * args.steps / (ms_e2e / 1e3)
    e2e_step = lambda i: H.apply_host(hin[i & 1][0], hin[i & 1][1], hout[0][0], hout[0][1])  # noqa: E731
    for i in range(max(1, args.warmup)):
        e2e_step(i)
    ms_serial = timed(e2e_step, args.steps)
    e2e_serial = world * args.steps / (ms_serial / 1e3)

    # profiled pass: per-launch CUDA events of every kernel of the same K steps
    ctx.lib.vrg_profile(ctx.h, 1)
    for i in range(args.steps):
        step(i)
    prof = profile_dump(ctx)
    ctx.lib.vrg_profile(ctx.h, 0)

    # back-to-back timing of each matvec kernel class (roofline denominator)
    kernels = {}
    band = ctypes.c_int()
    ctx.check(ctx.lib.vrg_hess_band_path(H.h, ctypes.byref(band)))
    classes = KERNEL_CLASSES_BAND if band.value else KERNEL_CLASSES_PLAIN
    for kid, (name, per_mv, bytes_f) in classes.items():
        out_ms = ctypes.c_double()
        ctx.check(ctx.lib.vrg_hess_bench_kernel(H.h, kid, 50, ctypes.byref(out_ms)))
        kernels[name] = {"avg_us": out_ms.value * 1e3, "launches_per_matvec": per_mv,
                         "bytes_per_launch": bytes_f * F_BYTES,
                         "gbps": bytes_f * F_BYTES / (out_ms.value / 1e3) / 1e9,
                         "ncu_kernel": NCU_NAMES.get(kid) if band.value else None}

    # SL transport unit: one SL state step m_j = I[m_{j-1}](X_D) at 1024^2 (config 4 unit ii)
    sl = sl_step_rate(ctx, H)
    # logical operation counts of one steady-state apply (the reference's counters::, which it
    # would execute) next to what the device executes (per-iterate invariants cached, the
    # reference recomputes them in every apply): separates caching from hardware speed-up
    ctx.reset_counters()
    H.apply((vts[0][0], vts[0][1]), out=(out[0], out[1]))
    ctx.sync()
    logical = ctx.counters()
    return dict(value=value, per_call=per_call, ms=ms, launches=launches, clocks=clk, e2e=e2e_value, ms_e2e=ms_e2e, e2e_serial=e2e_serial,
                wall_e2e=wall_e2e, prof=prof, sl=sl, kernels=kernels, ctx=ctx, api=api, logical=logical)


def ctypes_launches(ctx):
    import ctypes as C

    n = C.c_longlong()
    ctx.lib.vrg_launch_count(ctx.h, C.byref(n))
    return n.value


def profile_dump(ctx):
    import ctypes as C

    buf = C.create_string_buffer(1 << 16)
    ctx.check(ctx.lib.vrg_profile_dump(ctx.h, buf, len(buf)))
    prof = {}
    for line in buf.value.decode().splitlines():
        tag, cnt, tot = line.split("\t")
        prof[tag] = (int(cnt), float(tot))
    return prof


def sl_step_rate(ctx, H):
    """Config 4 unit (ii): one SL state step m_j = I[m_{j-1}](X_D) at 1024^2, back-to-back steps
    on the device (band form: gather + write m_j + the next prefilter's row pass, then the
    column pass; plain form: prefilter rows + cols + gather)."""
    band = ctypes.c_int()
    ctx.check(ctx.lib.vrg_hess_band_path(H.h, ctypes.byref(band)))
    res = {"unit": "one SL state step (prefilter rows+cols + 16-tap gather + write m_j), 1024^2",
           "algorithmic_bytes": 4 * F_BYTES}
    for kid, name in ((9, "band"), (10, "plain")):
        if kid == 9 and not band.value:
            continue
        out_ms = ctypes.c_double()
        ctx.check(ctx.lib.vrg_hess_bench_kernel(H.h, kid, 50, ctypes.byref(out_ms)))
        res[name] = {"us_per_step": out_ms.value * 1e3, "gbps": 4 * F_BYTES / (out_ms.value / 1e3) / 1e9}
    best = res.get("band", res["plain"])
    res["us_per_step"] = best["us_per_step"]
    res["gbps"] = best["gbps"]
    return res


# ------------------------------------------------------------------------------ CPU reference
def reference_sample(threads: int, matvecs_per_thread: int = 1):
    """One steady-state reference matvec (HessianOperator::apply, 1024^2, nt=16) per thread,
    threads in parallel (ctypes releases the GIL).  Returns (seconds, matvecs)."""
    from oracle import ref

    mT, v, vtA, _ = make_problem(0)
    ops = [None] * threads

    def build(i):
        ops[i] = ref.Hessian(v[0], v[1], mT, mT, NORM, BETA, 0, NT)
        ops[i].apply(vtA[0], vtA[1])  # first apply builds the lazy caches

    ths = [threading.Thread(target=build, args=(i,)) for i in range(threads)]
    [t.start() for t in ths]
    [t.join() for t in ths]

    def work(i):
        for _ in range(matvecs_per_thread):
            ops[i].apply(vtA[0], vtA[1])

    t0 = time.perf_counter()
    ths = [threading.Thread(target=work, args=(i,)) for i in range(threads)]
    [t.start() for t in ths]
    [t.join() for t in ths]
    return time.perf_counter() - t0, threads * matvecs_per_thread, ops


def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def run_reference(args, rank):
    if rank != 0:
        return None
    from oracle import ref

    if not ref.available():
        return {"impl": "reference", "unavailable": "oracle/_ref/libveloreg_ref.so not built (make -C oracle)"}
    threads = min(cpu_threads(), 64)
    from oracle import ref as R
    mT, v, vtA, _ = make_problem(0)
    ops = []
    lock = threading.Lock()

    def build():
        h = R.Hessian(v[0], v[1], mT, mT, NORM, BETA, 0, NT)
        h.apply(vtA[0], vtA[1])
        with lock:
            ops.append(h)

    ths = [threading.Thread(target=build) for _ in range(threads)]
    [t.start() for t in ths]
    [t.join() for t in ths]

    def one_step():
        ws = [threading.Thread(target=lambda h=h: h.apply(vtA[0], vtA[1])) for h in ops]
        [w.start() for w in ws]
        [w.join() for w in ws]

    for _ in range(args.warmup):
        one_step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        one_step()
    dt = time.perf_counter() - t0
    value = threads * args.steps / dt
    sample = (f"each step = {threads} concurrent steady-state HessianOperator::apply calls (one per host thread) "
              f"of the unmodified reference, 1024^2 nt=16 H2, FFT backend = repo FFTW3-API shim")
    fft = fft_backend_probe()
    return {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": dict(CONFIG, parallelism=f"pairs{args.gpus}"),  # the GPU arm's config at N=gpus
            "impl": "reference",
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference", "sample": sample,
                             "fft_backend": fft},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def fft_backend_probe():
    """The reference's FFT on this host: libfftw3 is looked up with `ldconfig -p` (use it
    if present); the reference as built here uses the repo's FFTW3-API shim (oracle/fftw_shim,
    FFTW3 is not in the image), timed per 1024^2 transform (spectral::gradient = 1 r2c + 2 c2r)."""
    from oracle import ref

    try:
        out = subprocess.run(["ldconfig", "-p"], capture_output=True, text=True, timeout=30).stdout
        fftw = sorted({ln.split()[0] for ln in out.splitlines() if "fftw3" in ln})
    except (OSError, subprocess.SubprocessError):
        fftw = None
    u = np.random.default_rng(0).standard_normal((N_GRID, N_GRID))
    ref.gradient(u)
    t0 = time.perf_counter()
    for _ in range(3):
        ref.gradient(u)
    per_fft = (time.perf_counter() - t0) / 9
    t0 = time.perf_counter()
    for _ in range(3):
        np.fft.irfft2(np.fft.rfft2(u), s=u.shape)
    per_np = (time.perf_counter() - t0) / 6
    return {"libfftw3_on_host": fftw if fftw else "absent (ldconfig -p)",
            "backend_used": "repo FFTW3-API shim (oracle/fftw_shim: radix-2 complex FFT, real transforms by "
                            "half-length packing)",
            "ms_per_fft_1024": per_fft * 1e3,
            "numpy_pocketfft_ms_per_fft_1024": per_np * 1e3,
            "logical_ffts_per_reference_matvec": 6 * NT + 10}


def cpu_baseline_leg():
    from oracle import ref

    if not ref.available():
        return None
    threads = min(cpu_threads(), 32)
    dt, nmv, _ = reference_sample(threads)
    return {"value": nmv / dt, "unit": UNIT, "cores": threads, "kind": "reference",
            "sample": f"{nmv} steady-state reference HessianOperator::apply calls at 1024^2 nt=16, one per host "
                      f"thread in parallel ({dt:.1f} s); FFT via the repo's FFTW3-API shim",
            "fft_backend": fft_backend_probe()}


# ------------------------------------------------------------------------------ time to solution
# Full inexact Gauss-Newton-Krylov registrations (newtonSolve) of the BASELINE configs that a
# bench run can afford: configs 1 and 2 (against the reference on one host core) and one
# config-3 pair (GPU only; the reference needs minutes per matvec-heavy solve at 512^2).
TTS_RUNS = {
    "config1_64_nt4_H2_1e-2_2L-pcg": dict(n=64, nt=4, norm=2, beta=1e-2, cheb=False, cpu=True),
    "config2_256_nt8_H1_1e-3_2L-cheb10": dict(n=256, nt=8, norm=1, beta=1e-3, cheb=True, cpu=True),
    "config2i_256_nt8_H1_1e-3_2L-cheb10_incompressible": dict(n=256, nt=8, norm=1, beta=1e-3, cheb=True, cpu=True,
                                                              deformation=1),
    "config3_512_nt16_H2_1e-3_2L-cheb10_pair0": dict(n=512, nt=16, norm=2, beta=1e-3, cheb=True, cpu=False),
    # one GPU, one run (no warm-up solve), reference's default cap of 50 outer iterations
    "config5a_4096_nt32_H2_1e-4_2L-cheb10_single_gpu": dict(n=4096, nt=32, norm=2, beta=1e-4, cheb=True, cpu=False,
                                                            runs=1),
}


def tts_problem(cfg):
    from paper_1604_02153_b200 import synth

    n, nt = cfg["n"], cfg["nt"]
    if n <= 256:
        mT, (v1, v2) = synth.config12_fields(n)
    else:
        mT = synth.smoothed_noise(n, n, 1000)
        v1, v2 = synth.smooth_velocity(n, n, 2000)
    return mT, v1, v2


def time_to_solution(ctx, api, with_cpu):
    """Wall time of newtonSolve (tolRelGrad 1e-2) through the C ABI with host images, and the
    reference's on one host core for configs 1-2.  The reference image m_R is the template
    transported by the known velocity with the device SL solver (bit-compatible with the
    reference's, see tests/test_gpu_parity.py)."""
    import torch

    out = {}
    for name, cfg in TTS_RUNS.items():
        mT, v1, v2 = tts_problem(cfg)
        mR = api.Solver(ctx, (ctx.field(v1), ctx.field(v2)), cfg["nt"]).solve_state_final(ctx.field(mT)).cpu().numpy()
        kw = dict(nt=cfg["nt"], kind=api.PC_TWO_LEVEL, coarse_solver=api.COARSE_CHEB if cfg["cheb"] else api.COARSE_PCG,
                  cheb_iters=10, tol_rel=1e-2)
        deform = cfg.get("deformation", api.COMPRESSIBLE)
        nruns = cfg.get("runs", 2)
        if nruns > 1:
            api.newton_solve(ctx, mR, mT, cfg["norm"], cfg["beta"], deform, **kw)  # warm (plans, modules)
        runs = []
        for _ in range(nruns):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            _, _, recs, summ = api.newton_solve(ctx, mR, mT, cfg["norm"], cfg["beta"], deform, **kw)
            torch.cuda.synchronize()
            runs.append(time.perf_counter() - t0)
        dt = min(runs)
        entry = {"gpu_s": dt, "gpu_s_runs": runs, "newton_iterations": summ["iterations"],
                 "krylov_iterations": int(sum(r["innerIterations"] for r in recs)),
                 "final_grad_norm_rel": summ["finalGradNormRel"], "status": summ["status"]}
        if with_cpu and cfg["cpu"]:
            from oracle import ref

            if ref.available():
                t0 = time.perf_counter()
                _, _, rrep, rs = ref.newton_solve(mR, mT, cfg["norm"], cfg["beta"], deform, nt=cfg["nt"], two_level=True,
                                                  cheb=cfg["cheb"], cheb_iters=10, tol_rel=1e-2)
                entry["cpu_reference_s"] = time.perf_counter() - t0
                entry["cpu_cores"] = 1
                entry["same_newton_and_krylov_iterations"] = bool(
                    int(rs[1]) == summ["iterations"]
                    and all(int(q[5]) == r["innerIterations"] for q, r in zip(rrep, recs)))
                entry["speedup_vs_cpu"] = entry["cpu_reference_s"] / dt
        out[name] = entry
    return out


# Batched pairs (BASELINE configs 5b and 3) on this GPU: lanes of lockstep batches
# (batch.py --lanes L --batch B; csrc/batch.cu), the second pass timed.
BATCH_RUNS = {
    # lanes x batch from the sweep of tools/gpu_s4g.sh (profiles/r2s3_batch_sweep.txt)
    "config5b_64pairs_256_nt16_H2_1e-3_2L-cheb10": dict(n=256, pairs=64, lanes=4, batch=16),
    "config3_8pairs_512_nt16_H2_1e-3_2L-cheb10": dict(n=512, pairs=8, lanes=4, batch=2),
}


def batched_pairs(ctx, api):
    import torch

    from paper_1604_02153_b200 import batch

    out = {}
    for name, cfg in BATCH_RUNS.items():
        n, nt = cfg["n"], 16
        images = {p: batch.make_images(ctx, n, p, nt) for p in range(cfg["pairs"])}
        ps = list(range(cfg["pairs"]))
        chunks = [ps[i:i + cfg["batch"]] for i in range(0, len(ps), cfg["batch"])]
        ctxs = [ctx] + [api.Context(0, stream=torch.cuda.Stream(0)) for _ in range(1, cfg["lanes"])]
        walls = []
        for _ in range(3):  # plans, graphs and the block cache of every lane warm after two passes
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            res = [r for c in batch.run_lanes(list(range(len(chunks))),
                                              lambda lane: batch.batched_runner(ctxs[lane], n, nt, 1e-3, 2, 10, 1e-2,
                                                                                images, chunks), cfg["lanes"])
                   for r in c["pairs"]]
            torch.cuda.synchronize()
            walls.append(time.perf_counter() - t0)
        out[name] = {"pairs_per_s": cfg["pairs"] / walls[-1], "wall_s": walls[-1], "lanes": cfg["lanes"],
                     "batch": cfg["batch"], "newton_iterations": sum(r["newton_iterations"] for r in res),
                     "krylov_iterations": sum(r["inner_iterations"] for r in res),
                     "status_counts": {str(s): sum(r["status"] == s for r in res) for s in sorted({r["status"] for r in res})},
                     "errors": sum(r["error"] != 0 for r in res),
                     "note": "pairs solved in lockstep batches (api.newton_solve_batch), batches on concurrent "
                             "lanes; images made before the timed region; third pass timed; status 0 converged, "
                             "1 the reference's 50-iteration cap"}
        del ctxs[1:]
    return out


# ------------------------------------------------------------------------------ main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="vrg", choices=["vrg", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-tts", action="store_true", help="skip the time-to-solution registrations")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 0)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        res = run_reference(args, rank)
        if res is not None:
            print(json.dumps(res), flush=True)
        return

    import torch

    if world > 1:
        torch.cuda.set_device(local_rank)
        torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    r = run_vrg(args, rank, world, local_rank)
    if rank == 0:
        prof = r["prof"]
        kernels = r["kernels"]
        # dominant kernel class: largest (launches per matvec x back-to-back launch time)
        tag, kd = max(kernels.items(), key=lambda kv: kv[1]["avg_us"] * kv[1]["launches_per_matvec"])
        avg_s = kd["avg_us"] / 1e6
        bytes_launch = kd["bytes_per_launch"]
        peaks = {}
        try:
            with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
                peaks = json.load(f)
        except OSError:
            pass
        peak = float(peaks.get("hbm_gbs", 6650.0))
        # DRAM traffic of the dominant kernel per launch, from the committed ncu --set full
        # capture (profiles/, cold-cache replay: an upper bound of the warm per-launch traffic)
        traffic = None
        traffic_file = next((f for f in ("r2s3_ncu_traffic.json", "r2_ncu_traffic.json", "r1_ncu_traffic.json")
                             if os.path.exists(os.path.join(ROOT, "profiles", f))), "r1_ncu_traffic.json")
        try:
            with open(os.path.join(ROOT, "profiles", traffic_file)) as f:
                tmap = json.load(f)
            pat = kd.get("ncu_kernel")
            hits = [v for k, v in tmap.items() if pat and pat in k]
            traffic = hits[0] if hits else None
        except (OSError, ValueError):
            pass
        achieved = bytes_launch / avg_s / 1e9 if bytes_launch else None
        prof_total = sum(t for _, t in prof.values())
        mv_bytes = matvec_algorithmic_bytes()
        line = {
            "metric": METRIC, "value": r["value"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": r["ms"] / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": dict(CONFIG, parallelism=f"pairs{world}"),
            "per_call": {"value": r["per_call"], "unit": UNIT,
                         "call": "vrg_hess_apply, one call per matvec (the guard is read back before each call "
                                 "returns: one host round trip per matvec)"},
            "e2e": {"value": r["e2e"], "unit": UNIT, "h2d_bytes_per_step": 2 * F_BYTES, "d2h_bytes_per_step": 2 * F_BYTES,
                    "call": "vrg_hess_apply_host_batch over the K steps (pinned host buffers; H2D/D2H of "
                            "neighbouring matvecs overlap the current matvec)",
                    "serial": {"value": r["e2e_serial"], "call": "vrg_hess_apply_host, one call per step"}},
            "gpu_launches": r["launches"],
            "clocks": r["clocks"],
            "roofline": {"bound": "hbm", "kernel": tag, "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                         "traffic_source": f"profiles/{traffic_file} (ncu --set full, dram__bytes_read+write)",
                         "bytes_per_launch": bytes_launch, "avg_launch_us": avg_s * 1e6,
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured)" if peaks else "fallback 6650",
                         "note": "algorithmic bytes count operands that stay L2-resident across steps (departure "
                                 "cells, vt, vt_D, div v), so frac can exceed 1: the kernel is bound by the L2->SM "
                                 "path; l2_frac = achieved / the 10.2 TB/s an 80 MB L2-resident stream reaches on "
                                 "B200 (tools/probe/l2probe.cu, DESIGN.md section 4)",
                         "l2_frac": (achieved / L2_STREAM_GBS) if achieved else None},
            "matvec_roofline": {"algorithmic_bytes": mv_bytes, "model": "(24 nt + 12) F, SURVEY 8(d)",
                                "achieved_gbps": mv_bytes * r["value"] / world / 1e9,
                                "frac": mv_bytes * r["value"] / world / 1e9 / peak},
            "sl_interp": r["sl"],
            "op_counts_per_matvec": {
                "logical": {"ffts": r["logical"][0], "interps": r["logical"][1],
                            "note": "the reference's counters:: per apply (what the reference executes)"},
                "executed": {"ffts": 2 * (prof.get("cufft_d2z", (0, 0))[0] + prof.get("cufft_z2d", (0, 0))[0]) // args.steps,
                             "interps": (sum(prof.get(k, (0, 0))[0] for k in ("evaluate/adjoint_bodyforce", "evaluate/incstate",
                                                                               "evaluate/incstate_seed"))
                                         + 2 * prof.get("evaluate/store2", (0, 0))[0]) // args.steps,
                             "note": "field transforms / scalar-field gathers the device runs per apply (cuFFT calls "
                                     "are batched over the 2 components); grad m_j, (grad m_{j-1})_D, X_D, div v, "
                                     "(div v)_D are per-iterate invariants cached at HessianOperator construction"}},
            "kernels": kernels,
            "kernel_model_ms_per_matvec": sum(k["avg_us"] * k["launches_per_matvec"] for k in kernels.values()) / 1e3,
            "event_profile": {"note": "per-launch event pairs (each pair adds its own overhead); shares only",
                              "share": {k: round(t / prof_total, 4)
                                        for k, (c, t) in sorted(prof.items(), key=lambda kv: -kv[1][1])},
                              "launches_per_step": {k: c // args.steps for k, (c, t) in prof.items()}},
        }
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline_leg()
        if not args.no_tts:
            line["time_to_solution"] = time_to_solution(r["ctx"], r["api"], world == 1 and not args.no_cpu_baseline)
            if world == 1:
                line["batched_pairs"] = batched_pairs(r["ctx"], r["api"])
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
