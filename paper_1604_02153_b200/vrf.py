"""Field files and solver reports of the reference (veloreg::io, src/io.cpp), host side.

VRF1: "VRF1", then n1, n2, components as little-endian uint32, then the components' samples
as little-endian binary64, row-major (io.cpp:16-94, 112-154).  Binary PGM (P5) images are
read as one period of a periodic field in [0, 1] and, if their size differs from the target
grid, resampled spectrally on the device (io.cpp:156-216).  `solver_report_csv` writes the
per-iteration records with the reference's columns and number format (io.cpp:227-239), and
`summary_json` the run summary of the reference's CLI (proj/tools/main.cpp:254-272).
"""
from __future__ import annotations

import struct

import numpy as np

MAGIC = b"VRF1"


def write_field(path, u):
    """u: (n1, n2) scalar field or a pair / (2, n1, n2) vector field."""
    comps = [np.asarray(c, dtype="<f8") for c in (u if isinstance(u, (tuple, list)) else
                                                   (list(u) if np.ndim(u) == 3 else [u]))]
    n1, n2 = comps[0].shape
    with open(path, "wb") as f:
        f.write(MAGIC + struct.pack("<III", n1, n2, len(comps)))
        for c in comps:
            f.write(np.ascontiguousarray(c, dtype="<f8").tobytes())


def _header(f, path):
    head = f.read(16)
    if len(head) < 4 or head[:4] != MAGIC:
        raise RuntimeError(f"{path}: not a VRF1 field file")
    if len(head) < 16:
        raise RuntimeError(f"{path}: corrupt field header")
    n1, n2, nc = struct.unpack("<III", head[4:16])
    if nc < 1 or nc > 16:
        raise RuntimeError(f"{path}: corrupt field header")
    return n1, n2, nc


def field_components(path):
    with open(path, "rb") as f:
        return _header(f, path)[2]


def _read(path, want):
    with open(path, "rb") as f:
        n1, n2, nc = _header(f, path)
        if nc != want:
            raise RuntimeError(f"{path}: expected a {'one' if want == 1 else 'two'}-component field")
        data = np.frombuffer(f.read(), dtype="<f8")
    if data.size < n1 * n2 * nc:
        raise RuntimeError(f"{path}: truncated field file")
    return data[:n1 * n2 * nc].astype(np.float64).reshape(nc, n1, n2)


def read_scalar_field(path):
    return _read(path, 1)[0]


def read_vector_field(path):
    v = _read(path, 2)
    return v[0], v[1]


def write_graymap(path, u):
    """16-bit binary PGM of u clamped to [0, 1] (io.cpp:156-166)."""
    u = np.asarray(u, dtype=np.float64)
    n1, n2 = u.shape
    s = np.floor(np.clip(u, 0.0, 1.0) * 65535.0 + 0.5).astype(">u2")
    with open(path, "wb") as f:
        f.write(f"P5\n{n2} {n1}\n65535\n".encode())
        f.write(s.tobytes())


def _pgm_token(buf, pos):
    n = len(buf)
    while pos < n and (chr(buf[pos]).isspace() or buf[pos] == ord("#")):
        if buf[pos] == ord("#"):
            while pos < n and buf[pos] != ord("\n"):
                pos += 1
        pos += 1
    start = pos
    while pos < n and chr(buf[pos]).isdigit():
        pos += 1
    if start == pos:
        raise RuntimeError("graymap: malformed header")
    return int(buf[start:pos]), pos


def read_graymap(path, shape, ctx=None):
    """P5 graymap as a field on `shape` (n1, n2); resampled spectrally (api.resample on ctx)
    when the image size differs (io.cpp:168-216)."""
    with open(path, "rb") as f:
        buf = f.read()
    if buf[:2] != b"P5":
        raise RuntimeError(f"{path}: not a binary graymap (P5)")
    width, pos = _pgm_token(buf, 2)
    height, pos = _pgm_token(buf, pos)
    maxval, pos = _pgm_token(buf, pos)
    if width < 1 or height < 1 or maxval < 1 or maxval > 65535:
        raise RuntimeError(f"{path}: unsupported graymap header")
    pos += 1  # the single whitespace after maxval
    count = width * height
    if maxval < 256:
        raw = np.frombuffer(buf[pos:pos + count], dtype=np.uint8)
    else:
        raw = np.frombuffer(buf[pos:pos + 2 * count], dtype=">u2")
    if raw.size < count:
        raise RuntimeError(f"{path}: truncated graymap")
    img = (raw.astype(np.float64) / float(maxval)).reshape(height, width)
    if (height, width) == tuple(shape):
        return img
    if height % 2 or width % 2 or height < 4 or width < 4:
        raise RuntimeError(f"{path}: graymap size must be even and >= 4 to resample")
    return _resample(ctx, img, shape)


def _resample(ctx, img, shape):
    from . import api

    if ctx is None:
        ctx = api.Context(0)
    return api.resample(ctx, ctx.field(img), shape).cpu().numpy()


def read_image(path, shape, ctx=None):
    """VRF1 scalar field or P5 graymap on `shape` (io.cpp:218-225)."""
    with open(path, "rb") as f:
        magic = f.read(4)
    if magic == MAGIC:
        u = read_scalar_field(path)
        return u if u.shape == tuple(shape) else _resample(ctx, u, shape)
    return read_graymap(path, shape, ctx)


COLUMNS = ("iter,grad_inf,grad_rel,objective,mismatch,inner_iters,ls_steps,step_length,"
           "wall_time_sec,ffts,interps")


def solver_report_csv(records):
    """The reference's convergence table (io.cpp:227-239); records as api.newton_solve returns."""
    lines = [COLUMNS]
    for r in records:
        lines.append(",".join([
            str(int(r["iter"])), f"{r['gradNormInf']:.12e}", f"{r['gradNormRel']:.12e}", f"{r['objective']:.12e}",
            f"{r['mismatch']:.12e}", str(int(r["innerIterations"])), str(int(r["lineSearchSteps"])),
            f"{r['stepLength']:.12e}", f"{r['wallTimeSec']:.12e}", str(int(r["ffts"])), str(int(r["interps"]))]))
    return "\n".join(lines) + "\n"


STATUS_NAMES = {0: "converged", 1: "iteration-limit", 2: "line-search-failure"}


def summary_json(config, summary, ffts, interps):
    """summary.json of a registration run, as the reference's CLI writes it (proj/tools/main.cpp:
    254-272, nlohmann::json dump(2): keys sorted, two-space indent): `config` is the run's
    configuration echo (main.cpp:97-117), `summary` api.newton_solve's summary dict, ffts /
    interps the process operation counters after the run."""
    import json

    jmin, jmax = float(summary["jacMin"]), float(summary["jacMax"])
    doc = {"config": config, "status": STATUS_NAMES[int(summary["status"])],
           "outer_iterations": int(summary["iterations"]), "grad_rel": float(summary["finalGradNormRel"]),
           "residual_rel": float(summary["finalResidualRel"]), "jacobian_min": jmin, "jacobian_max": jmax,
           "max_abs_jacobian_deviation": max(abs(jmin - 1.0), abs(jmax - 1.0)), "ffts": int(ffts),
           "interps": int(interps), "time_sec": float(summary["totalTimeSec"])}
    return json.dumps(doc, indent=2, sort_keys=True, ensure_ascii=False) + "\n"
