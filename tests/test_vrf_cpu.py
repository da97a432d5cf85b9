"""CPU: VRF1 field files, P5 graymaps and the convergence CSV (veloreg::io, io.cpp) against the
compiled reference's own writers and readers (byte-identical files, identical text)."""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np
import pytest

from paper_1604_02153_b200 import vrf


@pytest.fixture(scope="module")
def R():
    from oracle import ref

    if not ref.available():
        pytest.skip("oracle/_ref not built")
    return ref.lib()


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def test_vrf1_bytes_and_roundtrip(R, tmp_path):
    rng = np.random.default_rng(3)
    u = rng.standard_normal((12, 20))
    v = rng.standard_normal((2, 12, 20))
    for data, comps in ((u, 1), (v, 2)):
        ours, theirs = tmp_path / f"o{comps}.vrf", tmp_path / f"r{comps}.vrf"
        vrf.write_field(str(ours), data if comps == 1 else (data[0], data[1]))
        flat = np.ascontiguousarray(data, dtype=np.float64)
        assert R.ref_write_field(str(theirs).encode(), 12, 20, comps, _dp(flat)) == 0
        assert ours.read_bytes() == theirs.read_bytes()
        assert vrf.field_components(str(theirs)) == comps
        got = vrf.read_scalar_field(str(theirs)) if comps == 1 else np.stack(vrf.read_vector_field(str(theirs)))
        assert np.array_equal(got, data)
        n1, n2, nc = C.c_int(), C.c_int(), C.c_int()
        back = np.empty(data.size)
        assert R.ref_read_field(str(ours).encode(), C.byref(n1), C.byref(n2), C.byref(nc), _dp(back),
                                C.c_longlong(back.size)) == 0
        assert (n1.value, n2.value, nc.value) == (12, 20, comps) and np.array_equal(back.reshape(data.shape), data)
    with pytest.raises(RuntimeError, match="expected a two-component"):
        vrf.read_vector_field(str(tmp_path / "o1.vrf"))
    (tmp_path / "bad.vrf").write_bytes(b"XXXX" + bytes(12))
    with pytest.raises(RuntimeError, match="not a VRF1"):
        vrf.read_scalar_field(str(tmp_path / "bad.vrf"))


TOOL = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref", "ref_io_tool")


def _tool(*args):
    """The reference's stream-formatting I/O runs in its own process (oracle/ref_io_tool.cpp)."""
    if not os.path.exists(TOOL):
        pytest.skip("oracle/_ref/ref_io_tool not built")
    return subprocess.run([TOOL, *map(str, args)], capture_output=True, text=True, check=True).stdout


def test_graymap_bytes_and_read(tmp_path):
    rng = np.random.default_rng(4)
    u = rng.uniform(-0.2, 1.2, (10, 14))
    ours, theirs, src = tmp_path / "o.pgm", tmp_path / "r.pgm", tmp_path / "u.vrf"
    vrf.write_graymap(str(ours), u)
    vrf.write_field(str(src), u)
    _tool("write-graymap", src, theirs)
    assert ours.read_bytes() == theirs.read_bytes()
    _tool("read-graymap", ours, 10, 14, tmp_path / "back.vrf")
    assert np.array_equal(vrf.read_graymap(str(theirs), (10, 14)), vrf.read_scalar_field(str(tmp_path / "back.vrf")))
    # 8-bit graymap with a comment in the header
    (tmp_path / "b.pgm").write_bytes(b"P5\n# c\n4 4\n255\n" + bytes(range(16)))
    got = vrf.read_graymap(str(tmp_path / "b.pgm"), (4, 4))
    _tool("read-graymap", tmp_path / "b.pgm", 4, 4, tmp_path / "b.vrf")
    assert np.array_equal(got, vrf.read_scalar_field(str(tmp_path / "b.vrf")))
    assert np.array_equal(got, np.arange(16).reshape(4, 4) / 255.0)


def test_solver_report_csv(tmp_path):
    rows = np.array([[0, 1.5e-2, 1.0, 3.25, 3.0, 2, 1, 1.0, 0.0123, 40, 21],
                     [1, 2.5e-4, 1.6667e-2, 1.125, 1.0, 5, 2, 0.5, 1.25e-3, 140, 77]], dtype=np.float64)
    recs = [dict(iter=r[0], gradNormInf=r[1], gradNormRel=r[2], objective=r[3], mismatch=r[4], innerIterations=r[5],
                 lineSearchSteps=r[6], stepLength=r[7], wallTimeSec=r[8], ffts=r[9], interps=r[10]) for r in rows]
    (tmp_path / "rows.f64").write_bytes(np.ascontiguousarray(rows).tobytes())
    assert vrf.solver_report_csv(recs) == _tool("csv", tmp_path / "rows.f64", 2)


@pytest.mark.gpu
def test_graymap_resampled_on_device(tmp_path):
    """A graymap of another size is resampled spectrally (io.cpp:208-215) with the device
    resample; against the reference's own reader."""
    from paper_1604_02153_b200 import api

    ctx = api.Context(0)
    rng = np.random.default_rng(5)
    u = rng.uniform(0.0, 1.0, (24, 32))
    vrf.write_graymap(str(tmp_path / "g.pgm"), u)
    got = vrf.read_graymap(str(tmp_path / "g.pgm"), (48, 40), ctx)
    _tool("read-graymap", tmp_path / "g.pgm", 48, 40, tmp_path / "g.vrf")
    ref = vrf.read_scalar_field(str(tmp_path / "g.vrf"))
    assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max()


def test_summary_json_matches_reference_cli_format(tmp_path):
    """summary.json (proj/tools/main.cpp:254-272) byte-identical to the nlohmann::json document the
    reference's CLI builds from the same values (ref_io_tool summary, oracle/ref_io_tool.cpp)."""
    if not os.path.exists(TOOL):
        pytest.skip("oracle/_ref/ref_io_tool not built")
    config = {"mr": "data/ref.vrf", "mt": "data/tmpl.vrf", "grid": 256, "norm": "h1", "betav": 0.001,
              "model": "compressible", "betaw": 0.1, "scheme": "sl", "cfl": 1.0, "pc": "2l-cheb", "cheb_iters": 10,
              "tol_rel": 0.01, "tol_abs": 1e-05, "maxit": 50, "sigma": 0.0, "out": "out dir", "seed": 1234,
              "protocol": "none", "problem": "file"}
    for status, summ in [(0, dict(iterations=5, finalGradNormRel=0.0028532699925499488, finalResidualRel=0.0321754197,
                                  jacMin=0.788873058129, jacMax=1.35304261003, totalTimeSec=0.0391)),
                         (2, dict(iterations=50, finalGradNormRel=0.35, finalResidualRel=0.96, jacMin=0.5,
                                  jacMax=2.25, totalTimeSec=10.4))]:
        summ["status"] = status
        got = vrf.summary_json(config, summ, 4445, 1915)
        spec = tmp_path / "in.txt"
        lines = []
        for k, v in config.items():
            t = "s" if isinstance(v, str) else ("i" if isinstance(v, int) else "d")
            lines.append(f"config {k} {t} {v!r}" if t == "d" else f"config {k} {t} {v}")
        lines += [f"status {status}", f"outer_iterations {summ['iterations']}",
                  f"grad_rel {summ['finalGradNormRel']!r}", f"residual_rel {summ['finalResidualRel']!r}",
                  f"jacobian_min {summ['jacMin']!r}", f"jacobian_max {summ['jacMax']!r}", "ffts 4445", "interps 1915",
                  f"time_sec {summ['totalTimeSec']!r}"]
        spec.write_text("\n".join(lines) + "\n")
        want = subprocess.run([TOOL, "summary", str(spec)], capture_output=True, text=True, check=True).stdout
        assert got == want
