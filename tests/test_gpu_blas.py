"""GPU: the field BLAS-1 reductions (field.cpp:19-119: dot = h1 h2 sum(a b) per component, then
added; normLinf = max |x| with NaN ignored, std::max semantics).  The reductions finish in one
launch (the last block reduces the partials, runtime.cu lastBlockOf / finalOf); checked against
numpy at one-block, full-grid and grid-stride sizes, repeated (the tickets reset themselves), for
scalar and vector fields, and per pair of a batch (bit-identical to reducing the pair alone)."""
from __future__ import annotations

import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def api():
    from paper_1604_02153_b200 import api as A

    return A


@pytest.mark.parametrize("n1,n2", [(4, 4), (16, 32), (64, 64), (1024, 1024), (2048, 2048)])
def test_dot_and_norm_linf(ctx, api, n1, n2):
    rng = np.random.default_rng(n1 * 7 + n2)
    a = rng.standard_normal((2, n1, n2))
    b = rng.standard_normal((2, n1, n2))
    h = (2 * math.pi / n1) * (2 * math.pi / n2)
    A, B = ctx.field(a), ctx.field(b)
    want = h * float((a[0] * b[0]).sum()) + h * float((a[1] * b[1]).sum())
    got = [api.dot(ctx, (A[0], A[1]), (B[0], B[1])) for _ in range(3)]
    assert got[0] == got[1] == got[2]  # deterministic, tickets reset between calls
    assert abs(got[0] - want) <= 1e-12 * (h * float(np.abs(a * b).sum()))
    s = api.dot(ctx, A[0], B[0])
    assert abs(s - h * float((a[0] * b[0]).sum())) <= 1e-12 * (h * float(np.abs(a[0] * b[0]).sum()))
    assert api.norm_linf(ctx, (A[0], A[1])) == float(np.abs(a).max())
    assert api.norm_linf(ctx, A[1]) == float(np.abs(a[1]).max())


def test_norm_linf_ignores_nan(ctx, api):
    a = np.zeros((64, 64))
    a[3, 5] = np.nan
    a[10, 11] = -7.5
    assert api.norm_linf(ctx, ctx.field(a)) == 7.5
