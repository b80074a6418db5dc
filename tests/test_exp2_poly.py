"""CPU emulation (float32, numpy) of the kernel's FMA-pipe exp2 (ex2_poly2 in
paper_2604_12798_b200/csrc/vfa_kernel.cuh): coefficients are parsed from the source so the
test tracks the kernel. Pins accuracy (< 4e-6 relative), exact zeros for x <= -127 and
masked -inf (so l == 0 underflow semantics match MUFU.EX2.FTZ), +inf for x >= 128."""

import os
import re

import numpy as np

SRC = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                   "paper_2604_12798_b200", "csrc", "vfa_kernel.cuh")


def _coeffs():
    body = open(SRC).read()
    body = body[body.index("float2 ex2_poly2"):]
    body = body[: body.index("return y;")]
    vals = [float(x) for x in re.findall(r"make_float2\(([0-9.e-]+)f, \1f\)", body)]
    # order in source: c4, c3 (first ffma2), c2, c1, c0 -> drop the magic constants
    return [v for v in vals if abs(v) < 2.0]


def ex2_poly(x, c):
    x = np.float32(min(max(np.float32(x), np.float32(-127.0)), np.float32(128.0)))
    magic = np.float32(12582912.0)
    r = np.float32(x + magic)
    jf = np.float32(r - magic)
    f = np.float32(x - jf)
    p = np.float32(c[0])
    for k in c[1:]:
        p = np.float32(p * f + np.float32(k))
    bits = (int(np.array(p, np.float32).view(np.uint32)) + (int(np.array(r, np.float32).view(np.uint32)) << 23))
    return float(np.array(bits & 0xFFFFFFFF, np.uint32).view(np.float32))


def test_coefficients_parsed():
    c = _coeffs()
    assert len(c) == 5 and c[-1] == 1.0  # p(0) == 1 exactly: 2^128 -> inf, 2^-127 -> 0


def test_accuracy_and_special_values():
    c = _coeffs()
    xs = np.random.default_rng(0).uniform(-60, 20, 20000).astype(np.float32).astype(np.float64)
    err = max(abs(ex2_poly(x, c) / 2.0 ** x - 1) for x in xs)
    assert err < 4e-6
    assert ex2_poly(-np.inf, c) == 0.0
    assert ex2_poly(-127.0, c) == 0.0
    assert ex2_poly(-2164.0, c) == 0.0
    assert ex2_poly(0.0, c) == 1.0
    assert ex2_poly(128.0, c) == np.inf and ex2_poly(1e4, c) == np.inf
    assert np.isfinite(ex2_poly(127.6, c))
    assert 0 < ex2_poly(-126.0, c) < 1.2e-38
