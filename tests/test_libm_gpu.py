"""GPU: the device exp / log / pow (csrc/strait_libm.cuh) return exactly the
bits of the host libm that the reference runs on (CPython math.exp, math.log,
float.__pow__ -> glibc), over the argument ranges of the estimator and the
ground truth plus the special cases."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def device_math(fn, x, y=None):
    import torch

    from paper_2604_28175_b200 import _device as D

    dx = D.dev(np.ascontiguousarray(x, dtype=np.float64))
    dy = D.dev(np.ascontiguousarray(y, dtype=np.float64)) if y is not None else None
    out = D.empty(len(x))
    D.check(D.lib().strait_math(fn, D.ptr(dx), D.ptr(dy), len(x), D.ptr(out), D.stream_handle()))
    return D.host(out)


def bits(a):
    return np.asarray(a, dtype=np.float64).view(np.uint64)


def host(f, *args):
    out = []
    for a in zip(*args):
        try:
            out.append(f(*a))
        except OverflowError:
            out.append(math.inf)
        except (ValueError, ZeroDivisionError):
            out.append(math.nan)
    return np.array(out)


def _check(fn, f, x, y=None):
    got = device_math(fn, x, y)
    want = host(f, x) if y is None else host(f, x, y)
    nan = np.isnan(want)
    assert np.array_equal(np.isnan(got), nan)
    diff = np.flatnonzero(bits(got)[~nan] != bits(want)[~nan])
    assert diff.size == 0, f"{diff.size} of {len(x)} differ; e.g. x={np.asarray(x)[~nan][diff[:3]]}"


def test_exp_bit_exact(cuda):
    rng = np.random.default_rng(7)
    x = np.concatenate([rng.uniform(-30, 30, 200_000), rng.uniform(-745, 710, 50_000), rng.normal(0, 1e-3, 20_000),
                        rng.uniform(-1e-17, 1e-17, 1000), [0.0, -0.0, 1.0, -1.0, 709.78, 709.8, -745.2, -708.5,
                                                           math.log(2), 500.0, -1022 * math.log(2)]])
    x = np.concatenate([x, np.nextafter(x, np.inf)])
    _check(0, math.exp, x)
    got = device_math(0, np.array([np.inf, -np.inf, np.nan]))
    assert got[0] == np.inf and got[1] == 0.0 and np.isnan(got[2])


def test_log_bit_exact(cuda):
    rng = np.random.default_rng(8)
    x = np.concatenate([rng.uniform(1e-6, 60, 200_000), 1.0 + rng.uniform(-0.07, 0.07, 50_000),
                        np.exp(rng.uniform(-700, 700, 50_000)), rng.uniform(0, 1e-308, 1000),
                        [1.0, 1.0 + 1e-6, math.e, 2.0, 0.5, 5e-324]])
    _check(1, math.log, x)


def test_pow_bit_exact(cuda):
    rng = np.random.default_rng(9)
    base = np.concatenate([np.full(100_000, math.e), rng.uniform(1.000001, 8, 100_000), rng.uniform(1e-3, 1, 20_000)])
    expo = np.concatenate([rng.uniform(-20, 40, 100_000), rng.uniform(-60, 60, 100_000), rng.uniform(-200, 200, 20_000)])
    special_b = np.array([2.0, 2.0, 1.0, math.e, math.e, math.e, 0.5, 10.0, 10.0])
    special_e = np.array([0.0, -0.0, 123.0, 1e-30, -1e-30, 1e20, 1074.5, 400.0, -400.0])
    _check(2, lambda a, b: a ** b, np.concatenate([base, special_b]), np.concatenate([expo, special_e]))


def test_log1p_bit_exact(cuda):
    """numpy's ziggurat tails call log1p(-u), u in [0, 1) (distributions.c)."""
    rng = np.random.default_rng(10)
    u = (rng.integers(0, 2 ** 53, 300_000, dtype=np.int64) * 2.0 ** -53)
    x = np.concatenate([-u, rng.uniform(-0.999, 5.0, 100_000), rng.normal(0, 1e-6, 20_000),
                        np.exp(rng.uniform(-40, 40, 20_000)), [0.0, -0.0, -0.5, -0.2929, 0.41422, 1e-300,
                                                                -1e-20, 3e-9, 2.0 ** 53, 1e300]])
    _check(3, math.log1p, x)


def test_certified_division_equals_ieee(cuda):
    """The replay engine's shared-divisor division (div_shared: one reciprocal,
    a Markstein step, an exact residual certificate, __ddiv_rn otherwise)
    equals IEEE binary64 division bit for bit: random operands over wide and
    TWA-like ranges, quotients at powers of two and at ties, and the special
    values that take the fallback."""
    rng = np.random.default_rng(11)
    n = 1_000_000
    a = np.concatenate([rng.uniform(0, 50, n), np.exp(rng.uniform(-700, 700, n // 4)) * rng.choice([-1, 1], n // 4),
                        rng.integers(1, 1 << 53, n // 4).astype(np.float64)])
    b = np.concatenate([rng.uniform(1e-3, 30, n), np.exp(rng.uniform(-700, 700, n // 4)),
                        rng.integers(1, 1 << 20, n // 4).astype(np.float64)])
    # exact quotients (powers of two, small integers) and halfway-adjacent cases
    k = rng.integers(1, 1 << 20, 50_000).astype(np.float64)
    a = np.concatenate([a, k * 8.0, k * 3.0, k + 0.5, [1.0, 0.0, -0.0, np.inf, -np.inf, np.nan, 5e-324, 1e308, 3.0]])
    b = np.concatenate([b, k, np.full(50_000, 3.0), np.full(50_000, 2.0),
                        [3.0, 7.0, 7.0, 2.0, 2.0, 2.0, 3.0, 1e-308, 0.0]])
    got = device_math(4, a, b)
    with np.errstate(all="ignore"):
        want = a / b
    nan = np.isnan(want)
    assert np.array_equal(np.isnan(got), nan)
    diff = np.flatnonzero(bits(got)[~nan] != bits(want)[~nan])
    assert diff.size == 0, f"{diff.size} differ; e.g. {a[~nan][diff[:3]]} / {b[~nan][diff[:3]]}"
