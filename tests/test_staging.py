"""Host-side staging conversions of the drop-in entries (csrc/hostpool.cpp),
checked on the CPU against numpy: no device needed.

The native-precision histogram ships fp32 rounded toward -inf, which must
keep floor(v * 2^k) of the float64 value for every v (the reference bins
in float64, tasklets.py:432-433); the native query narrows a chunk only if
every value round-trips (otherwise it keeps float64)."""

import ctypes

import numpy as np
import pytest

from paper_1902_10345_b200 import _lib

L = _lib.load()


def _conv(kind, src, dst, lo=0, hi=0):
    return L.sdfgb_host_convert(kind, src.ctypes.data, dst.ctypes.data if dst is not None else None,
                                src.size, lo, hi)


def _edge_values(rng, n):
    f = rng.random(n)
    specials = np.array([0.0, -0.0, 1.0, 1 - 2.0 ** -25, 1 - 2.0 ** -53, 0.5, 0.5 - 2.0 ** -40, -1e-300, 1e-300,
                         -2.0 ** -149, 2.0 ** -150, 3.4028235e38, 3.5e38, -3.5e38, np.inf, -np.inf, np.nan,
                         255.99999999, -0.0039, 16777217.0, -16777217.0])
    mixed = np.concatenate([f, f * 1e6 - 5e5, np.nextafter(f, 2), np.nextafter(f, -2),
                            f.astype(np.float32).astype(np.float64), specials])
    return mixed


def test_round_toward_minus_infinity_is_the_largest_float_below():
    rng = np.random.default_rng(0)
    v = _edge_values(rng, 100000)
    out = np.empty(v.size, np.float32)
    _conv(1, v, out)
    fin = ~np.isnan(v)
    o = out[fin].astype(np.float64)
    assert np.all(o <= v[fin])
    # nothing representable lies strictly between: the next float up is above v
    with np.errstate(over="ignore"):
        up = np.nextafter(out[fin], np.float32(np.inf)).astype(np.float64)
    assert np.all((up > v[fin]) | (out[fin] == np.float32(np.inf)))
    assert np.isnan(out[~fin]).all()


@pytest.mark.parametrize("scale,div", [(256.0, 1.0), (1.0, 1.0), (4096.0, 16.0), (2.0 ** 20, 1.0), (0.5, 2.0)])
def test_power_of_two_binning_survives_rounding_down(scale, div):
    """floor(v*S/D) of the float64 value == floor of the fp32 value rounded
    toward -inf, for power-of-two S, D -- including values just below a bin
    edge that round-to-nearest would push into the next bin."""
    rng = np.random.default_rng(1)
    v = _edge_values(rng, 200000)
    v = v[np.isfinite(v)]
    out = np.empty(v.size, np.float32)
    _conv(1, v, out)
    with np.errstate(over="ignore", invalid="ignore"):
        ref = np.floor(v * scale / div)
        got = np.floor(out.astype(np.float64) * scale / div)
    inside = (ref >= 0) & (ref < 2 ** 24)
    np.testing.assert_array_equal(got[inside], ref[inside])
    # outside stays outside (the out-of-bounds count is exact too)
    assert np.all((got[~inside] < 0) | (got[~inside] >= 2 ** 24) | ~np.isfinite(got[~inside]))
    # round-to-nearest would not be exact here
    rn = np.empty(v.size, np.float32)
    _conv(0, v, rn)
    assert np.any(np.floor(rn.astype(np.float64) * scale / div) != ref)


def test_exact_narrowing_detects_any_inexact_value():
    rng = np.random.default_rng(2)
    x = rng.random(300000, dtype=np.float32).astype(np.float64)
    out = np.empty(x.size, np.float32)
    assert _conv(2, x, out) == 1
    np.testing.assert_array_equal(out, x.astype(np.float32))
    for bad in (1 / 3, np.nan, 1e-50, 1e39):
        y = x.copy()
        y[rng.integers(0, y.size)] = bad
        assert _conv(2, y, out) == 0


def test_widen_and_round_to_nearest_match_numpy():
    rng = np.random.default_rng(3)
    v = _edge_values(rng, 50000)
    out = np.empty(v.size, np.float32)
    _conv(0, v, out)
    with np.errstate(over="ignore"):
        np.testing.assert_array_equal(out, v.astype(np.float32))
    w = np.empty(v.size, np.float64)
    _conv(3, out, w)
    np.testing.assert_array_equal(w, out.astype(np.float64))


def test_index_narrowing_counts_out_of_range():
    rng = np.random.default_rng(4)
    idx = rng.integers(0, 1000, 500000).astype(np.int64)
    out = np.empty(idx.size, np.int32)
    assert _conv(4, idx, out, 0, 1000) == 0
    np.testing.assert_array_equal(out, idx.astype(np.int32))
    idx[[7, 123456, 499999]] = [-1, 1000, 2 ** 40]
    assert _conv(4, idx, out, 0, 1000) == 3


def test_non_decreasing_across_task_boundaries():
    rp = np.arange(1 << 18, dtype=np.int64) // 3
    assert _conv(5, rp, None) == 1
    for pos in (1, 1 << 16, (1 << 16) + 1, rp.size - 1):  # inside a task and at task edges
        bad = rp.copy()
        bad[pos] = bad[pos - 1] - 1
        assert _conv(5, bad, None) == 0


def test_host_threads_reported():
    assert L.sdfgb_host_threads() >= 1
