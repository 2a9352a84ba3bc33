"""Pins of the oracle's EPS-v1 generator (docs/EPS.md) against things other than itself.

* Philox4x32-10: Random123 known-answer vectors (tests/golden/philox_kat.txt).
* LOG24 / SINCOS2PI24 / radius: exhaustive sweeps of all 2^24 inputs against fp64 libm.
* ε: distribution (moments, KS vs Φ), Box–Muller pairing identity, reparameterisation
  check of SPEC.md:156 (variational-layers / sample_weights).
"""
import math
import os

import numpy as np
import pytest

import oracle as O

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "philox_kat.txt")


def _kat():
    rows = []
    for line in open(GOLDEN):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        v = [int(t, 16) for t in line.split()]
        rows.append((v[0:4], v[4:6], v[6:10]))
    return rows


@pytest.mark.parametrize("ctr,key,expect", _kat())
def test_philox_known_answers(ctr, key, expect):
    assert [int(v) for v in O.philox(ctr, key)] == expect


def test_log24_exhaustive_vs_libm():
    L = O.log24_all().astype(np.float64)
    u = np.arange(1, (1 << 24) + 1, dtype=np.float64) * 2.0 ** -24
    ref = np.log(u)
    assert L[-1] == 0.0  # u = 1 exactly → ln 1 = 0 exactly
    nz = ref != 0
    ulp = np.spacing(np.abs(ref[nz]).astype(np.float32)).astype(np.float64)
    ulps = np.abs(L[nz] - ref[nz]) / ulp
    assert ulps.max() <= 1.5, ulps.max()
    assert np.all(L <= 0.0)


def test_sincos2pi24_exhaustive_vs_libm():
    c, s = O.sincos2pi24_all()
    ang = 2.0 * np.pi * np.arange(1 << 24, dtype=np.float64) / 2.0 ** 24
    assert np.abs(c - np.cos(ang)).max() <= 1.0e-7
    assert np.abs(s - np.sin(ang)).max() <= 1.0e-7
    # exact special angles
    assert (c[0], s[0]) == (1.0, 0.0)
    assert (c[1 << 22], s[1 << 22]) == (0.0, 1.0)
    assert (c[1 << 23], s[1 << 23]) == (-1.0, 0.0)
    assert (c[3 << 22], s[3 << 22]) == (0.0, -1.0)
    # |(c, s)| = 1 to fp32 accuracy
    assert np.abs(c.astype(np.float64) ** 2 + s.astype(np.float64) ** 2 - 1).max() < 3e-7


def test_radius_exhaustive_vs_libm():
    L = O.log24_all()
    R = np.sqrt((L * np.float32(-2.0)).astype(np.float32)).astype(np.float64)
    u = np.arange(1, (1 << 24) + 1, dtype=np.float64) * 2.0 ** -24
    ref = np.sqrt(-2.0 * np.log(u))
    pos = ref > 0
    rel = np.abs(R[pos] - ref[pos]) / ref[pos]
    assert rel.max() <= 2.0 * 2.0 ** -24, rel.max() / 2.0 ** -24
    assert R.max() <= math.sqrt(48.0 * math.log(2.0)) * (1 + 1e-7)


def test_eps_box_muller_pairing():
    """Columns 4q+{0,1} (and 4q+{2,3}) are the cos/sin halves of one Box–Muller pair."""
    e = O.eps_fill(0x5EED, 3, 5, 2, 7, 1, 0, 4096).ravel().astype(np.float64)
    r2_a = e[0::4] ** 2 + e[1::4] ** 2
    r2_b = e[2::4] ** 2 + e[3::4] ** 2
    for q in range(0, 1024, 37):
        y = O.philox([q, 7, (2 << 20) | 5, 3], [0x5EED, 0])
        for r2, a in ((r2_a[q], y[0]), (r2_b[q], y[2])):
            u = ((int(a) >> 8) + 1) * 2.0 ** -24
            assert r2 == pytest.approx(-2.0 * math.log(u), rel=1e-6, abs=1e-12)
    # the two halves are different draws (a dropped term would make them equal)
    assert not np.allclose(r2_a, r2_b)


def test_eps_distribution():
    from scipy import stats
    e = O.eps_fill(1234, 0, 0, 0, 0, 2048, 0, 1024).ravel().astype(np.float64)
    n = e.size
    assert abs(e.mean()) < 5 / math.sqrt(n)
    assert abs(e.var() - 1) < 5 * math.sqrt(2 / n)
    assert abs(stats.skew(e)) < 5 * math.sqrt(6 / n)
    assert abs(stats.kurtosis(e, fisher=False) - 3) < 5 * math.sqrt(24 / n)
    assert stats.kstest(e, "norm").pvalue > 1e-4
    assert np.abs(e).max() <= math.sqrt(48 * math.log(2)) + 1e-6


def test_eps_keys_are_distinct_streams():
    a = O.eps_fill(7, 0, 0, 0, 0, 4, 0, 256)
    for args in [(8, 0, 0, 0), (7, 1, 0, 0), (7, 0, 1, 0), (7, 0, 0, 1)]:
        seed, step, s, t = args
        b = O.eps_fill(seed, step, s, t, 0, 4, 0, 256)
        assert not np.array_equal(a, b)
    # rows differ too
    assert not np.array_equal(a[0], a[1])
    # determinism
    assert np.array_equal(a, O.eps_fill(7, 0, 0, 0, 0, 4, 0, 256))


def test_reparameterisation_moments():
    """μ=1, σ=0.5, 1e5 draws → mean 1±0.01, std 0.5±0.01."""
    e = O.eps_fill(99, 0, 0, 0, 0, 100, 0, 1000).ravel().astype(np.float64)
    w = 1.0 + 0.5 * e
    assert abs(w.mean() - 1.0) < 0.01
    assert abs(w.std() - 0.5) < 0.01


def test_aug_params_ranges_and_uniformity():
    dxs, dys, fls = [], [], []
    for b in range(4000):
        dx, dy, fl = O.aug_params(5, 1, 3, b)
        dxs.append(dx); dys.append(dy); fls.append(fl)
    for v, hi in ((dxs, 8), (dys, 8), (fls, 1)):
        v = np.array(v)
        assert v.min() == 0 and v.max() == hi
        counts = np.bincount(v, minlength=hi + 1)
        exp = len(v) / (hi + 1)
        assert np.all(np.abs(counts - exp) < 6 * math.sqrt(exp))
