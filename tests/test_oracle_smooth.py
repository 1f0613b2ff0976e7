"""Pins of the oracle's smooth operators (§II-A) against
closed forms, limits and invariants (SPEC examples S:33-77)."""
import math

import numpy as np
import pytest

TAU = 1e-3


def test_sigmoid_examples(oracle_mod):
    O = oracle_mod
    # sigma((x-a)/tau) at x = a, a + tau, a + 40 tau
    assert O.sigmoid(0.0) == 0.5
    assert abs(O.sigmoid(1.0) - 1.0 / (1.0 + math.exp(-1.0))) < 1e-15
    assert abs(O.sigmoid(40.0) - 1.0) < 1e-12
    # complement
    for x in np.linspace(-50, 50, 101):
        assert abs(O.sigmoid(x) + O.sigmoid(-x) - 1.0) < 1e-12
    # overflow-safe far tails
    assert O.sigmoid(-800.0) == 0.0 and O.sigmoid(800.0) == 1.0


def test_softplus_examples(oracle_mod):
    O = oracle_mod
    # S:48-50
    assert abs(O.softplus(0.0, TAU) - TAU * math.log(2.0)) < 1e-18
    assert abs(O.softplus(100 * TAU, TAU) - 100 * TAU) <= 1e-12 * 100 * TAU
    assert abs(O.softplus(-100 * TAU, TAU)) < 1e-12
    # s+(x) >= max(x,0), s+(x) - max(x,0) <= tau ln 2, and s+(x) - s+(-x) = x
    for x in np.linspace(-0.01, 0.01, 201):
        s = O.softplus(x, TAU)
        assert s >= max(x, 0.0)
        assert s - max(x, 0.0) <= TAU * math.log(2.0) + 1e-18
        assert abs(s - O.softplus(-x, TAU) - x) < 1e-15


def test_softclip_limits(oracle_mod):
    """The composition lo + s+(x-lo) - s+(x-hi) saturates exactly at
    lo and hi (S:58 is wrong), and is the identity inside."""
    O = oracle_mod
    assert abs(O.softclip(1.0 + 100 * TAU, 0.0, 1.0, TAU) - 1.0) < 1e-12
    assert abs(O.softclip(-100 * TAU, 0.0, 1.0, TAU)) < 1e-12
    assert O.softclip(0.5, 0.0, 1.0, TAU) == pytest.approx(0.5, abs=1e-15)
    for x in np.linspace(5 * TAU, 1 - 5 * TAU, 97):
        assert abs(O.softclip(x, 0.0, 1.0, TAU) - x) < 0.01 * TAU
    # monotone, and range (lo, hi)
    xs = np.linspace(-0.01, 1.01, 1001)
    ys = [O.softclip(x, 0.0, 1.0, TAU) for x in xs]
    assert all(b >= a for a, b in zip(ys, ys[1:]))
    assert min(ys) >= 0.0 and max(ys) <= 1.0
    # at the bounds: softclip(lo) = lo + tau ln 2 (to within e^{-(hi-lo)/tau})
    assert abs(O.softclip(0.0, 0.0, 1.0, TAU) - TAU * math.log(2.0)) < 1e-15


def test_lse_examples_and_sandwich(oracle_mod):
    O = oracle_mod
    tau = 1e-2
    a = 0.37
    assert O.lse([a], tau) == a
    assert abs(O.lse([a, a], tau) - (a + tau * math.log(2.0))) < 1e-15
    v = O.lse([0.0, 10 * tau, -5 * tau], tau)
    assert 10 * tau <= v <= 10 * tau + tau * math.log(3.0)
    rng = np.random.default_rng(0)
    for _ in range(2000):
        k = rng.integers(1, 9)
        x = rng.normal(0, 0.05, k)
        v = O.lse(x, tau)
        assert x.max() - 1e-15 <= v <= x.max() + tau * math.log(k) + 1e-15
        # min form: min(x) - tau ln k <= -lse(-x) <= min(x)
        m = -O.lse(-x, tau)
        assert x.min() - tau * math.log(k) - 1e-15 <= m <= x.min() + 1e-15
    # shift stability: inputs of hundreds of tau
    assert abs(O.lse([500 * tau, 0.0], tau) - 500 * tau) < 1e-15


def test_softargmax(oracle_mod):
    O = oracle_mod
    tau = 1e-2
    w = O.softargmax([0.0, tau * math.log(3.0)], tau)
    assert np.allclose(w, [0.25, 0.75], atol=1e-14)
    assert np.allclose(O.softargmax([0.3] * 5, tau), 0.2)
    w = O.softargmax([0.0, 50 * tau, 0.01], tau)
    assert w[1] > 1 - 1e-12
    rng = np.random.default_rng(1)
    for _ in range(500):
        x = rng.normal(0, 0.03, 6)
        w = O.softargmax(x, tau)
        assert abs(w.sum() - 1.0) < 1e-12
        assert np.allclose(O.softargmax(x + 0.123, tau), w, atol=1e-14)
        assert np.argmax(w) == np.argmax(x)
