"""Pins for oracle/learner.py (CPU only): the SPEC's worked examples,
closed forms and invariants of PAPER.md Eq. (1)-(3), and the direct double-sum
definition of Eq. (2) against the backward recursion."""
import math
import random

import numpy as np
import pytest

from oracle.learner import LearnerError, gae_advantages, ppo_terms, reinforcepp_advantages, token_staleness


# ---------------------------------------------------------------- Eq. (3)
def test_reinforcepp_spec_example():
    """rewards [1,0,1,0] -> mu 0.5, sigma 0.5 -> [1,-1,1,-1]."""
    np.testing.assert_array_equal(reinforcepp_advantages([1, 0, 1, 0]), [1.0, -1.0, 1.0, -1.0])


def test_reinforcepp_degenerate_and_error():
    np.testing.assert_array_equal(reinforcepp_advantages([0.7] * 5), np.zeros(5))
    with pytest.raises(LearnerError):
        reinforcepp_advantages([3.0])


def test_reinforcepp_normalisation_invariant():
    """mean 0 and POPULATION std 1 (not the n-1 sample std) to 1e-9."""
    rng = np.random.default_rng(0)
    for n in (2, 3, 64, 1024):
        a = reinforcepp_advantages(rng.normal(3, 2, size=n))
        assert abs(a.mean()) < 1e-9 and abs(np.sqrt((a * a).mean()) - 1) < 1e-9
    a = reinforcepp_advantages([0.0, 3.0])                # population std of {0,3} is 1.5
    np.testing.assert_allclose(a, [-1.0, 1.0], rtol=0, atol=1e-15)


# ---------------------------------------------------------------- Eq. (2)
def test_gae_spec_examples():
    """gamma=lambda=1, values 0, rewards [1,0,2] -> [3,2,2]; lambda=0 -> delta;
    zeros -> zeros."""
    np.testing.assert_array_equal(gae_advantages([1, 0, 2], [0, 0, 0, 0], 1.0, 1.0), [3.0, 2.0, 2.0])
    r, v = [0.5, -1.0, 2.0], [0.1, 0.2, 0.3, 0.4]
    delta = [r[t] + 0.9 * v[t + 1] - v[t] for t in range(3)]
    np.testing.assert_allclose(gae_advantages(r, v, 0.9, 0.0), delta, rtol=0, atol=1e-15)
    np.testing.assert_array_equal(gae_advantages([0, 0], [0, 0, 0], 0.99, 0.95), [0.0, 0.0])
    with pytest.raises(LearnerError):
        gae_advantages([1, 2], [0, 0], 1.0, 1.0)


def test_gae_recursion_equals_direct_double_sum():
    """S:388 / S:408: the backward recursion equals the direct definition
    A_t = sum_l (gamma lambda)^l delta_{t+l} on 1000 random instances (1e-12 rel)."""
    rng = random.Random(1)
    for _ in range(1000):
        T = rng.randint(1, 64)
        r = [rng.uniform(-2, 2) for _ in range(T)]
        v = [rng.uniform(-2, 2) for _ in range(T + 1)]
        g, lam = rng.uniform(0, 1), rng.uniform(0, 1)
        delta = [r[t] + g * v[t + 1] - v[t] for t in range(T)]
        direct = [sum((g * lam) ** l * delta[t + l] for l in range(T - t)) for t in range(T)]
        got = gae_advantages(r, v, g, lam)
        for a, b in zip(got, direct):
            assert abs(a - b) <= 1e-12 * max(1.0, abs(b))


def test_gae_lambda_one_is_discounted_return_minus_value():
    """lambda = 1 telescopes: A_t = sum_l gamma^l r_{t+l} + gamma^(T-t) V_T - V_t."""
    r, v, g = [1.0, -0.5, 2.0, 0.25], [0.3, -0.2, 0.5, 0.1, 0.7], 0.9
    T = len(r)
    want = [sum(g ** l * r[t + l] for l in range(T - t)) + g ** (T - t) * v[T] - v[t] for t in range(T)]
    np.testing.assert_allclose(gae_advantages(r, v, g, 1.0), want, rtol=0, atol=1e-14)


# ---------------------------------------------------------------- Eq. (1)
def test_ppo_spec_examples():
    """identity ratios -> mean advantage; ratio 2, A=1, eps .2 -> 1.2;
    ratio .5, A=-1 -> min(-0.5, -0.8) = -0.8."""
    a = np.array([0.3, -1.2, 2.0])
    ratio, term, grad, obj = ppo_terms(np.zeros(3), np.zeros(3), a, 0.2, 0.2)
    np.testing.assert_array_equal(ratio, [1, 1, 1])
    assert obj == pytest.approx(a.mean(), abs=1e-15)
    _, term, grad, _ = ppo_terms([math.log(2.0)], [0.0], [1.0], 0.2, 0.2)
    assert term[0] == pytest.approx(1.2, abs=1e-15) and grad[0] == 0.0
    _, term, grad, _ = ppo_terms([math.log(0.5)], [0.0], [-1.0], 0.2, 0.2)
    assert term[0] == pytest.approx(-0.8, abs=1e-15) and grad[0] == 0.0


def test_ppo_clip_higher_and_gradient_branches():
    """Clip-higher: the upper bound uses eps_high, the lower eps_low.  With A > 0
    the ratio is capped at 1 + eps_high, with A < 0 floored at 1 - eps_low; inside the
    range the term is rho A with derivative rho A (d rho / d log pi = rho)."""
    lp = [math.log(1.25), math.log(1.25), math.log(0.7), math.log(0.7), math.log(1.05)]
    A = [1.0, -1.0, 1.0, -1.0, 2.0]
    ratio, term, grad, obj = ppo_terms(lp, [0.0] * 5, A, 0.2, 0.28)
    np.testing.assert_allclose(term, [1.25, -1.25, 0.7, -0.8, 2.1], atol=1e-14)
    np.testing.assert_allclose(grad, [1.25, -1.25, 0.7, 0.0, 2.1], atol=1e-14)
    assert obj == pytest.approx(np.mean([1.25, -1.25, 0.7, -0.8, 2.1]), abs=1e-14)
    _, term, grad, _ = ppo_terms([math.log(1.4)], [0.0], [1.0], 0.2, 0.28)
    assert term[0] == pytest.approx(1.28, abs=1e-14) and grad[0] == 0.0
    with pytest.raises(LearnerError):
        ppo_terms([float("nan")], [0.0], [1.0], 0.2, 0.2)


# ---------------------------------------------------------------- staleness
def test_token_staleness_spec_segments():
    """S:366 segments (v3:5)(v4:7)(v5:2), updated at version 5 -> 2 x5, 1 x7, 0 x2."""
    assert token_staleness([3] * 5 + [4] * 7 + [5] * 2, 5) == {2: 5, 1: 7, 0: 2}
