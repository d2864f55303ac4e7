"""Pins for oracle/philox.py, oracle/logf.py and oracle/sampler.py (CPU only)."""
import os
import shutil
import subprocess
import tempfile

import numpy as np
import pytest

from oracle.logf import logf
from oracle.philox import bits_to_uniform, philox4x32_10, sampler_bits
from oracle.sampler import gumbel, sample_row

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _kat_rows():
    rows = []
    with open(os.path.join(GOLD, "philox4x32_10_kat.txt")) as fh:
        for line in fh:
            if line.startswith("#") or not line.strip():
                continue
            rows.append([int(x, 16) for x in line.split()])
    return rows


def test_philox_known_answer_vectors():
    """Random123 kat_vectors (tests/golden/philox4x32_10_kat.txt)."""
    for c0, c1, c2, c3, k0, k1, *want in _kat_rows():
        got = philox4x32_10(c0, c1, c2, c3, k0, k1)
        assert [int(x) for x in got] == want


_CURAND_PROG = r"""
#define QUALIFIERS static inline
#include <vector_types.h>
#include <curand_philox4x32_x.h>
#include <stdio.h>
int main(){
  unsigned s = 12345u;
  for (int i = 0; i < 64; ++i) {
    s = s * 1664525u + 1013904223u; unsigned a = s;
    s = s * 1664525u + 1013904223u; unsigned b = s;
    s = s * 1664525u + 1013904223u; unsigned c = s;
    s = s * 1664525u + 1013904223u; unsigned d = s;
    s = s * 1664525u + 1013904223u; unsigned k0 = s;
    s = s * 1664525u + 1013904223u; unsigned k1 = s;
    uint4 ctr = {a, b, c, d}; uint2 key = {k0, k1};
    uint4 r = curand_Philox4x32_10(ctr, key);
    printf("%u %u %u %u %u %u %u %u %u %u\n", a, b, c, d, k0, k1, r.x, r.y, r.z, r.w);
  }
  return 0;
}
"""


@pytest.mark.skipif(not os.path.exists("/usr/local/cuda/include/curand_philox4x32_x.h")
                    or shutil.which("g++") is None, reason="needs the CUDA headers and g++")
def test_philox_matches_curand_host_implementation():
    """Independent implementation: NVIDIA curand's Philox4x32-10 (host path of the header)."""
    with tempfile.TemporaryDirectory() as d:
        src, exe = os.path.join(d, "p.cpp"), os.path.join(d, "p")
        with open(src, "w") as fh:
            fh.write(_CURAND_PROG)
        subprocess.check_call(["g++", "-O1", "-I/usr/local/cuda/include", src, "-o", exe])
        out = subprocess.check_output([exe]).decode().split("\n")
    rows = [list(map(int, l.split())) for l in out if l.strip()]
    assert len(rows) == 64
    for a, b, c, d, k0, k1, *want in rows:
        got = philox4x32_10(a, b, c, d, k0, k1)
        assert [int(x) for x in got] == want


def test_uniform_exact_and_open_interval():
    x = np.array([0, 1, 511, 512, 0xFFFFFFFF, 0x80000000], dtype=np.uint32)
    u = bits_to_uniform(x)
    assert u.dtype == np.float32
    np.testing.assert_array_equal(u.astype(np.float64), (2.0 * (x.astype(np.float64) // 512) + 1) * 2.0 ** -24)
    assert (u > 0).all() and (u < 1).all()


def test_sampler_bits_counter_layout():
    """word j&3 of Philox(counter=(j>>2, n, traj, restarts), key=(seed_lo, seed_hi))."""
    seed = 0x123456789
    j = np.arange(10)
    got = sampler_bits(seed, j, 5, 77, 2)
    for jj in j:
        w = philox4x32_10(jj >> 2, 5, 77, 2, seed & 0xFFFFFFFF, seed >> 32)
        assert int(got[jj]) == int(w[jj & 3])


def _ulp32(x):
    x = np.abs(np.asarray(x, dtype=np.float32))
    return np.spacing(x).astype(np.float64)


def test_logf_within_one_ulp_of_exact_log():
    """msun logf's documented error bound is < 1 ulp; a transcription slip breaks it."""
    rng = np.random.default_rng(0)
    xs = np.concatenate([
        rng.uniform(0, 1, 200000).astype(np.float32),
        rng.uniform(0, 20, 200000).astype(np.float32),
        np.exp(rng.uniform(-80, 80, 100000)).astype(np.float32),
        (1 + rng.uniform(-2e-3, 2e-3, 50000)).astype(np.float32),    # the |f| < 2^-9 branch
        np.array([2.0 ** -24, 1 - 2.0 ** -24, 0.5, 2.0, 3.0, 1e-30, 1e-40, 3e38], dtype=np.float32),
    ])
    xs = xs[xs > 0]
    got = logf(xs).astype(np.float64)
    exact = np.log(xs.astype(np.float64))
    err = np.abs(got - exact)
    assert (err <= _ulp32(got) * 1.0 + 1e-300).all(), float((err / _ulp32(got)).max())


def test_logf_special_values():
    assert logf(np.float32(1.0))[0] == 0.0
    assert np.isneginf(logf(np.float32(0.0))[0])
    assert np.isnan(logf(np.float32(-1.0))[0])
    assert np.isposinf(logf(np.float32(np.inf))[0])
    # log(2^k) = k*ln2 rounded (k*ln2_hi + k*ln2_lo)
    for k in (-100, -3, 1, 7, 100):
        v = logf(np.float32(2.0 ** k))[0]
        assert abs(float(v) - k * np.log(2.0)) <= np.spacing(np.float32(abs(v)))


def test_gumbel_noise_distribution():
    """g = -log(-log(u)) ~ Gumbel(0,1): mean = Euler gamma, var = pi^2/6."""
    g = np.concatenate([gumbel(3, 4096, n, 1, 0) for n in range(64)]).astype(np.float64)
    assert abs(g.mean() - 0.5772156649) < 0.01
    assert abs(g.var() - np.pi ** 2 / 6) < 0.03


def test_sampler_low_temperature_is_argmax():
    rng = np.random.default_rng(1)
    z = rng.normal(size=512).astype(np.float32)
    tok, lp, _ = sample_row(z, np.float32(1e6), 3, 0, 0, 0)
    assert tok == int(np.argmax(z))


def test_sampler_logprob_closed_forms():
    """log pi(tok) for logits z_j = ln w_j is ln(w_tok / sum w) (P:180 caches this
    value); at temperature T the policy is softmax(z / T), i.e. p_j ~ w_j^(1/T);
    a common shift of the logits changes nothing."""
    w = np.array([1.0, 2.0, 3.0, 4.0])
    z = np.log(w).astype(np.float32)
    for n in range(20):
        tok, lp, _ = sample_row(z, np.float32(1.0), 3, n, 9, 1)
        assert abs(lp - np.log(w[tok] / w.sum())) < 1e-6
        tok2, lp2, _ = sample_row(z + np.float32(5.0), np.float32(1.0), 3, n, 9, 1)
        assert tok2 == tok and abs(lp2 - lp) < 1e-6
        T = 0.5
        tok3, lp3, _ = sample_row(z, np.float32(1.0 / T), 3, n, 9, 1)
        assert abs(lp3 - np.log(w[tok3] ** 2 / (w ** 2).sum())) < 1e-6
    tok, lp, _ = sample_row(np.zeros(8, np.float32), np.float32(1.0), 3, 0, 0, 0)
    assert abs(lp + np.log(8.0)) < 1e-12


def test_gumbel_max_frequencies_match_softmax_chi2():
    """Gumbel-max draws are softmax samples (chi-square over 8 categories)."""
    from scipy.stats import chisquare
    z = np.array([0.0, 1.0, -1.0, 0.5, 2.0, -0.5, 0.25, 1.5], dtype=np.float32)
    p = np.exp(z - z.max()).astype(np.float64)
    p /= p.sum()
    counts = np.zeros(8)
    N = 20000
    for n in range(N):
        tok, _, _ = sample_row(z, np.float32(1.0), 11, n, 5, 0)
        counts[tok] += 1
    stat, pval = chisquare(counts, p * N)
    assert pval > 1e-3, (counts, p * N)


def test_sampler_ties_lowest_index():
    """Two perturbed scores made exactly equal (fp32) and larger than all others:
    the token is the lower index, wherever the pair sits."""
    from oracle.sampler import gumbel
    for (i, j) in [(0, 1), (3, 6), (2, 7)]:
        g = gumbel(3, 8, 0, 0, 0)
        z = np.full(8, -1e4, np.float32)
        z[i] = np.float32(0.0)
        target = np.float32(g[i])                     # s_i = 0 + g_i
        d = np.float32(target - g[j])
        for _ in range(64):                           # nudge z_j until fl(z_j + g_j) == s_i exactly
            s_j = np.float32(d + g[j])
            if s_j == target:
                break
            d = np.nextafter(d, np.float32(np.inf) if s_j < target else np.float32(-np.inf), dtype=np.float32)
        z[j] = d
        tok, _, s = sample_row(z, np.float32(1.0), 3, 0, 0, 0)
        assert s[i] == s[j] == s.max()
        assert tok == i


# ------------------------------------------------------------------ top-k / top-p (N4)
def test_truncation_set_definitions():
    """top-k keeps the k best by (logit desc, index asc); top-p the shortest ranked
    prefix reaching mass p under the (top-k) softmax, including the crossing token."""
    from oracle.sampler import truncation_set
    z = np.log(np.array([0.1, 0.4, 0.2, 0.2, 0.05, 0.05])).astype(np.float32)
    m, _, _ = truncation_set(z, top_k=3)
    assert m.tolist() == [False, True, True, True, False, False]          # ties 0.2/0.2 both in, 0.1 out
    m, _, _ = truncation_set(z, top_k=2)
    assert m.tolist() == [False, True, True, False, False, False]         # tie broken by the lower index
    m, lo, hi = truncation_set(z, top_p=0.5)
    assert m.tolist() == [False, True, True, False, False, False] and abs(hi - 0.6) < 1e-6
    m, lo, hi = truncation_set(z, top_p=0.39)
    assert m.tolist() == [False, True, False, False, False, False]        # the first token already reaches p
    m, lo, hi = truncation_set(z, top_p=0.41)
    assert m.tolist() == [False, True, True, False, False, False]         # the crossing token is included
    m, _, _ = truncation_set(z, top_k=3, top_p=0.55)                      # renormalised over top-3: .5 .25 .25
    assert m.tolist() == [False, True, True, False, False, False]
    m, _, _ = truncation_set(z, top_k=3, top_p=0.45)
    assert m.tolist() == [False, True, False, False, False, False]
    m, _, _ = truncation_set(z, top_k=0, top_p=1.0)
    assert m.all()


def test_top_k_one_is_greedy_and_logprob_zero():
    z = np.random.default_rng(4).normal(size=1000).astype(np.float32)
    for n in range(5):
        tok, lp, _ = sample_row(z, np.float32(1.0), 3, n, 7, 0, top_k=1)
        assert tok == int(np.argmax(z)) and lp == 0.0


def test_top_p_draws_follow_the_renormalised_distribution():
    """Gumbel-max over the truncation set samples softmax restricted to it (chi-square),
    and the returned logprob is the log of that renormalised probability."""
    from scipy.stats import chisquare
    p = np.array([0.3, 0.25, 0.2, 0.15, 0.06, 0.04])
    z = np.log(p).astype(np.float32)
    q = p[:3] / p[:3].sum()                       # top_p 0.7 keeps 0.3 + 0.25 + 0.2 = 0.75
    counts = np.zeros(6)
    for n in range(12000):
        tok, lp, _ = sample_row(z, np.float32(1.0), 5, n, 1, 0, top_p=0.7)
        counts[tok] += 1
        assert abs(lp - np.log(q[tok])) < 1e-6
    assert counts[3:].sum() == 0
    assert chisquare(counts[:3], q * counts.sum()).pvalue > 1e-3
