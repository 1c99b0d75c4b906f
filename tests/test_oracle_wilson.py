"""Pins for the oracle's statistics: Eq. 3, Eq. 4, Fig. 2 and z.  No GPU."""
import json
import math
import os

import mpmath
import numpy as np
import pytest

from oracle import normal_quantile, round_estimate, wilson_interval, wilson_procedure, wilson_sample_size

HERE = os.path.dirname(os.path.abspath(__file__))
Z99 = normal_quantile(0.99)


def test_z_values_spec():
    # q=0.975 -> 1.95996398, q=0.995 -> 2.57582930 (+-1e-8)
    assert abs(normal_quantile(0.95) - 1.95996398) < 1e-8
    assert abs(normal_quantile(0.99) - 2.57582930) < 1e-8


@pytest.mark.parametrize("c", [0.5, 0.8, 0.9, 0.95, 0.99, 0.995, 0.999, 0.9999, 0.99999])
def test_z_is_nearest_double(c):
    """Phi(z) = (1+c)/2 at 50 digits; z beats both neighbouring doubles."""
    z = normal_quantile(c)
    with mpmath.workdps(60):
        q = (1 + mpmath.mpf(c)) / 2

        def err(v):
            return abs(mpmath.ncdf(mpmath.mpf(v)) - q)
        e = err(z)
        assert e <= err(np.nextafter(z, np.inf)) and e <= err(np.nextafter(z, -np.inf))
        assert e < mpmath.mpf("1e-15")


def test_eq4_paper_values():
    # conservative (p = 0.5) sample size at 99 %, eps = 0.025
    assert wilson_sample_size(0.5, 0.025, Z99) == 2648
    # start at p = 1
    assert wilson_sample_size(1.0, 0.025, Z99) == 127
    # floor after rounding p = 0 -> 0.025
    assert wilson_sample_size(0.025, 0.025, Z99) == 304
    # "up to 88%": 1 - 304/2648
    assert math.floor(100 * (1 - 304 / 2648)) == 88


def test_eq4_closed_form_p1():
    # at p = 1 the bracket is -2e^2 + sqrt(4 e^2 0.25) = e - 2e^2
    for eps in [0.1, 0.025, 0.005, 1e-4]:
        z = normal_quantile(0.999)
        with mpmath.workdps(50):
            exact = mpmath.mpf(z) ** 2 * (eps - 2 * mpmath.mpf(eps) ** 2) / (2 * mpmath.mpf(eps) ** 2)
        assert wilson_sample_size(1.0, eps, z) == int(mpmath.ceil(exact))


def test_eq4_symmetry_and_maximum():
    for eps in [0.025, 0.005]:
        ps = np.linspace(0, 1, 201)
        ns = [wilson_sample_size(p, eps, Z99) for p in ps]
        for p, n in zip(ps, ns):
            assert abs(n - wilson_sample_size(1 - p, eps, Z99)) <= 1   # symmetric up to rounding of 1-p
        assert max(ns) == wilson_sample_size(0.5, eps, Z99)


def test_eq3_against_mpmath_grid():
    g = np.random.default_rng(0)
    for _ in range(1000):
        n = int(g.integers(1, 10**7))
        k = int(g.integers(0, n + 1))
        c = float(g.choice([0.9, 0.95, 0.99, 0.999, 0.9999]))
        z = normal_quantile(c)
        lo, hi = wilson_interval(k / n, n, z)
        with mpmath.workdps(50):
            p = mpmath.mpf(k) / n
            zz = mpmath.mpf(z) ** 2
            cen = p + zz / (2 * n)
            r = mpmath.mpf(z) * mpmath.sqrt(p * (1 - p) / n + zz / (4 * mpmath.mpf(n) ** 2))
            den = 1 + zz / n
            L = max(mpmath.mpf(0), (cen - r) / den)
            U = min(mpmath.mpf(1), (cen + r) / den)
        assert abs(lo - L) <= 1e-9 and abs(hi - U) <= 1e-9      # S:484 bar
        assert abs(lo - L) <= 4e-15 * max(1.0, float(hi)) and abs(hi - U) <= 4e-15


def test_eq3_spec_example_and_zero():
    z = normal_quantile(0.95)
    lo, hi = wilson_interval(0.5, 100, z)
    assert abs(lo - 0.40383) < 1e-5 and abs(hi - 0.59617) < 1e-5
    lo, hi = wilson_interval(0.0, 1000, Z99)
    assert lo < 1e-15                                                 # S:341 (algebraic zero)
    # large-n: width -> Wald width 2 z sqrt(p(1-p)/n)
    lo, hi = wilson_interval(0.3, 10**6, Z99)
    wald = 2 * Z99 * math.sqrt(0.3 * 0.7 / 1e6)
    assert abs((hi - lo) / wald - 1) < 0.01


def _trunc(x, digits):
    return math.floor(x * 10**digits) / 10**digits


def test_table3_rows_from_counts():
    """Table 3 rows 2, 4, 5 reproduced from integer counts; the paper truncates."""
    t3 = json.load(open(os.path.join(HERE, "golden", "table3.json")))
    for row in t3["rows"]:
        n, s = row["N"], row["successes"]
        p = s / n
        lo, hi = wilson_interval(p, n, Z99)
        for printed, val in [(row["p_hat"], p), (row["L"], lo), (row["U"], hi)]:
            d = len(printed.split(".")[1])
            assert _trunc(val, d) == float(printed), (row, printed, val)


def test_fig2_scripted_extremes():
    # always-0 source: 127, then N' = 304, second batch 177, stop at 304
    calls = []

    def zero(first, n):
        calls.append((first, n))
        return 0
    r = wilson_procedure(zero, 0.025, 0.99)
    assert calls == [(0, 127), (127, 177)]
    assert r["n_total"] == 304 and r["p_hat"] == 0.0
    # always-1 source is the mirror image
    r1 = wilson_procedure(lambda f, n: n, 0.025, 0.99)
    assert r1["n_total"] == 304 and r1["p_hat"] == 1.0
    # Fig. 2 rounding: towards 0.5
    assert round_estimate(0.2, 0.025) == 0.2 + 0.025 and round_estimate(0.8, 0.025) == 0.8 - 0.025
    assert round_estimate(0.5, 0.025) == 0.525


def _bernoulli_source(p, g):
    return lambda first, n: int(g.binomial(n, p))


def test_fig2_half_reaches_conservative():
    """p = 0.5: iterative N concentrates at the conservative 2648 ("using the same sample size
    for p close to 0.5").  Fig. 2 rounds p-hat by +-eps, so p' is rarely
    exactly 0.5 and N' = Eq. 4(p') <= 2648: the mean sits just below 2648 (S:485's lower
    bound 2648 does not hold for Fig. 2 as written)."""
    g = np.random.default_rng(5)
    ns = [wilson_procedure(_bernoulli_source(0.5, g), 0.025, 0.99)["n_total"] for _ in range(100)]
    assert 0.99 * 2648 <= np.mean(ns) <= 2648
    assert max(ns) <= 2648


def test_fig2_reduction_at_extremes():
    """S:485 / P:392: mean N at p in {0.01, 0.99} <= 25 % of 2648."""
    g = np.random.default_rng(6)
    for p in [0.01, 0.99]:
        ns = [wilson_procedure(_bernoulli_source(p, g), 0.025, 0.99)["n_total"] for _ in range(100)]
        assert np.mean(ns) <= 0.25 * 2648


def test_fig2_coverage():
    """coverage >= 97 % for p in {0.05, ..., 0.95} (nominal 99 %)."""
    g = np.random.default_rng(7)
    for p in np.arange(0.05, 1.0, 0.1):
        hits = 0
        reps = 500
        for _ in range(reps):
            r = wilson_procedure(_bernoulli_source(float(p), g), 0.025, 0.99)
            hits += r["lower"] <= p <= r["upper"]
        assert hits / reps >= 0.97, (p, hits)


def test_fig2_monotone_batches():
    g = np.random.default_rng(8)
    for p in [0.0, 0.02, 0.3, 0.5, 0.9]:
        r = wilson_procedure(_bernoulli_source(p, g), 0.005, 0.99)
        ns = [e["n"] for e in r["log"]]
        assert all(n > 0 for n in ns)
        assert r["n_total"] <= wilson_sample_size(0.5, 0.005, Z99)
