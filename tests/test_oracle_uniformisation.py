"""Brute-force pins for SSA + on-the-fly checker: transient solution of tiny
CTMCs (<= 200 states for the generic cases) by the matrix exponential, i.e. the
CME the SSA samples, made absorbing for top-level
lower-bound-0 until formulas.  No GPU.

P(phi' U[0,T] phi'') = P(the jump chain enters a phi''-state at time <= T
having visited only phi'-states before) = mass on the absorbing success set at
T when phi''-states and (not phi' and not phi'')-states are made absorbing."""
import math

import numpy as np
import pytest
from scipy.linalg import expm

from oracle import normal_quantile, wilson_interval
from oracle import oracle as O


def _mass_action(x, reactants, c):
    h = 1
    for s, st in reactants:
        if x[s] < st:
            return 0.0
        h *= x[s] if st == 1 else x[s] * (x[s] - 1) // 2
    return c * h


def _until_probability(x0, reactions, phi1, phi2, T, max_states=5000):
    """reactions: [(reactants, change dict, c)].  BFS over reachable states."""
    idx = {}
    states = []
    todo = [tuple(x0)]
    idx[tuple(x0)] = 0
    states.append(tuple(x0))
    while todo:
        x = todo.pop()
        if phi2(x) or not phi1(x):
            continue              # absorbing: no outgoing transitions needed
        for reac, change, c in reactions:
            if _mass_action(x, reac, c) > 0:
                y = list(x)
                for s, d in change.items():
                    y[s] += d
                y = tuple(y)
                if y not in idx:
                    idx[y] = len(states)
                    states.append(y)
                    todo.append(y)
                    assert len(states) <= max_states
    n = len(states)
    Q = np.zeros((n, n))
    for i, x in enumerate(states):
        if phi2(x) or not phi1(x):
            continue
        for reac, change, c in reactions:
            a = _mass_action(x, reac, c)
            if a > 0:
                y = list(x)
                for s, d in change.items():
                    y[s] += d
                Q[i, idx[tuple(y)]] += a
                Q[i, i] -= a
    p0 = np.zeros(n)
    p0[0] = 1.0
    pT = p0 @ expm(Q * T)
    return sum(pT[i] for i, x in enumerate(states) if phi2(x)), n


def _cfg(species, x0, reactions):
    R = []
    for reac, change, c in reactions:
        prods = []
        # rebuild products from reactants + change
        tot = {s: st for s, st in reac}
        for s, d in change.items():
            tot[s] = tot.get(s, 0) + d
        for s, v in sorted(tot.items()):
            if v > 0:
                prods.append([s, v])
        R.append(dict(reactants=[list(r) for r in reac], products=prods, rate=c, hill=None))
    return dict(name="tiny", species=species, x0=x0, reactions=R)


def _check(cfg, formula, exact, n, seed):
    m = O.OracleModel(cfg)
    f = O.OracleFormula(formula, cfg["species"])
    c, v, e = O.run(m, f, seed, 0, n)
    z = normal_quantile(0.999)
    lo, hi = wilson_interval(c["n_true"] / n, n, z)
    lo2, hi2 = wilson_interval(exact, n, z)
    assert lo <= exact <= hi and lo2 <= c["n_true"] / n <= hi2, (formula, exact, c)


CASES = []
# two independent deaths A0 = B0 = 5 (36 states): (A > 1) U[0,T] (B == 0)
_deaths = ([([(0, 1)], {0: -1}, 1.0), ([(1, 1)], {1: -1}, 1.0)], ["A", "B"], [5, 5])
for T in [1.0, 2.0, 5.0]:
    CASES.append((_deaths, "(A > 1) U[0,%r] (B == 0)" % T, lambda x: x[0] > 1, lambda x: x[1] == 0, T))
# isomerisation A -> B (1), B -> A (0.5), A + B = 10 (11 states)
_iso = ([([(0, 1)], {0: -1, 1: +1}, 1.0), ([(1, 1)], {0: +1, 1: -1}, 0.5)], ["A", "B"], [10, 0])
for T in [1.0, 3.0]:
    CASES.append((_iso, "F[0,%r](A == 0)" % T, lambda x: True, lambda x: x[0] == 0, T))
# small Michaelis-Menten E0 = 2, S0 = 20, k1 = k2 = k3 = 0.1
_mm = ([([(0, 1), (1, 1)], {0: -1, 1: -1, 2: +1}, 0.1), ([(2, 1)], {0: +1, 1: +1, 2: -1}, 0.1),
        ([(2, 1)], {0: +1, 2: -1, 3: +1}, 0.1)], ["E", "S", "ES", "P"], [2, 20, 0, 0])
for T in [20.0, 50.0]:
    CASES.append((_mm, "F[0,%r](P >= 10)" % T, lambda x: True, lambda x: x[3] >= 10, T))
# dimerisation 2A -> B (homodimer, reading R8), B -> 2A
_dim = ([([(0, 2)], {0: -2, 1: +1}, 0.05), ([(1, 1)], {0: +2, 1: -1}, 0.3)], ["A", "B"], [20, 0])
CASES.append((_dim, "(A >= 4) U[0,2] (B >= 6)", lambda x: x[0] >= 4, lambda x: x[1] >= 6, 2.0))


@pytest.mark.parametrize("case", range(len(CASES)))
def test_until_vs_uniformisation(case):
    (reactions, species, x0), formula, phi1, phi2, T = CASES[case]
    exact, nstates = _until_probability(x0, reactions, phi1, phi2, T)
    assert nstates <= 200
    _check(_cfg(species, x0, reactions), formula, exact, 40_000, 1000 + case)


def test_globally_isomerisation():
    """G[0,T](A >= 2) = 1 - F[0,T](A < 2)."""
    reactions, species, x0 = _iso
    for i, T in enumerate([1.0, 3.0]):
        pf, _ = _until_probability(x0, reactions, lambda x: True, lambda x: x[0] < 2, T)
        _check(_cfg(species, x0, reactions), "G[0,%r](A >= 2)" % T, 1 - pf, 40_000, 2000 + i)


def test_known_survey_values():
    """The survey's independently computed values are reproduced by this brute force."""
    (reactions, species, x0) = _deaths
    p, _ = _until_probability(x0, reactions, lambda x: x[0] > 1, lambda x: x[1] == 0, 1.0)
    assert abs(p - 0.076536291957534) < 1e-12
    (reactions, species, x0) = _iso
    p, _ = _until_probability(x0, reactions, lambda x: True, lambda x: x[0] == 0, 3.0)
    assert abs(p - 0.092238797931607) < 1e-12
    # cross-check by the integral of f_tauB(t) P(A(t) >= 2): A, B independent deaths
    from scipy import integrate, stats

    def integrand(t):
        f = 5 * (1 - math.exp(-t)) ** 4 * math.exp(-t)
        return f * stats.binom.sf(1, 5, math.exp(-t))
    val, _ = integrate.quad(integrand, 0, 1.0, epsabs=1e-14)
    assert abs(val - 0.076536291957534) < 1e-10
