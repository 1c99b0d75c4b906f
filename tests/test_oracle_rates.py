"""Pins for the oracle's explicit (non-mass-action) rate expressions (Table 2,
P:513-538; explicit propensities, the guard still applies).
No GPU.

* an explicit constant immigration rate reproduces the immigration-death closed form;
* an explicit Michaelis-Menten degradation rate Vmax*S/(Km+S) reproduces the
  first-passage probability of the pure-death chain with those rates, solved by the
  matrix exponential (brute force, 21 states);
* an explicit rate that equals the mass-action law on exactly representable values
  reproduces the mass-action trajectories replica for replica (same Philox streams);
* the guard: an explicit rate on a reaction whose reactant is absent is 0;
  a negative value is a bad propensity (the replica ends in error);
* parse errors name the position."""
import math

import numpy as np
import pytest
from scipy.linalg import expm

import workloads
from oracle import normal_quantile, wilson_interval
from oracle import oracle as O

rx = workloads._rx


def _cfg(species, x0, reactions, formula, seed=1):
    return dict(name="rates", species=species, x0=x0, reactions=reactions, formula=formula, t_max=0.0, seed=seed,
                sampling=dict(mode="fixed", n=0))


def _inside(p_exact, k, n, conf=0.999):
    lo, hi = wilson_interval(k / n, n, normal_quantile(conf))
    return lo <= p_exact <= hi


def test_explicit_constant_immigration_is_poisson():
    # 0 -> A at the explicit rate "5", A -> 0 mass action mu = 1, from A = 0:
    # A(2) ~ Poisson(5 (1 - e^-2)), P(A(2) >= 5) = 0.434066218452784.
    cfg = _cfg(["A"], [0], [dict(rx([], [(0, 1)], 1.0), rate_expr="5"), rx([(0, 1)], [], 1.0)],
               "F[0,2](A >= 5)")
    m = O.OracleModel(cfg)                      # A(2) read off the sampled trace
    lam = 5 * (1 - math.exp(-2))
    exact = 1 - sum(math.exp(-lam) * lam ** i / math.factorial(i) for i in range(5))
    assert abs(exact - 0.434066218452784) < 1e-12
    n, k = 4000, 0
    for i in range(n):
        tr = m.simulate(7, i, 2.0)
        j = np.searchsorted(tr["t"], 2.0, side="right") - 1
        k += int(tr["x"][j][0] >= 5)
    assert _inside(exact, k, n)


def test_explicit_michaelis_menten_degradation_vs_matrix_exponential():
    vmax, km, s0, T = 10.0, 5.0, 20, 2.5
    cfg = _cfg(["S"], [s0], [dict(rx([(0, 1)], [], 1.0), rate_expr="10*S/(5+S)")], "F[0,2.5](S == 0)", seed=3)
    Q = np.zeros((s0 + 1, s0 + 1))
    for s in range(1, s0 + 1):
        mu = vmax * s / (km + s)
        Q[s, s] = -mu
        Q[s, s - 1] = mu
    p0 = np.zeros(s0 + 1)
    p0[s0] = 1.0
    exact = float((p0 @ expm(Q * T))[0])
    assert 0.05 < exact < 0.95
    m = O.OracleModel(cfg)
    f = O.OracleFormula(cfg["formula"], cfg["species"])
    n = 20000
    c, v, e = O.run(m, f, cfg["seed"], 0, n)
    assert c["errors"] == 0
    assert _inside(exact, c["n_true"], n)
    assert m.propensity(0, [7]) == 10 * 7 / (5 + 7)
    assert m.propensity(0, [0]) == 0.0                  # guard: reactant absent


def test_explicit_equal_to_mass_action_replays_the_trajectories():
    # 0.0078125*A*B (= 2^-7 A B) evaluated as (c*A)*B in binary64 equals the mass-action
    # c*(A*B) exactly: identical propensities, identical Philox streams, identical replicas.
    base = [rx([(0, 1), (1, 1)], [(2, 1)], 0.0078125), rx([(2, 1)], [(0, 1), (1, 1)], 0.5)]
    expl = [dict(base[0], rate_expr="0.0078125*A*B"), dict(base[1], rate_expr="C*0.5")]
    cfg_m = _cfg(["A", "B", "C"], [30, 20, 0], base, "F[0,2](C >= 6)", seed=9)
    cfg_e = dict(cfg_m, reactions=expl)
    om, oe = O.OracleModel(cfg_m), O.OracleModel(cfg_e)
    f = O.OracleFormula(cfg_m["formula"], cfg_m["species"])
    cm, vm, em = O.run(om, f, 9, 0, 3000)
    ce, ve, ee = O.run(oe, f, 9, 0, 3000)
    assert (vm == ve).all() and (em == ee).all()
    assert 0 < vm.mean() < 1


def test_negative_explicit_rate_is_an_error():
    cfg = _cfg(["A"], [3], [dict(rx([(0, 1)], [], 1.0), rate_expr="1 - A")], "F[0,1](A == 0)")
    m = O.OracleModel(cfg)
    assert math.isnan(m.propensity(0, [3]))
    f = O.OracleFormula(cfg["formula"], cfg["species"])
    c, v, e = O.run(m, f, 1, 0, 10)
    assert c["errors"] == 10


@pytest.mark.parametrize("expr,pos", [("2*", 2), ("(A", 2), ("A $ 2", 2), ("Z", 1), ("2 A", 2)])
def test_rate_parse_errors(expr, pos):
    cfg = _cfg(["A"], [3], [dict(rx([(0, 1)], [], 1.0), rate_expr=expr)], "F[0,1](A == 0)")
    with pytest.raises(ValueError, match="rate expression"):
        O.OracleModel(cfg)
