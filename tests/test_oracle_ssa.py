"""Pins for the oracle's SSA + on-the-fly checker against
closed forms and exact event counts.  No GPU.

Each estimate check is two-sided: p_exact in WI(p_hat, n) and
p_hat in WI(p_exact, n), at a fixed seed chosen before the first run."""
import math

import numpy as np
import pytest
from scipy import stats

import workloads
from oracle import normal_quantile, wilson_interval
from oracle import oracle as O


def _model(species, x0, reactions):
    return dict(name="t", species=species, x0=x0, reactions=[
        dict(reactants=[list(a) for a in r[0]], products=[list(b) for b in r[1]], rate=float(r[2]), hill=None)
        for r in reactions])


def _estimate(cfg, formula, n, seed, t_max=0.0, mode="stream"):
    m = O.OracleModel(cfg)
    f = O.OracleFormula(formula, cfg["species"], t_max)
    c, v, e = O.run(m, f, seed, 0, n, mode)
    assert c["errors"] == 0
    return c, v, e


def _contains(p_exact, k, n, conf=0.999):
    z = normal_quantile(conf)
    lo, hi = wilson_interval(k / n, n, z)
    lo2, hi2 = wilson_interval(p_exact, n, z)
    return lo <= p_exact <= hi and lo2 <= k / n <= hi2


def test_c1_closed_form():
    """C1 (configs[0]): P(F[0,2](A==0)) = (1 - e^-2)^10 for pure decay, k = 1, A0 = 10."""
    cfg = workloads.c1()
    exact = (1 - math.exp(-2.0)) ** 10
    assert abs(exact - 0.2336024409784545) < 1e-15
    c, v, e = _estimate(cfg, cfg["formula"], 10_000, cfg["seed"])
    assert _contains(exact, c["n_true"], 10_000, conf=0.99)
    c, v, e = _estimate(cfg, cfg["formula"], 200_000, 11)
    assert _contains(exact, c["n_true"], 200_000)


def test_c1_worked_example():
    """Bit-level worked example: seed 1, trajectories 0..2."""
    cfg = workloads.c1()
    m = O.OracleModel(cfg)
    tr = m.simulate(1, 0, 2.0)
    assert tr["t"][1] == 0.01162426530573836 and tr["t"][2] == 0.055790878029171945
    assert tr["t"][3] == 0.23038373651755334
    assert len(tr["t"]) - 1 == 9 and tr["t"][-1] + tr["tau"][-1] == 2.9142962961493746
    c, v, e = _estimate(cfg, cfg["formula"], 3, 1)
    assert list(v) == [0, 0, 1] and list(e) == [9, 7, 10]


def test_pure_death_two():
    """F[0,1](x==0), X0 = 2, k = 1 -> 1 - 2e^-1 + e^-2."""
    cfg = _model(["x"], [2], [([(0, 1)], [], 1.0)])
    exact = 1 - 2 * math.exp(-1) + math.exp(-2)
    c, v, e = _estimate(cfg, "F[0,1](x == 0)", 100_000, 21)
    assert _contains(exact, c["n_true"], 100_000)


def test_pure_death_general_decay():
    """(1 - e^{-kT})^{A0} for several (A0, k, T)."""
    for A0, k, T, seed in [(1, 2.0, 0.5, 31), (5, 0.5, 3.0, 32), (20, 1.0, 4.0, 33)]:
        cfg = _model(["A"], [A0], [([(0, 1)], [], k)])
        exact = (1 - math.exp(-k * T)) ** A0
        c, v, e = _estimate(cfg, "F[0,%r](A == 0)" % T, 50_000, seed)
        assert _contains(exact, c["n_true"], 50_000)


@pytest.mark.parametrize("n0", list(range(1, 51)))
def test_early_termination_exact_events(n0):
    """F(x == 0) on pure death from n0 applies exactly n0 events (trace stops on resolution)."""
    cfg = _model(["x"], [n0], [([(0, 1)], [], 1.0)])
    c, v, e = _estimate(cfg, "F(x == 0)", 20, 40 + n0, t_max=1e9)
    assert (v == 1).all() and (e == n0).all()


def test_pure_death_mean():
    """X0 = 100, k = 1: E[X(1)] = 100 e^-1 within 3 standard errors."""
    cfg = _model(["x"], [100], [([(0, 1)], [], 1.0)])
    m = O.OracleModel(cfg)
    xs = []
    for i in range(4000):
        tr = m.simulate(51, i, 1.0)
        xs.append(tr["x"][-1, 0])        # state occupied at t = 1 (last entry <= 1)
    xs = np.array(xs, float)
    mean = 100 * math.exp(-1)
    se = math.sqrt(100 * math.exp(-1) * (1 - math.exp(-1)) / len(xs))
    assert abs(xs.mean() - mean) < 3 * se


def test_tau_exponential():
    """single channel with a = 2: tau ~ Exp(2) (Eq. 2a)."""
    cfg = _model(["A"], [0], [([], [(0, 1)], 2.0)])
    m = O.OracleModel(cfg)
    taus = np.array([m.simulate(61, i, 1e-12, cap=4)["tau"][0] for i in range(20000)])
    se = 0.5 / math.sqrt(len(taus))
    assert abs(taus.mean() - 0.5) < 3 * se
    assert stats.kstest(taus, "expon", args=(0, 0.5)).pvalue > 1e-3


def test_selection_frequencies():
    """two channels a = (1, 3): P(j) = (0.25, 0.75) (Eq. 2b)."""
    cfg = _model(["A", "B"], [0, 0], [([], [(0, 1)], 1.0), ([], [(1, 1)], 3.0)])
    m = O.OracleModel(cfg)
    first = []
    for i in range(20000):
        tr = m.simulate(62, i, 1e9, cap=3)
        first.append(int(tr["x"][1, 1] == 1))
    p = np.mean(first)
    assert abs(p - 0.75) < 3 * math.sqrt(0.75 * 0.25 / len(first))


def test_pure_birth_poisson():
    """0 -> A (lambda = 2): F[0,3](A >= 8) = P(Poisson(6) >= 8)."""
    cfg = _model(["A"], [0], [([], [(0, 1)], 2.0)])
    exact = float(stats.poisson.sf(7, 6.0))
    c, v, e = _estimate(cfg, "F[0,3](A >= 8)", 50_000, 71)
    assert _contains(exact, c["n_true"], 50_000)


def test_immigration_death():
    """0 -> A (5), A -> 0 (1) from 0: A(t) ~ Poisson(5 (1 - e^-t)); stationary Poisson(5)."""
    cfg = _model(["A"], [0], [([], [(0, 1)], 5.0), ([(0, 1)], [], 1.0)])
    m = O.OracleModel(cfg)
    a2, a30 = [], []
    for i in range(6000):
        tr = m.simulate(81, i, 30.0)
        t, x = tr["t"], tr["x"][:, 0]
        a2.append(x[np.searchsorted(t, 2.0, side="right") - 1])
        a30.append(x[-1])
    a2 = np.array(a2)
    lam2 = 5 * (1 - math.exp(-2))
    k = int((a2 >= 5).sum())
    assert _contains(float(stats.poisson.sf(4, lam2)), k, len(a2))
    a30 = np.array(a30)
    # chi-square goodness of fit to Poisson(5) on bins 0..12+
    obs = np.array([(a30 == j).sum() for j in range(12)] + [(a30 >= 12).sum()])
    pr = np.array([stats.poisson.pmf(j, 5) for j in range(12)] + [stats.poisson.sf(11, 5)])
    chi = ((obs - pr * len(a30)) ** 2 / (pr * len(a30))).sum()
    assert stats.chi2.sf(chi, len(obs) - 1) > 1e-3


def test_monotone_death_nested_FG():
    """T5 with absorption: A0 = 10, k = 1: F[0,1] G[0,0.5](A <= 3) = P(Bin(10, 1 - e^-1) >= 7)."""
    cfg = _model(["A"], [10], [([(0, 1)], [], 1.0)])
    exact = float(stats.binom.sf(6, 10, 1 - math.exp(-1)))
    c, v, e = _estimate(cfg, "F[0,1] G[0,0.5](A <= 3)", 50_000, 91)
    assert _contains(exact, c["n_true"], 50_000)
    c2, v2, e2 = _estimate(cfg, "F[0,1] G[0,0.5](A <= 3)", 3000, 91, mode="literal")
    assert (v[:3000] == v2).all()


def test_homodimer_propensity():
    """Reading R8: 2A -> 0 has a = c x(x-1)/2; A + B -> C has c x y."""
    cfg = _model(["A", "B", "C"], [5, 3, 4], [([(0, 2)], [], 2.0), ([(0, 1), (1, 1)], [(2, 1)], 0.5)])
    m = O.OracleModel(cfg)
    assert m.propensity(0, [5, 3, 4]) == 20.0
    assert m.propensity(1, [3, 4, 0]) == 6.0
    assert m.propensity(0, [1, 3, 4]) == 0.0          # guard: below stoichiometry
    assert m.propensity(1, [0, 7, 0]) == 0.0


def test_hill_propensity():
    """Reading R9: c h / (1 + (x_r/K)^n), q^n a left-to-right product."""
    cfg = workloads.c3()
    m = O.OracleModel(cfg)
    x = [20, 0, 0, 7, 0, 30]
    assert m.propensity(0, x) == 5.0 / (1.0 + (30 / 50.0) * (30 / 50.0))
    assert m.propensity(1, x) == 5.0 / (1.0 + (7 / 50.0) * (7 / 50.0))
    assert m.propensity(3, x) == 1.0 * 20


def test_streaming_equals_literal_on_models():
    """On-the-fly verdicts == literal |= on the full trace for C1, C2 and C3."""
    for cfg, n in [(workloads.c1(), 2000), (workloads.c2(), 300), (workloads.c3(), 3), (workloads.c3r(), 60)]:
        c1, v1, e1 = _estimate(cfg, cfg["formula"], n, cfg["seed"], mode="stream")
        c2, v2, e2 = _estimate(cfg, cfg["formula"], n, cfg["seed"], mode="literal")
        assert (v1 == v2).all(), cfg["name"]
        assert (e1 <= e2).all()          # on-the-fly never generates more events


@pytest.mark.parametrize("atom", ["A*A >= 64", "A/2 >= 4", "sqrt(A) > 2.8", "pow(A, 3) >= 512", "min(A, 100) >= 7.5",
                                  "max(A, 0.5) > 7.9", "abs(-A) >= 8", "8.0 <= A", "(A - 0.5) * 2 >= 15"])
def test_general_val_atoms_pure_birth(atom):
    """General val atoms (val ~ val, func, Int, Real) that are equivalent to A >= 8 on
    integer counts give the pure-birth closed form P(Poisson(6) >= 8) -- and, on the same
    Philox streams, exactly the replicas of the integer atom (binary64 path vs int64 path)."""
    cfg = _model(["A"], [0], [([], [(0, 1)], 2.0)])
    exact = float(stats.poisson.sf(7, 6.0))
    c, v, e = _estimate(cfg, "F[0,3](%s)" % atom, 20_000, 71)
    ci, vi, ei = _estimate(cfg, "F[0,3](A >= 8)", 20_000, 71)
    assert (v == vi).all() and (e == ei).all()
    assert _contains(exact, c["n_true"], 20_000)


def test_general_val_atom_values():
    """Hand states for the paper's example atom X1 < sqrt(X2) and the binary64
    corner cases: division by zero gives inf (X2 / X1 > 1e300 true at X1 = 0), 0/0 is NaN
    (every comparison false, != true)."""
    cfg = _model(["X1", "X2"], [0, 0], [([], [(0, 1)], 1.0)])
    m = O.OracleModel(cfg)

    def holds(f, x1, x2):
        fo = O.OracleFormula(f, cfg["species"])
        t = np.array([0.0])
        return fo.check_literal(t, np.array([]), np.array([[x1, x2]]), True) == 1
    assert holds("X1 < sqrt(X2)", 3, 10) and not holds("X1 < sqrt(X2)", 4, 16) and holds("X1 <= sqrt(X2)", 4, 16)
    assert holds("X2 / X1 > 1e300", 0, 5) and not holds("X2 / X1 > 1e300", 1, 5)
    assert not holds("X1 / X2 >= 0", 0, 0) and not holds("X1 / X2 < 0", 0, 0) and holds("X1 / X2 != 0", 0, 0)
    assert holds("pow(X1, 0) == 1", 7, 0) and holds("min(X1, X2) == 2", 2, 9) and holds("max(X1, X2) == 9", 2, 9)
    assert holds("X2 / 3 == 3", 0, 9) and not holds("X2 / 3 == 3", 0, 10)
    del m
