"""Pins for the oracle's checkers: the literal |= against
hand traces, duality and monotonicity, and the streaming monitor against the
literal |= on random traces.  No GPU."""
import numpy as np
import pytest

from oracle import oracle as O

NAMES = ["A", "B", "C"]
F_, T_, U_ = 0, 1, 2


def trace(times, states, absorbed, tail_tau=None):
    t = np.asarray(times, float)
    tau = list(np.diff(t))
    if not absorbed:
        tau.append(tail_tau if tail_tau is not None else 1e9)
    return t, np.asarray(tau, float), np.asarray(states, np.int64), absorbed


def lit(text, tr, t_max=0.0):
    return O.OracleFormula(text, NAMES, t_max).check_literal(*tr)


def test_spec_hand_traces():
    # atom at sigma[0]
    tr = trace([0.0], [[7, 0, 0]], True)
    assert lit("A >= 5", tr) == T_
    # (a<=4) U (y>=5) on a:(0,3,5), y:(0,2,6): witness k=2, a<=4 at j=0,1 -> true
    tr = trace([0.0, 0.1, 0.2], [[0, 0, 0], [3, 2, 0], [5, 6, 0]], True)
    assert lit("(A <= 4) U (B >= 5)", tr) == T_
    # lower bound > 0 and witness only at elapsed 0 -> false
    tr = trace([0.0, 0.2], [[0, 9, 0], [0, 0, 0]], True)
    assert lit("true U[0.5,1.0] (B >= 5)", tr) == F_
    # X: successor must exist; delta(sigma,0) in I
    tr = trace([0.0, 0.3], [[0, 0, 0], [1, 0, 0]], True)
    assert lit("X[0,0.5](A == 1)", tr) == T_
    assert lit("X[0,0.2](A == 1)", tr) == F_
    assert lit("X[0,1](A == 1)", trace([0.0], [[0, 0, 0]], True)) == F_
    # unresolved at the end of a non-absorbed trace -> unknown (reading R4)
    tr = trace([0.0, 0.3], [[0, 0, 0], [1, 0, 0]], False, tail_tau=0.1)
    assert lit("F[0,1](A == 5)", tr) == U_
    assert lit("F[0,0.35](A == 5)", tr) == F_
    # absorbed: G holds on the remaining (infinite) sojourn (reading R7)
    tr = trace([0.0, 0.3], [[1, 0, 0], [1, 0, 0]], True)
    assert lit("G[0,10](A == 1)", tr) == T_


def test_index_semantics_lower_bound():
    """Reading R1: with a > 0 the state occupied at time a but entered earlier is not a witness."""
    tr = trace([0.0, 0.5, 2.0], [[0, 0, 0], [3, 0, 0], [0, 0, 0]], True)
    assert lit("F[1,1.5](A == 3)", tr) == F_
    assert lit("F[0.5,1.5](A == 3)", tr) == T_
    assert lit("F(0.5,1.5](A == 3)", tr) == F_       # open lower bound (reading R6)


def _rand_trace(g, n_species=3, max_len=40, vmax=5):
    n = int(g.integers(1, max_len))
    tau = g.exponential(0.25, size=n)
    t = np.concatenate([[0.0], np.cumsum(tau[:-1])]) if n > 1 else np.array([0.0])
    # build t from tau exactly as the SSA does: t_{k+1} = t_k + tau_k
    t = [0.0]
    for k in range(n - 1):
        t.append(t[-1] + tau[k])
    t = np.array(t)
    x = np.zeros((n, n_species), np.int64)
    x[0] = g.integers(0, vmax + 1, size=n_species)
    for k in range(1, n):
        x[k] = np.clip(x[k - 1] + g.integers(-1, 2, size=n_species), 0, vmax)
    absorbed = bool(g.random() < 0.3)
    if absorbed:
        return t, tau[:n - 1].copy(), x, True
    return t, tau[:n].copy(), x, False


def _bounds(g):
    a = float(g.choice([0.0, 0.0, 0.5, 1.0, 2.0]))
    b = a + float(g.choice([0.3, 1.0, 2.0, 4.0]))
    return a, b


def _formulas(g):
    a, b = _bounds(g)
    c1, c2 = int(g.integers(0, 5)), int(g.integers(0, 5))
    lo = "(" if g.random() < 0.2 else "["
    hi = ")" if g.random() < 0.2 else "]"
    I = "%s%r,%r%s" % (lo, a, b, hi)
    p, q = float(g.choice([0.5, 1.0, 2.0])), float(g.choice([0.2, 0.5, 1.0]))
    return {
        "T1": "F%s(A > %d)" % (I, c1),
        "T2": "G%s(A > %d)" % (I, c1),
        "T3": "(A > %d) U%s (B > %d)" % (c1, I, c2),
        "T4": "X%s(A > %d | B == %d)" % (I, c1, c2),
        "T5": "F[0,%r] G[0,%r] (A > B)" % (p, q),
        "T6": "G[0,%r] F[0,%r] (A > B)" % (p, q),
        "T7": "(G[0,%r](A < %d)) U[0,%r] (B > %d)" % (q, c1 + 1, p, c2),
        "root": "(A > %d) & (F%s(B > %d) | !G[0,%r](C != %d))" % (c1 - 1, I, c2, b, c1),
    }


@pytest.mark.parametrize("shape", ["T1", "T2", "T3", "T4", "T5", "T6", "T7", "root"])
def test_streaming_equals_literal_random(shape):
    g = np.random.default_rng(["T1", "T2", "T3", "T4", "T5", "T6", "T7", "root"].index(shape) + 17)
    agree = 0
    n = 10_000
    for _ in range(n):
        text = _formulas(g)[shape]
        tr = _rand_trace(g)
        f = O.OracleFormula(text, NAMES)
        lv = f.check_literal(*tr)
        sv, at = f.check_streaming(*tr)
        assert lv == sv, (text, tr, lv, sv)
        agree += 1
    assert agree == n


def test_duality_and_monotonicity():
    g = np.random.default_rng(99)
    for _ in range(3000):
        tr = _rand_trace(g)
        a, b = _bounds(g)
        c = int(g.integers(0, 5))
        G = lit("G[%r,%r](A > %d)" % (a, b, c), tr)
        nFn = lit("!F[%r,%r](!(A > %d))" % (a, b, c), tr)
        assert G == nFn
        f1 = lit("F[0,%r](A == %d)" % (b, c), tr)
        f2 = lit("F[0,%r](A == %d)" % (b + 1.0, c), tr)
        if f1 == T_:
            assert f2 == T_


def test_prefix_optimality_F():
    """on F(atom) the streaming monitor stops at the FIRST satisfying entry."""
    g = np.random.default_rng(5)
    for _ in range(2000):
        t, tau, x, ab = _rand_trace(g)
        f = O.OracleFormula("F[0,1000](A == 3)", NAMES)
        v, at = f.check_streaming(t, tau, x, ab)
        hits = np.nonzero(x[:, 0] == 3)[0]
        if len(hits):
            assert v == T_ and at == hits[0]


def test_unsupported_outside_fragment():
    f = O.OracleFormula("F[0,1](G[0.5,1](A > 1))", NAMES)
    assert not f.streamable
    assert O.OracleFormula("F[0,1] G[0,1] (A > 1)", NAMES).streamable


def test_parse_errors():
    for bad in ["F[0,1](Z > 1)", "F[0,1](A >)", "(A > 1", "F[2,1](A > 1)", "sqr(A) > 1", "pow(A, 1.5) > 1"]:
        with pytest.raises(ValueError):
            O.OracleFormula(bad, NAMES)


@pytest.mark.parametrize("formula", ["F[0,60](A >= 150)", "G[0,60](A <= 140)", "(A < 120) U[0,40] (A >= 130)",
                                     "F[0,20] G[0,2](A >= 90)", "X[0,1](A == 3) | F[0,50](A >= 160)"])
def test_literal_first_decision_pinned_to_streaming(formula):
    """On-the-fly halting: literal mode's event count is the first index at which
    the observed prefix decides |= (found from the stored trace).  For streamable formulas the
    streaming monitor -- an independently written automaton that stops the moment it decides --
    gives that index directly, so the two event counts must be EQUAL replica by replica (and
    the verdicts too).  A literal evaluator that ran to the horizon, or stopped one entry early
    or late, fails this."""
    rx = __import__("workloads")._rx
    cfg = dict(name="imd", species=["A"], x0=[0], reactions=[rx([], [(0, 1)], 10.0), rx([(0, 1)], [], 0.05)],
               formula=formula, t_max=0.0, seed=3, sampling=dict(mode="fixed", n=0))
    m = O.OracleModel(cfg)
    f = O.OracleFormula(formula, cfg["species"])
    assert f.streamable
    cs, vs, es = O.run(m, f, 3, 0, 300, mode="stream")
    cl, vl, el = O.run(m, f, 3, 0, 300, mode="literal")
    assert (vs == vl).all()
    assert (es == el).all(), [(i, es[i], el[i]) for i in np.nonzero(es != el)[0][:5]]
    H = f.reach
    early = sum(1 for i in range(300) if el[i] < len(m.simulate(3, i, H)["t"]) - 1)
    assert early > 30                        # replicas do stop before the horizon
