"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This module holds NO arithmetic of the method (no propensities, no SSA, no
monitor, no statistics): only model tables, formulas, seeds and the seeded
random-network generator of DESIGN.md §4.  Both sides import it;
neither side's arithmetic lives here.

A config is a dict:
  name, species [str], x0 [int], reactions [{reactants: [[s, st]..],
  products: [[s, st]..], rate: float, hill: None | {repressor, K, n}}],
  formula: str, t_max: float (0 = bounded), seed: int,
  sampling: {"mode": "fixed", "n": int} | {"mode": "wilson", "confidence", "half_width"}
The paper uses no public benchmark or dataset for this path (its own
cell-cycle model is out of scope for round 1); all inputs are synthetic.
"""
import copy
import json
import math
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
CONFIG_DIR = os.path.join(os.path.dirname(_HERE), "configs")


def _rx(reactants, products, rate, hill=None):
    return dict(reactants=[list(r) for r in reactants], products=[list(p) for p in products], rate=float(rate), hill=hill)


def c1():
    """C1 pure decay A -> 0, k = 1.0, A0 = 10; F[0,2](A == 0); 10^4 replicas, seed 1 (BASELINE.json configs[0])."""
    return dict(name="C1", species=["A"], x0=[10], reactions=[_rx([(0, 1)], [], 1.0)],
                formula="F[0,2.0](A == 0)", t_max=0.0, seed=1,
                sampling=dict(mode="fixed", n=10_000))


def c2():
    """C2 Michaelis-Menten E+S->ES (0.01), ES->E+S (0.1), ES->E+P (0.1); x0 = (100, 1000, 0, 0);
    F[0,50](P > 500); iterative Wilson 99 %, half-width 0.005 (configs[1]); seed 2."""
    E, S, ES, P = range(4)
    return dict(name="C2", species=["E", "S", "ES", "P"], x0=[100, 1000, 0, 0],
                reactions=[_rx([(E, 1), (S, 1)], [(ES, 1)], 0.01),
                           _rx([(ES, 1)], [(E, 1), (S, 1)], 0.1),
                           _rx([(ES, 1)], [(E, 1), (P, 1)], 0.1)],
                formula="F[0,50](P > 500)", t_max=0.0, seed=2,
                sampling=dict(mode="wilson", confidence=0.99, half_width=0.005))


def c3():
    """C3 three-gene repressilator (configs[2]); fixed parameter table of SURVEY §8(d) (reading G1):
    tx_i: 0 -> M_i, Hill c = 5.0, K = 50, n = 2, repressor P3 -> M1, P1 -> M2, P2 -> M3;
    tl_i: M_i -> M_i + P_i, c = 1.0;  md_i: M_i -> 0, c = 0.1;  pd_i: P_i -> 0, c = 0.1.
    x0 = (20, 0, 0, 0, 0, 0).  (G[0,100](P1 < 400)) U[0,200] (P2 > 300); 10^6 replicas; seed 3."""
    M1, M2, M3, P1, P2, P3 = range(6)
    Ms, Ps = [M1, M2, M3], [P1, P2, P3]
    rep = {0: P3, 1: P1, 2: P2}
    R = []
    for i in range(3):
        R.append(_rx([], [(Ms[i], 1)], 5.0, hill=dict(repressor=rep[i], K=50.0, n=2)))
    for i in range(3):
        R.append(_rx([(Ms[i], 1)], [(Ms[i], 1), (Ps[i], 1)], 1.0))
    for i in range(3):
        R.append(_rx([(Ms[i], 1)], [], 0.1))
    for i in range(3):
        R.append(_rx([(Ps[i], 1)], [], 0.1))
    return dict(name="C3", species=["M1", "M2", "M3", "P1", "P2", "P3"], x0=[20, 0, 0, 0, 0, 0],
                reactions=R, formula="(G[0,100](P1 < 400)) U[0,200] (P2 > 300)", t_max=0.0, seed=3,
                sampling=dict(mode="fixed", n=1_000_000))


def c3r(seed=3):
    """C3r parity-only stress input: same structure, rates log-uniform [0.01,10], K log-uniform [1,500],
    x0 uniform [0,500] (BASELINE.json configs[2] ranges; reading G1)."""
    cfg = c3()
    g = np.random.default_rng(seed)
    for r in cfg["reactions"]:
        r["rate"] = float(math.exp(g.uniform(math.log(0.01), math.log(10.0))))
        if r["hill"]:
            r["hill"]["K"] = float(math.exp(g.uniform(math.log(1.0), math.log(500.0))))
    cfg["x0"] = [int(v) for v in g.integers(0, 501, size=6)]
    cfg["name"] = "C3r"
    cfg["sampling"] = dict(mode="fixed", n=10_000)
    return cfg


def random_network(seed, n_species, n_reactions, redraw_null=True):
    """C4/C5 generator (reading G2/G3): for each reaction in order
    nr = integers(1,3), np = integers(0,3); nr reactant and np product draws of
    integers(n_species) with replacement, merged; c = exp(uniform(ln 1e-3, ln 1)).
    Then x0 = integers(10, 1001, size=n_species).  Null reactions (net change 0)
    are redrawn when redraw_null."""
    g = np.random.default_rng(seed)
    R = []
    n_redrawn = 0
    while len(R) < n_reactions:
        nr = int(g.integers(1, 3))
        npr = int(g.integers(0, 3))
        rs = [int(v) for v in g.integers(n_species, size=nr)]
        ps = [int(v) for v in g.integers(n_species, size=npr)]
        c = float(math.exp(g.uniform(math.log(1e-3), math.log(1.0))))
        rm, pm = {}, {}
        for s in rs:
            rm[s] = rm.get(s, 0) + 1
        for s in ps:
            pm[s] = pm.get(s, 0) + 1
        net = {s: pm.get(s, 0) - rm.get(s, 0) for s in set(rm) | set(pm)}
        if redraw_null and all(v == 0 for v in net.values()):
            n_redrawn += 1
            continue
        R.append(_rx(sorted(rm.items()), sorted(pm.items()), c))
    x0 = [int(v) for v in g.integers(10, 1001, size=n_species)]
    return dict(species=["S%d" % i for i in range(n_species)], x0=x0, reactions=R, null_redrawn=n_redrawn)


def swap_species(cfg, a, b):
    """Relabel species a <-> b (the S0/S1 pilot relabelling, reading G2)."""
    cfg = copy.deepcopy(cfg)
    perm = list(range(len(cfg["species"])))
    perm[a], perm[b] = b, a

    def m(s):
        return perm[s]
    cfg["x0"][a], cfg["x0"][b] = cfg["x0"][b], cfg["x0"][a]
    for r in cfg["reactions"]:
        r["reactants"] = sorted([[m(s), st] for s, st in r["reactants"]])
        r["products"] = sorted([[m(s), st] for s, st in r["products"]])
        if r["hill"]:
            r["hill"]["repressor"] = m(r["hill"]["repressor"])
    return cfg


def _load(name):
    path = os.path.join(CONFIG_DIR, name + ".json")
    with open(path) as fh:
        return json.load(fh)


def c4():
    """C4 50 x 200 random network (configs[3]); frozen by scripts/freeze_configs.py;
    F[0,10] G[0,1](S0 > S1); 10^7 replicas (over 8 GPUs); seed 4."""
    return _load("c4")


def c5():
    """C5 200 x 1000 scale network (configs[4]); frozen by scripts/freeze_configs.py;
    F[0,10] G[0,1](S0 > S1); iterative Wilson 99.9 %, half-width 1e-4; seed 5."""
    return _load("c5")


def bernoulli(p, seed=0):
    """A CTMC whose property is a Bernoulli(p) trial (Fig. 3 workload):
    one molecule A, decay A -> 0 at rate 1, F[0,T](A == 0) with T = -ln(1 - p), so
    P = 1 - e^{-T} = p (T = 0 for p = 0; T = 1000 for p = 1, e^{-1000} = 0 in binary64).
    Each replica applies at most one event."""
    T = 0.0 if p <= 0.0 else (1000.0 if p >= 1.0 else -math.log1p(-p))
    return dict(name="BERN(%g)" % p, species=["A"], x0=[1], reactions=[_rx([(0, 1)], [], 1.0)],
                formula="F[0,%r](A == 0)" % T, t_max=0.0, seed=seed,
                sampling=dict(mode="wilson", confidence=0.99, half_width=0.025))


def explicit_demo():
    """Explicit (non-mass-action) propensities (NEXT-3, Table 2 P:513-538 style):
    repressed production 0 -> S at 20/(1 + I/10), Michaelis-Menten conversion S -> P at
    10 S/(5 + S), mass-action P -> 0 (0.1) and P -> P + I (0.05), explicit I -> 0 at 0.2 I;
    x0 = 0; F[0,20](P > 80) (p ~ 0.61, ~540 events per replica); seed 12."""
    R = [dict(_rx([], [(0, 1)], 1.0), rate_expr="20/(1+I/10)"),
         dict(_rx([(0, 1)], [(1, 1)], 1.0), rate_expr="10*S/(5+S)"),
         _rx([(1, 1)], [], 0.1), _rx([(1, 1)], [(1, 1), (2, 1)], 0.05),
         dict(_rx([(2, 1)], [], 1.0), rate_expr="0.2*I")]
    return dict(name="EXPL", species=["S", "P", "I"], x0=[0, 0, 0], reactions=R, formula="F[0,20](P > 80)",
                t_max=0.0, seed=12, sampling=dict(mode="fixed", n=100_000))


CELL_CYCLE_FORMULAS = ["(a <= 4) U[0,1000] (y >= 5)", "(a <= 20) U[0,1000] (y >= 35)",
                       "(a <= 40) U[0,1000] (y >= 40 & y <= 42)"]      # Table 3 rows


def cell_cycle(formula=CELL_CYCLE_FORMULAS[0], seed=21):
    """Best-effort budding-yeast cell-cycle toy model (Table 1 P:475-511,
    Table 2).  Species x (Cdk/CycB), y (active APC/Cdh1),
    y_in (inactive APC/Cdh1), a (Cdc20).  Counts n = c / alpha (alpha = 0.00236012,
    Omega = 1/alpha ~ 424); propensities in counts per unit time:
      R1x 0 -> x              k1 / alpha
      R2x x -> 0              k2' x
      R3x x + y -> y          k2'' alpha x y
      R1y y_in -> y           k3' y_in / (J3 + alpha y_in)
      R2y y_in + a -> y + a   k3'' alpha a y_in / (J3 + alpha y_in)   (Table 2's k3-triple-prime)
      R3y x + y -> x + y_in   k4 m alpha x y / (J4 + alpha y)         (Table 2's k3-star)
      R1a 0 -> a              k5' / alpha
      R2a x -> x + a          k5'' m x / J5                           (Table 2's k5-star)
      R3a a -> 0              k6 a
    with Table 2's constants.  The paper gives no initial state; x0 = (212, 0, 424, 0)
    (CycB at half of Omega, APC all inactive, no Cdc20: "low level of activated APC, high
    Cdk/CycB, low Cdc20") is an assumption, so Table 3's probabilities are not
    reproduced (reading G4)."""
    alpha = 0.00236012
    k1, k2p, k2pp, k3p, k3pp, k4, J3, J4 = 0.04, 0.04, 1.0, 1.0, 10.0, 35.0, 0.04, 0.04
    k5p, k5pp, k6, J5, m = 0.005, 0.2, 0.1, 0.3, 0.8
    A = repr(alpha)
    R = [dict(_rx([], [(0, 1)], 1.0), rate_expr=repr(k1 / alpha)),
         _rx([(0, 1)], [], k2p),
         dict(_rx([(0, 1), (1, 1)], [(1, 1)], 1.0), rate_expr="%r*x*y" % (k2pp * alpha)),
         dict(_rx([(2, 1)], [(1, 1)], 1.0), rate_expr="%r*y_in/(%r+%s*y_in)" % (k3p, J3, A)),
         dict(_rx([(2, 1), (3, 1)], [(1, 1), (3, 1)], 1.0), rate_expr="%r*%s*a*y_in/(%r+%s*y_in)" % (k3pp, A, J3, A)),
         dict(_rx([(0, 1), (1, 1)], [(0, 1), (2, 1)], 1.0), rate_expr="%r*%r*%s*x*y/(%r+%s*y)" % (k4, m, A, J4, A)),
         dict(_rx([], [(3, 1)], 1.0), rate_expr=repr(k5p / alpha)),
         dict(_rx([(0, 1)], [(0, 1), (3, 1)], 1.0), rate_expr="%r*%r*x/%r" % (k5pp, m, J5)),
         _rx([(3, 1)], [], k6)]
    return dict(name="CC", species=["x", "y", "y_in", "a"], x0=[212, 0, 424, 0], reactions=R, formula=formula,
                t_max=0.0, seed=seed, sampling=dict(mode="wilson", confidence=0.99, half_width=0.025))


CONFIGS = dict(C1=c1, C2=c2, C3=c3, C4=c4, C5=c5, EXPL=explicit_demo, CC=cell_cycle)


def get(name):
    return CONFIGS[name.upper()]()


def with_sampling(cfg, **kw):
    cfg = copy.deepcopy(cfg)
    cfg["sampling"] = dict(kw)
    return cfg
