"""Variant 5 (ssa_delta.cuh): exact fixed-point group sums maintained by dependency deltas,
no stored propensities (reading R26).  Replica for replica against the oracle: the C4/C5
fixtures (tests/golden, written from oracle/ only) at every tile width, the edge cases
(absorbing start, event cap, count overflow, counts ~1e8 whose products exceed 2^53) and
random mass-action networks of the C4/C5 recipe."""
import json
import os

import numpy as np
import pytest

import workloads
from oracle import oracle as O

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _pair(smc, cfg, variant=5):
    m = smc.Model.from_config(cfg)
    m.set_variant(variant)
    p = smc.Property(m, cfg["formula"], t_max=cfg.get("t_max", 0.0))
    return m, p


def _fixture(name):
    return json.load(open(os.path.join(GOLDEN, "%s_oracle.json" % name.lower())))


@pytest.mark.parametrize("width", ["8", "16", "32"])
@pytest.mark.parametrize("name", ["C4", "C5"])
def test_fixture_every_tile_width(smc, name, width, monkeypatch):
    monkeypatch.setenv("SMC_TILE_WIDTH", width)
    fx = _fixture(name)
    cfg = workloads.get(name)
    m, p = _pair(smc, cfg)
    n = fx["n"] if name == "C5" else 1000
    v, e = m.run_verdicts(p, 0, n, fx["seed"])
    v, e = v.cpu().numpy(), e.cpu().numpy()
    assert m.last_launch(p)["variant"] == 5
    bad = np.nonzero((v != np.array(fx["verdicts"][:n])) | (e != np.array(fx["events"][:n])))[0]
    assert len(bad) == 0, (name, width, bad[:10])


def test_edge_cases(smc):
    """Absorbing start, event cap, count overflow (R17) and counts ~1e8 (h ~ 2e16 > 2^53: the
    fixed-point h is the exact int64 product, the in-group law the oracle's binary64 value)."""
    z = dict(workloads.c1(), x0=[0])
    m0, p0 = _pair(smc, z)
    assert m0.run(p0, 1000, 3) == dict(n_true=1000, n_false=0, events=0, errors=0)
    m2, p2 = _pair(smc, workloads.c2())
    m2.set_event_cap(5)
    c = m2.run(p2, 100, 2)
    assert c["errors"] == 100 and c["events"] == 500
    big = dict(species=["A"], x0=[2147483640], reactions=[dict(reactants=[], products=[[0, 2]], rate=1.0, hill=None)],
               formula="F[0,100](A < 0)")
    m3, p3 = _pair(smc, big)
    c = m3.run(p3, 50, 1)
    assert c["errors"] == 50 and c["events"] == 50 * 3
    rx = workloads._rx
    huge = dict(name="huge", species=["A", "B", "C"], x0=[200000000, 100000000, 0],
                reactions=[rx([(0, 1), (1, 1)], [(2, 1)], 3e-16), rx([(0, 2)], [(1, 1)], 1e-16),
                           rx([(2, 1)], [], 1e-9), rx([], [(0, 1)], 1e-9)],   # rates within 2^24 (R26)
                formula="F[0,3](C >= 12)", t_max=0.0, seed=8, sampling=dict(mode="fixed", n=400))
    m4, p4 = _pair(smc, huge)
    v, e = m4.run_verdicts(p4, 0, 400, 8)
    oc, ov, oe = O.run(O.OracleModel(huge), O.OracleFormula(huge["formula"], huge["species"]), 8, 0, 400)
    assert int(((v.cpu().numpy() != ov) | (e.cpu().numpy() != oe)).sum()) == 0


def test_small_models_and_templates(smc):
    """The delta kernel also runs small mass-action models (C1, C2) and every template."""
    for cfg, f in [(workloads.c1(), None), (workloads.c2(), None), (workloads.c2(), "G[0,40](P < 480)"),
                   (workloads.c2(), "(ES < 60) U[0,30] (P > 300)"), (workloads.c2(), "X[0,0.01](S < 1000)"),
                   (workloads.c2(), "G[0,30] F[0,5](ES > 40)")]:
        if f:
            cfg = dict(cfg, formula=f)
        m, p = _pair(smc, cfg)
        n = 3000
        v, e = m.run_verdicts(p, 0, n, 5)
        oc, ov, oe = O.run(O.OracleModel(cfg), O.OracleFormula(cfg["formula"], cfg["species"]), 5, 0, n)
        assert int(((v.cpu().numpy() != ov) | (e.cpu().numpy() != oe)).sum()) == 0, cfg["formula"]


@pytest.mark.parametrize("seed", range(8))
def test_random_mass_action_networks(smc, seed):
    """Random networks of the C4/C5 recipe (1-2 reactants, 0-2 products, homodimers, rates
    log-uniform in [1e-3, 1]) at several sizes and tile widths, every template formula."""
    g = np.random.default_rng(500 + seed)
    N = int(g.integers(20, 120))
    M = int(g.integers(40, 700))
    net = workloads.random_network(600 + seed, N, M)
    x0 = net["x0"]
    forms = ["F[0,0.02](S0 > %d)" % (x0[0] + 10), "G[0,0.02](S1 > %d)" % (x0[1] - 10),
             "F[0,0.03] G[0,0.005](S0 > S1)", "(S0 < %d) U[0,0.02] (S1 > %d)" % (x0[0] + 30, x0[1] + 5)]
    cfg = dict(name="rn", species=net["species"], x0=x0, reactions=net["reactions"], formula=forms[seed % 4],
               t_max=0.0, seed=seed, sampling=dict(mode="fixed", n=300))
    oc, ov, oe = O.run(O.OracleModel(cfg), O.OracleFormula(cfg["formula"], cfg["species"]), seed, 0, 300)
    os_env = os.environ
    os_env["SMC_TILE_WIDTH"] = ["8", "16", "32"][seed % 3]
    try:
        m, p = _pair(smc, cfg)
        v, e = m.run_verdicts(p, 0, 300, seed)
    finally:
        os_env.pop("SMC_TILE_WIDTH", None)
    bad = int(((v.cpu().numpy() != ov) | (e.cpu().numpy() != oe)).sum())
    assert bad == 0, (seed, N, M, cfg["formula"], bad)
    assert oe.mean() > 20


def test_set_cursor_resumes_the_stream(smc):
    """smc_set_cursor (checkpoint / resume): [0, n) in two resumed halves equals
    one run of n, and a Fig. 2 loop driven round by round through smc_run from a fresh
    model per round (the chunked C5 Wilson-stop driver's pattern) equals smc_estimate."""
    cfg = workloads.c2()
    m, p = _pair(smc, cfg, variant=0)
    whole = m.run(p, 6000, 2)
    m2, p2 = _pair(smc, cfg, variant=0)
    a = m2.run(p2, 2500, 2)
    m3, p3 = _pair(smc, cfg, variant=0)
    m3.set_cursor(2500, 2)
    b = m3.run(p3, 3500, 2)
    assert {k: a[k] + b[k] for k in a} == whole
    # Fig. 2 by hand, one fresh model per round, resumed by cursor
    conf, eps = 0.99, 0.01
    n_tot = yes = cursor = rounds = 0
    N = smc.smc_wilson_sample_size(1.0, eps, conf)
    while True:
        mr, pr = _pair(smc, cfg, variant=0)
        mr.set_cursor(cursor, 7)
        c = mr.run(pr, N, 7)
        cursor += N
        n_tot += c["n_true"] + c["n_false"]
        yes += c["n_true"]
        rounds += 1
        ph = yes / n_tot
        n_new = smc.smc_wilson_sample_size(ph + eps if ph <= 0.5 else ph - eps, eps, conf) - n_tot
        if n_new <= 0:
            break
        N = n_new
    me, pe = _pair(smc, cfg, variant=0)
    est = smc.estimate(me, pe, conf, eps, 7)
    assert (est["n_total"], est["n_true"], est["rounds"]) == (n_tot, yes, rounds)
    assert (est["lower"], est["upper"]) == smc.smc_wilson_interval(yes, n_tot, conf)
