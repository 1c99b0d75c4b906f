"""GPU parity: the CUDA path through the C ABI against the oracle, element by
element, on identical seeded inputs (north star bar: Philox and Wilson
bit-exact; per-replica verdicts agree on >= 99.99 %; p-hat within 5e-4 at
10^6 samples; estimates inside the 99 % Wilson interval of the closed form)."""
import math

import numpy as np
import pytest

import workloads
from oracle import normal_quantile, wilson_interval, wilson_procedure
from oracle import oracle as O

pytestmark = pytest.mark.gpu

AGREE = 0.9999     # per-replica verdict agreement (log rounding may differ, north star)


def _pair(smc, cfg, variant=0):
    m = smc.Model.from_config(cfg)
    if variant:
        m.set_variant(variant)
    p = smc.Property(m, cfg["formula"], t_max=cfg.get("t_max", 0.0))
    return m, p


def _oracle(cfg, seed, first, n, procs=None):
    if n * 1 <= 4000 or procs == 1:
        om = O.OracleModel(cfg)
        of = O.OracleFormula(cfg["formula"], cfg["species"], cfg.get("t_max", 0.0))
        return O.run(om, of, seed, first, n)
    return O.run_parallel(cfg, cfg["formula"], seed, first, n, procs=procs, t_max=cfg.get("t_max", 0.0))


def _compare(smc, cfg, seed, first, n, variant=0, oracle=None):
    m, p = _pair(smc, cfg, variant)
    v, e = m.run_verdicts(p, first, n, seed)
    v, e = v.cpu().numpy(), e.cpu().numpy().astype(np.int64)
    oc, ov, oe = oracle if oracle is not None else _oracle(cfg, seed, first, n)
    agree_v = float((v == ov).mean())
    agree_ve = float(((v == ov) & (e == oe)).mean())
    return agree_v, agree_ve, v, e, ov, oe


def test_philox_stream_bit_exact(smc):
    for seed, traj, step0 in [(1, 0, 0), (2**64 - 1, 2**40 + 7, 2**33), (12345, 999_999, 17_000)]:
        blocks = smc.smc_philox_blocks(seed, traj, step0, 64)
        for q, b in enumerate(blocks):
            assert b == O.philox(seed, traj, step0 + q)


@pytest.mark.parametrize("variant", [1, 2, 4])
def test_c1_all_replicas(smc, variant):
    cfg = workloads.c1()
    a, ae, v, e, ov, oe = _compare(smc, cfg, cfg["seed"], 0, 10_000, variant)
    assert a >= AGREE and ae >= AGREE
    assert list(v[:3]) == [0, 0, 1] and list(e[:3]) == [9, 7, 10]     # worked example
    exact = (1 - math.exp(-2.0)) ** 10
    z = normal_quantile(0.99)
    lo, hi = wilson_interval(v.sum() / 10_000, 10_000, z)
    assert lo <= exact <= hi


@pytest.mark.parametrize("variant", [1, 2, 4])
def test_c2_replicas(smc, variant):
    cfg = workloads.c2()
    a, ae, *_ = _compare(smc, cfg, cfg["seed"], 0, 3000, variant)
    assert a >= AGREE and ae >= AGREE


def test_c2_wilson_estimate(smc):
    """C2 (configs[1]): Fig. 2 at 99 %, eps = 0.005; identical to the oracle's loop on the same
    stream; both contain the exact P = 0.2146528874 (uniformisation)."""
    cfg = workloads.c2()
    m, p = _pair(smc, cfg)
    est = smc.estimate(m, p, 0.99, 0.005, cfg["seed"])
    om = O.OracleModel(cfg)
    of = O.OracleFormula(cfg["formula"], cfg["species"])

    def batch(first, n):
        c, _, _ = O.run_parallel(cfg, cfg["formula"], cfg["seed"], first, n)
        return c["n_true"]
    ref = wilson_procedure(batch, 0.005, 0.99)
    assert abs(est["p_hat"] - ref["p_hat"]) <= 5e-4
    assert abs(est["n_total"] - ref["n_total"]) <= 0.01 * ref["n_total"]
    exact = 0.2146528874
    assert est["lower"] <= exact <= est["upper"]
    assert ref["lower"] <= exact <= ref["upper"]
    assert est["errors"] == 0
    del om, of


@pytest.mark.parametrize("variant", [1, 2, 4])
def test_c3_replicas(smc, variant):
    cfg = workloads.c3()
    a, ae, *_ = _compare(smc, cfg, cfg["seed"], 0, 400, variant)
    assert a == 1.0 and ae == 1.0              # 400 replicas: 0 mismatches (verdict and event count)


def test_c3r_stress(smc):
    cfg = workloads.c3r()
    a, ae, *_ = _compare(smc, cfg, cfg["seed"], 0, 3000)
    assert a >= AGREE


def test_c3_full_size_sampled(smc):
    """Full C3 size (10^6 replicas) in the bench launch configuration; the oracle checks a sample."""
    cfg = workloads.c3()
    m, p = _pair(smc, cfg)
    n = cfg["sampling"]["n"]
    v, e = m.run_verdicts(p, 0, n, cfg["seed"])
    v, e = v.cpu().numpy(), e.cpu().numpy()
    assert set(np.unique(v)) <= {0, 1}
    g = np.random.default_rng(0)
    idx = np.sort(g.choice(n, 64, replace=False))
    om = O.OracleModel(cfg)
    of = O.OracleFormula(cfg["formula"], cfg["species"])
    bad = 0
    for i in idx:
        c, ov, oe = O.run(om, of, cfg["seed"], int(i), 1)
        bad += int(ov[0] != v[i] or oe[0] != e[i])
    assert bad == 0
    # counts path == per-replica path on the same indices
    m.reset()
    c = m.run(p, n, cfg["seed"])
    assert c["n_true"] == int(v.sum()) and c["events"] == int(e.astype(np.int64).sum())
    assert abs(c["n_true"] / n - 0.512) < 0.02          # survey pilot p ~ 0.512 (sanity, not a pin)


def test_edge_cases(smc):
    cfg = workloads.c1()
    m, p = _pair(smc, cfg)
    assert m.run(p, 0, 1) == dict(n_true=0, n_false=0, events=0, errors=0)
    c1 = m.run(p, 1, 1)
    assert c1["n_true"] + c1["n_false"] == 1
    # absorbing start: A0 = 0 -> a0 = 0 at sigma[0]; F(A == 0) decided at entry 0 without events
    z = dict(cfg, x0=[0])
    m0, p0 = _pair(smc, z)
    assert m0.run(p0, 1000, 3) == dict(n_true=1000, n_false=0, events=0, errors=0)
    m1 = smc.Model.from_config(z)
    p1 = smc.Property(m1, "G[0,5](A == 1)")
    assert m1.run(p1, 10, 3) == dict(n_true=0, n_false=10, events=0, errors=0)
    p2 = smc.Property(m1, "F[0,5](A == 1)")            # absorbed immediately -> F false
    assert m1.run(p2, 10, 3)["n_false"] == 10
    # event cap -> counted as errors
    m2, p2 = _pair(smc, workloads.c2())
    m2.set_event_cap(5)
    c = m2.run(p2, 100, 2)
    assert c["errors"] == 100 and c["events"] == 500
    # count overflow -> error: birth from near INT32_MAX
    big = dict(species=["A"], x0=[2147483640], reactions=[dict(reactants=[], products=[[0, 2]], rate=1.0, hill=None)],
               formula="F[0,100](A < 0)")
    m3, p3 = _pair(smc, big)
    c = m3.run(p3, 50, 1)
    assert c["errors"] == 50 and c["events"] == 50 * 3
    # unbounded formula with t_max (pessimistic), oracle parity
    cfgu = dict(cfg, formula="F(A == 0)", t_max=1.5)
    a, ae, *_ = _compare(smc, cfgu, 9, 0, 5000)
    assert a >= AGREE and ae >= AGREE


@pytest.mark.parametrize("variant,xd", [(1, None), (2, None), (4, "1"), (4, "0")])
def test_edge_cases_every_variant(smc, variant, xd, monkeypatch):
    """Edge cases on every kernel family (sweep with binary64 and int32 count columns):
    absorbing start, event cap, count overflow (R17), and counts >= 2^26 whose products
    exceed 2^53 (int64 -> double rounding; the sweep's int32 columns take their general
    conversion path) replica for replica against the oracle."""
    if xd is not None:
        monkeypatch.setenv("SMC_SW_XD", xd)
    z = dict(workloads.c1(), x0=[0])
    m0, p0 = _pair(smc, z, variant)
    assert m0.run(p0, 1000, 3) == dict(n_true=1000, n_false=0, events=0, errors=0)
    assert m0.last_launch(p0)["variant"] == variant
    m2, p2 = _pair(smc, workloads.c2(), variant)
    m2.set_event_cap(5)
    c = m2.run(p2, 100, 2)
    assert c["errors"] == 100 and c["events"] == 500
    big = dict(species=["A"], x0=[2147483640], reactions=[dict(reactants=[], products=[[0, 2]], rate=1.0, hill=None)],
               formula="F[0,100](A < 0)")
    m3, p3 = _pair(smc, big, variant)
    c = m3.run(p3, 50, 1)
    assert c["errors"] == 50 and c["events"] == 50 * 3
    rx = workloads._rx
    huge = dict(name="huge", species=["A", "B", "C"], x0=[200000000, 100000000, 0],
                reactions=[rx([(0, 1), (1, 1)], [(2, 1)], 3e-16), rx([(0, 2)], [(1, 1)], 1e-16),
                           rx([(2, 1)], [], 0.5), rx([], [(0, 1)], 2.0)],
                formula="F[0,3](C >= 12)", t_max=0.0, seed=8, sampling=dict(mode="fixed", n=400))
    a, ae, v, e, ov, oe = _compare(smc, huge, 8, 0, 400, variant)
    assert ae == 1.0, (variant, xd, a, ae)
    assert 0.05 < v.mean() < 0.95 and e.mean() > 10


@pytest.mark.parametrize("formula", [
    "G[0,1](A >= 8)", "(A >= 7) U[0.2,1.5] (A <= 5)", "X[0,0.3](A == 9)", "F[0,1] G[0,0.5](A <= 6)",
    "G[0,1.5] F[0,0.3](A >= 5)", "(G[0,0.5](A > 3)) U[0,2] (A <= 6)", "F(0.5,2](A == 7) & !G[0,0.2](A == 10)",
    "(A == 10) | F[0,0.1](A < 9)"])
def test_templates_vs_oracle(smc, formula):
    cfg = dict(workloads.c1(), formula=formula)
    for variant in (1, 2, 4):
        a, ae, *_ = _compare(smc, cfg, 4, 0, 5000, variant)
        assert a >= AGREE and ae >= AGREE, (formula, variant, a, ae)


def test_shard_invariance(smc):
    """Same (seed, n) split over G emulated ranks (no allreduce) sums to the unsharded counts."""
    cfg = workloads.c2()
    m, p = _pair(smc, cfg)
    whole = m.run(p, 20_000, 11)
    for G in (2, 4, 8):
        tot = dict(n_true=0, n_false=0, events=0, errors=0)
        for r in range(G):
            smc.smc_set_shard(r, G)
            m.reset()
            c = m.run(p, 20_000, 11)
            for k in tot:
                tot[k] += c[k]
        smc.smc_set_shard(0, 1)
        assert tot == whole


@pytest.mark.parametrize("name,variant", [("C4", 2), ("C4", 4), ("C4", 5), ("C5", 2), ("C5", 4), ("C5", 5)])
def test_large_networks_vs_oracle_fixture(smc, name, variant):
    """Tile and sweep variants (smem/TMA-staged tables) vs the oracle's per-replica verdicts and
    event counts (tests/golden/<cfg>_oracle.json, written by scripts/make_fixtures.py from oracle/ only)."""
    import json
    import os
    fx = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "%s_oracle.json" % name.lower())))
    cfg = workloads.get(name)
    assert fx["formula"] == cfg["formula"] and fx["seed"] == cfg["seed"]
    m, p = _pair(smc, cfg, variant)
    v, e = m.run_verdicts(p, fx["first"], fx["n"], fx["seed"])
    v, e = v.cpu().numpy(), e.cpu().numpy()
    ov, oe = np.array(fx["verdicts"]), np.array(fx["events"])
    mism = int(((v != ov) | (e != oe)).sum())
    assert mism == 0, (name, variant, mism)
    assert m.last_launch(p)["variant"] == variant


@pytest.mark.parametrize("xd,block,fmaacc", [("0", None, "1"), ("1", "96", "1"), ("0", "224", "1"), ("1", None, "0")])
def test_sweep_shapes_vs_fixture(smc, xd, block, fmaacc, monkeypatch):
    """The sweep variant with int32 count columns (exact fma laws, I2F in the selection), other
    CTA sizes (the column stride and the pre-scaled law offsets follow it) and with / without
    the fused accumulation of reading R25 gives the oracle's C4 replicas."""
    import json
    import os
    monkeypatch.setenv("SMC_SW_XD", xd)
    monkeypatch.setenv("SMC_SW_FMAACC", fmaacc)
    if block:
        monkeypatch.setenv("SMC_SW_BLOCK", block)
    fx = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "c4_oracle.json")))
    cfg = workloads.c4()
    m, p = _pair(smc, cfg, variant=4)
    n = 600
    v, e = m.run_verdicts(p, 0, n, fx["seed"])
    v, e = v.cpu().numpy(), e.cpu().numpy()
    mism = int(((v != np.array(fx["verdicts"][:n])) | (e != np.array(fx["events"][:n]))).sum())
    assert mism == 0, (xd, block, mism)
    info = m.last_launch(p)
    assert info["variant"] == 4 and info["block_threads"] <= int(block or 384)   # launched CTA <= the compiled one


@pytest.mark.parametrize("N,M,form", [(64, 512, "F[0,0.01](S0 > {a})"), (64, 512, "G[0,0.01](S1 > {b})"),
                                       (100, 400, "F[0,0.01](S0 > {c})")])
def test_sweep_mid_size_networks_vs_oracle(smc, N, M, form):
    """The sweep at the sizes its automatic choice covers beyond C4 (groups of 18 laws read in
    chunks of 6, 288-thread CTAs; 100 species: 256-thread CTAs at the register cap) against
    the oracle replica for replica (C4/C5-recipe random networks)."""
    net = workloads.random_network(11, N, M)
    x0 = net["x0"]
    f = form.format(a=x0[0] + 15, b=x0[1] - 15, c=x0[0] + 40)
    cfg = dict(name="rn%d_%d" % (N, M), species=net["species"], x0=x0, reactions=net["reactions"], formula=f,
               t_max=0.0, seed=7, sampling=dict(mode="fixed", n=60))
    a, ae, v, e, ov, oe = _compare(smc, cfg, 7, 0, 60)
    assert ae == 1.0, (N, M, f, a, ae)
    assert e.mean() > 100
    m, p = _pair(smc, cfg)
    assert m.run(p, 1, 7) and m.last_launch(p)["variant"] == 4


@pytest.mark.parametrize("width", ["4", "8", "16", "32"])
def test_tile_widths_vs_fixture(smc, width, monkeypatch):
    """Every tile width of variant 2 (4/8/16/32 lanes per trajectory) gives the oracle's replicas."""
    import json
    import os
    monkeypatch.setenv("SMC_TILE_WIDTH", width)
    fx = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "c4_oracle.json")))
    cfg = workloads.c4()
    m, p = _pair(smc, cfg, variant=2)
    n = 600
    v, e = m.run_verdicts(p, 0, n, fx["seed"])
    v, e = v.cpu().numpy(), e.cpu().numpy()
    mism = int(((v != np.array(fx["verdicts"][:n])) | (e != np.array(fx["events"][:n]))).sum())
    assert mism == 0
    for name in ("C2", "C3"):
        cfg = workloads.get(name)
        a, ae, *_ = _compare(smc, cfg, cfg["seed"], 0, 300, variant=2)
        assert ae == 1.0


def test_c4_full_size_shard_sampled(smc):
    """C4 (configs[3]: 10^7 replicas over 8 GPUs): rank 0's shard of 1.25e6 replicas in the bench
    launch configuration; the oracle checks sampled replicas one by one."""
    cfg = workloads.c4()
    lo, hi = smc.smc_shard_range(0, cfg["sampling"]["n"], 0, 8)
    m, p = _pair(smc, cfg)
    v, e = m.run_verdicts(p, lo, hi - lo, cfg["seed"])
    v, e = v.cpu().numpy(), e.cpu().numpy()
    assert set(np.unique(v)) <= {0, 1}
    idx = np.sort(np.random.default_rng(1).choice(hi - lo, 16, replace=False))
    om = O.OracleModel(cfg)
    of = O.OracleFormula(cfg["formula"], cfg["species"])
    bad = 0
    for i in idx:
        c, ov, oe = O.run(om, of, cfg["seed"], int(lo + i), 1)
        bad += int(ov[0] != v[i] or oe[0] != e[i])
    assert bad == 0
    assert abs(v.mean() - 0.54) < 0.03          # fixture estimate 0.5415 (2000 oracle replicas)


@pytest.mark.parametrize("name,eps", [("C1", 0.01), ("C2", 0.005), ("C3", 0.02), ("C1", 0.0005), ("C1", 0.0003)])
def test_speculative_rounds_identical(smc, name, eps):
    """Prefix-exact speculation changes only the schedule: the
    Fig. 2 estimate equals the one from exactly-sized rounds, bit for bit."""
    cfg = workloads.get(name)
    m, p = _pair(smc, cfg)
    on = smc.estimate(m, p, 0.99, eps, 17)
    m.set_speculation(False)
    off = smc.estimate(m, p, 0.99, eps, 17)
    assert on == off
    assert on["rounds"] >= 2
    # eps = 5e-4 / 3e-4: Eq. 4(0.5) (6.6e6 / 1.8e7) exceeds the resident lanes, so rounds run
    # over several speculative batches, partly covered ones included


def test_c5_first_round_sampled(smc):
    """C5 (configs[4]): the first Fig. 2 round at 99.9 %, eps = 1e-4 (54,128 replicas), sampled."""
    cfg = workloads.c5()
    n = smc.smc_wilson_sample_size(1.0, 1e-4, 0.999)
    assert n == 54128
    m, p = _pair(smc, cfg)
    v, e = m.run_verdicts(p, 0, n, cfg["seed"])
    v, e = v.cpu().numpy(), e.cpu().numpy()
    idx = np.sort(np.random.default_rng(2).choice(n, 6, replace=False))
    om = O.OracleModel(cfg)
    of = O.OracleFormula(cfg["formula"], cfg["species"])
    bad = 0
    for i in idx:
        c, ov, oe = O.run(om, of, cfg["seed"], int(i), 1)
        bad += int(ov[0] != v[i] or oe[0] != e[i])
    assert bad == 0


def _law_kinds_cfg():
    """Every propensity law shape (readings R8/S8): h = 1, x, x(x-1)/2, x*y with a product
    above 2^31, C(x,2)*y (order 3) and C(x,2)*C(y,2) (order 4), at counts where the int64
    count and its double differ from any 32-bit shortcut."""
    rx = workloads._rx
    return dict(name="laws", species=["A", "B", "C", "D"], x0=[40000, 50000, 3, 100],
                reactions=[rx([(0, 2)], [(2, 1)], 1e-9),            # 2A -> C        (homodimer)
                           rx([(0, 1), (1, 1)], [(3, 1)], 1e-10),   # A + B -> D     (h ~ 2e9)
                           rx([(0, 2), (1, 1)], [(2, 1)], 1e-15),   # 2A + B -> C    (order 3)
                           rx([(2, 2), (3, 2)], [(0, 1)], 1e-5),    # 2C + 2D -> A   (order 4)
                           rx([(3, 1)], [], 0.1),                   # D -> 0
                           rx([], [(2, 1)], 1.0)],                  # 0 -> C         (h = 1)
                formula="F[0,5](C > 8)", t_max=0.0, seed=11, sampling=dict(mode="fixed", n=2000))


@pytest.mark.parametrize("variant", [1, 2, 4])
def test_all_law_kinds_vs_oracle(smc, variant):
    """The tile kernel forms h in fp64 for order <= 2 and in int64 for order 3-4; the thread
    kernel always in int64.  Both must reproduce the oracle's replicas exactly."""
    cfg = _law_kinds_cfg()
    a, ae, v, e, ov, oe = _compare(smc, cfg, cfg["seed"], 0, 2000, variant)
    assert ae >= 1999 / 2000, (variant, a, ae)
    assert 0 < v.mean() < 1 and e.mean() > 20


def test_draws_vs_oracle(smc):
    """The device draw (Philox -> u53 -> fast -log, reading R18) against the oracle's:
    u2 bit-exact, e = -log(u1) within 1 ulp of glibc and bit-identical for >= 90 %."""
    import struct
    n_exact = n_tot = 0
    for seed, traj, step0 in [(1, 0, 0), (7, 123456, 10_000), (2**64 - 1, 2**40 + 7, 2**33)]:
        d = smc.smc_draw_blocks(seed, traj, step0, 4096)
        for q, (e, u2) in enumerate(d):
            u1o, u2o = O.uniforms(seed, traj, step0 + q)
            assert u2 == u2o
            eo = -math.log(u1o)
            ulp = abs(struct.unpack("<q", struct.pack("<d", e))[0] - struct.unpack("<q", struct.pack("<d", eo))[0])
            assert ulp <= 1, (seed, traj, step0 + q, e, eo)
            n_exact += ulp == 0
            n_tot += 1
    assert n_exact / n_tot >= 0.90


@pytest.mark.parametrize("p", [0.0, 0.05, 0.5, 0.95, 1.0])
def test_fig3_modes_vs_oracle(smc, p):
    """NEXT-4: conservative (start 0.5) and iterative (Fig. 2) estimates of a
    Bernoulli(p) CTMC through the GPU path equal the oracle's Fig. 2 on the oracle SSA,
    replica for replica; the conservative size is Eq. 4(0.5) = 2648 at 2 eps = 0.05 / 99 %."""
    cfg = workloads.bernoulli(p)
    m, prop = _pair(smc, cfg)
    om = O.OracleModel(cfg)
    of = O.OracleFormula(cfg["formula"], cfg["species"])
    for seed in (1, 2, 3):
        for start in (1.0, 0.5):
            g = smc.estimate(m, prop, 0.99, 0.025, seed, start=start)
            o = wilson_procedure(lambda f, n: O.run(om, of, seed, f, n, per_traj=False)[0]["n_true"], 0.025, 0.99,
                                 start=start)
            assert (g["n_total"], g["n_true"]) == (o["n_total"], o["n_true"]), (p, seed, start)
            assert (g["p_hat"], g["lower"], g["upper"]) == (o["p_hat"], o["lower"], o["upper"])
            if start == 0.5:
                assert g["n_total"] == 2648 and g["rounds"] == 1
    if p in (0.0, 1.0):                          # the 88 % of P:392: 1 - 304 / 2648
        assert smc.estimate(m, prop, 0.99, 0.025, 1)["n_total"] == 304


@pytest.mark.parametrize("variant", [1, 2, 4])
def test_explicit_rates_vs_oracle(smc, variant):
    """NEXT-3: explicit propensities (repressed production, Michaelis-Menten conversion,
    explicit decay) mixed with mass-action laws, thread and tile variants, replica by
    replica against the oracle's independent parser / evaluator."""
    cfg = workloads.explicit_demo()
    a, ae, v, e, ov, oe = _compare(smc, cfg, cfg["seed"], 0, 3000, variant)
    assert ae >= AGREE, (variant, a, ae)
    assert 0.5 < v.mean() < 0.7


def test_explicit_michaelis_menten_degradation_gpu_vs_matrix_exponential(smc):
    """The GPU estimate of F[0,2.5](S == 0) for S -> 0 at 10 S/(5+S), S0 = 20, contains the
    matrix-exponential value (the same pin as the oracle's, tests/test_oracle_rates.py)."""
    from scipy.linalg import expm
    rx = workloads._rx
    cfg = dict(name="MMdeg", species=["S"], x0=[20], reactions=[dict(rx([(0, 1)], [], 1.0), rate_expr="10*S/(5+S)")],
               formula="F[0,2.5](S == 0)", t_max=0.0, seed=3, sampling=dict(mode="fixed", n=10 ** 6))
    Q = np.zeros((21, 21))
    for s in range(1, 21):
        Q[s, s], Q[s, s - 1] = -10 * s / (5 + s), 10 * s / (5 + s)
    exact = float(expm(Q * 2.5)[20, 0])
    m, p = _pair(smc, cfg)
    c = m.run(p, 10 ** 6, 3)
    n = c["n_true"] + c["n_false"]
    lo, hi = wilson_interval(c["n_true"] / n, n, normal_quantile(0.999))
    assert c["errors"] == 0 and lo <= exact <= hi


@pytest.mark.parametrize("row", [0, 1, 2])
def test_cell_cycle_rows_vs_oracle(smc, row):
    """NEXT-3 workload: the best-effort cell-cycle model (explicit Table 2 rates) with the
    three Table 3 formulas, GPU replicas against the oracle's."""
    cfg = workloads.cell_cycle(workloads.CELL_CYCLE_FORMULAS[row])
    a, ae, *_ = _compare(smc, cfg, cfg["seed"], 0, 2000)
    assert ae >= AGREE, (row, a, ae)


@pytest.mark.parametrize("variant", [1, 2, 4])
def test_general_val_atoms_vs_oracle(smc, variant):
    """NEXT-2: general val atoms -- non-linear int64 products, '/', Real constants,
    sqrt / abs / min / max / pow -- in the GPU monitors, replica by replica against the
    oracle (the decision event is part of the comparison)."""
    cfg = workloads.c2()
    for f in ["F[0,50](sqrt(P) > 22.5)", "(E < sqrt(S) + 70) U[0,50] (P / 2 >= 250.5)",
              "F[0,50](P * S > 140000)", "F[0,50](abs(ES - 30.5) < 1 & max(E, 60) == E)",
              "G[0,30](pow(ES, 2) / 7 <= min(E, 90.5) * 30)"]:
        a, ae, *_ = _compare(smc, dict(cfg, formula=f), 2, 0, 1500, variant)
        assert ae >= AGREE, (f, variant, a, ae)


def test_c2_million_replicas_vs_oracle(smc):
    """North star at 10^6 samples (C2, configs[1] model, the fixed-N parity run of SURVEY
    §8(d)): per-replica agreement >= 99.99 %, |p_hat_gpu - p_hat_oracle| <= 5e-4, and both
    99 % Wilson intervals contain the exact P = 0.2146528874 (uniformisation)."""
    cfg = workloads.c2()
    n = 10 ** 6
    m, p = _pair(smc, cfg)
    v, e = m.run_verdicts(p, 0, n, cfg["seed"])
    v, e = v.cpu().numpy(), e.cpu().numpy().astype(np.int64)
    oc, ov, oe = O.run_parallel(cfg, cfg["formula"], cfg["seed"], 0, n)
    assert float(((v == ov) & (e == oe)).mean()) >= AGREE
    pg, po = float(v.mean()), oc["n_true"] / n
    assert abs(pg - po) <= 5e-4
    z = normal_quantile(0.99)
    for ph in (pg, po):
        lo, hi = wilson_interval(ph, n, z)
        assert lo <= 0.2146528874 <= hi


def test_c3_million_replicas_vs_oracle(smc):
    """C3 (configs[2]: 10^6 replicas) in full against the oracle on the same streams:
    per-replica agreement >= 99.99 % and |p_hat_gpu - p_hat_oracle| <= 5e-4 (north star)."""
    cfg = workloads.c3()
    n = cfg["sampling"]["n"]
    m, p = _pair(smc, cfg)
    v, e = m.run_verdicts(p, 0, n, cfg["seed"])
    v, e = v.cpu().numpy(), e.cpu().numpy().astype(np.int64)
    oc, ov, oe = O.run_parallel(cfg, cfg["formula"], cfg["seed"], 0, n)
    assert float(((v == ov) & (e == oe)).mean()) >= AGREE
    assert abs(float(v.mean()) - oc["n_true"] / n) <= 5e-4


def _iso_cfg():
    rx = workloads._rx
    return dict(name="iso", species=["A", "B"], x0=[10, 0], reactions=[rx([(0, 1)], [(1, 1)], 1.0), rx([(1, 1)], [(0, 1)], 0.5)],
                formula="", t_max=0.0, seed=5, sampling=dict(mode="fixed", n=2000))


NESTED = [("iso", "F[0,3](A <= 5 & G[0,0.5](B >= 4))"), ("iso", "G[0,1.5](!(A < 7) | F[0.2,1](B <= 3))"),
          ("iso", "F[0.5,3](X[0,0.3](A == 6))"), ("iso", "F[0,3](G[0.2,0.6](A > 4))"),
          ("iso", "(F[0,1](B > 3)) U[0,3] (A < 5)"), ("iso", "!F[0,1](A == 7) | G[0,0.5](X[0,0.2](B > 2))"),
          ("iso", "F[0,4]((A > 6) U[0.1,1] (B > 3))"), ("iso", "G(A + B == 10) & F(0,2](G[0,0.3](A == B))"),
          ("c2", "F[0,3](P > 25 & G[0,0.5](P < 33))"), ("c2", "G[0,2](F[0.05,0.3](ES >= E / 4))")]


@pytest.mark.parametrize("case", range(len(NESTED)))
def test_nested_formulas_literal_variant_vs_oracle(smc, case):
    """NEXT-2: formulas outside the streaming templates (nested temporal operators, non-zero
    inner lower bounds, X inside F, unbounded with t_max) run through the literal variant
    (the window monitor on the device, R27) and equal the oracle's literal mode replica for
    replica, verdicts and event counts."""
    name, f = NESTED[case]
    cfg = dict(_iso_cfg() if name == "iso" else workloads.c2(), formula=f)
    t_max = 4.0 if "G(" in f else 0.0
    cfg["t_max"] = t_max
    m, p = _pair(smc, cfg)
    v, e = m.run_verdicts(p, 0, 2000, 5)
    v, e = v.cpu().numpy(), e.cpu().numpy().astype(np.int64)
    assert m.last_launch(p)["variant"] == 3
    om = O.OracleModel(cfg)
    of = O.OracleFormula(f, cfg["species"], t_max)
    oc, ov, oe = O.run(om, of, 5, 0, 2000, mode="literal")
    assert float(((v == ov) & (e == oe)).mean()) == 1.0, (f, float((v == ov).mean()), float((e == oe).mean()))


@pytest.mark.parametrize("case", range(len(NESTED)))
def test_nested_formulas_tile_recording_monitor_vs_oracle(smc, case):
    """NEXT-2 in the tile kernel (window monitor, readings R23/R27): the NESTED formulas with
    the models forced to variant 2 equal the oracle's literal mode replica for replica."""
    name, f = NESTED[case]
    cfg = dict(_iso_cfg() if name == "iso" else workloads.c2(), formula=f)
    t_max = 4.0 if "G(" in f else 0.0
    cfg["t_max"] = t_max
    m, p = _pair(smc, cfg, variant=2)
    v, e = m.run_verdicts(p, 0, 1000, 5)
    v, e = v.cpu().numpy(), e.cpu().numpy().astype(np.int64)
    assert m.last_launch(p)["variant"] == 2
    oc, ov, oe = O.run(O.OracleModel(cfg), O.OracleFormula(f, cfg["species"], t_max), 5, 0, 1000, mode="literal")
    assert float(((v == ov) & (e == oe)).mean()) == 1.0, (f, float((v == ov).mean()), float((e == oe).mean()))


def test_nested_formula_on_c4_tile_vs_oracle(smc):
    """A formula outside R16 on the 50 x 200 network (the sweep kernel with the window monitor)."""
    f = "F[0.01,0.03](X[0,0.0001](S1 > S0 - 40))"
    cfg = dict(workloads.c4(), formula=f)
    m, p = _pair(smc, cfg)
    v, e = m.run_verdicts(p, 0, 40, 4)
    v, e = v.cpu().numpy(), e.cpu().numpy().astype(np.int64)
    assert m.last_launch(p)["variant"] == 4                 # the sweep hosts the window monitor
    oc, ov, oe = O.run(O.OracleModel(cfg), O.OracleFormula(f, cfg["species"]), 4, 0, 40, mode="literal")
    assert int(((v != ov) | (e != oe)).sum()) == 0


def _random_case(seed):
    """A random small network (mass action orders 0-2, Hill repression, explicit rates) and a
    random formula (every streaming template, Kleene roots, nested shapes outside R16)."""
    g = np.random.default_rng(seed)
    N = int(g.integers(2, 5))
    sp = ["A", "B", "C", "D"][:N]
    rx = workloads._rx
    R = []
    for _ in range(int(g.integers(2, 7))):
        nr = int(g.integers(0, 3))
        reac = {}
        for _ in range(nr):
            s = int(g.integers(0, N))
            reac[s] = reac.get(s, 0) + 1
        prods = {}
        for _ in range(int(g.integers(0, 3))):
            s = int(g.integers(0, N))
            prods[s] = prods.get(s, 0) + 1
        r = rx(list(reac.items()), list(prods.items()), float(np.exp(g.uniform(np.log(0.05), np.log(2.0)))))
        kind = g.random()
        if kind < 0.15 and nr == 0:
            r["hill"] = dict(repressor=int(g.integers(0, N)), K=float(g.uniform(2, 10)), n=int(g.integers(1, 3)))
        elif kind < 0.3:
            s = sp[int(g.integers(0, N))]
            r["rate_expr"] = "%r * (1 + %s) / (2 + %s)" % (float(g.uniform(0.2, 2)), s, s)
        R.append(r)
    R.append(rx([], [(0, 1)], 0.5))                      # keep something happening
    R.append(rx([(0, 1)], [], 0.2))
    x0 = [int(v) for v in g.integers(0, 8, size=N)]
    a, b = sp[0], sp[min(1, N - 1)]
    c1, c2 = int(g.integers(1, 8)), int(g.integers(1, 8))
    T = float(g.choice([1.0, 2.0, 4.0]))
    lo = float(g.choice([0.0, 0.0, 0.3]))
    forms = ["F[%r,%r](%s >= %d)" % (lo, T, a, c1), "G[%r,%r](%s < %d)" % (lo, T, b, c2),
             "(%s < %d) U[%r,%r] (%s >= %d)" % (a, c1, lo, T, b, c2), "X[0,%r](%s > %d | %s == 0)" % (T / 4, a, c1, b),
             "F[0,%r] G[0,%r](%s > %s)" % (T, T / 4, a, b), "G[0,%r] F[0,%r](%s >= %s)" % (T, T / 4, a, b),
             "(G[0,%r](%s < %d)) U[0,%r] (%s > %d)" % (T / 4, a, c1 + 3, T, b, c2),
             "!(F[0,%r](%s == %d)) & (G[0,%r](%s >= 0) | F(0,%r](%s > %d))" % (T, a, c1, T / 2, b, T, a, c2),
             "F[0,%r](%s > %d & G[0.1,%r](%s > 0))" % (T, a, c1, T / 3, b),
             "G[0,%r](%s / 2 <= sqrt(%s + 1) * 3 | X[0,0.5](%s > %d))" % (T, a, b, a, c1)]
    f = forms[int(g.integers(0, len(forms)))]
    return dict(name="rnd%d" % seed, species=sp, x0=x0, reactions=R, formula=f, t_max=0.0, seed=seed,
                sampling=dict(mode="fixed", n=400))


@pytest.mark.parametrize("seed", range(24))
def test_random_models_and_formulas_vs_oracle(smc, seed):
    """Fuzz: random networks x random formulas, thread and tile variants, replica for replica
    against the oracle (its streaming monitor inside the fragment, its literal |= outside)."""
    cfg = _random_case(seed)
    of = O.OracleFormula(cfg["formula"], cfg["species"])
    mode = "stream" if of.streamable else "literal"
    oc, ov, oe = O.run(O.OracleModel(cfg), of, seed, 0, 400, mode=mode)
    for variant in (1, 2, 4):
        m, p = _pair(smc, cfg, variant)
        v, e = m.run_verdicts(p, 0, 400, seed)
        v, e = v.cpu().numpy(), e.cpu().numpy().astype(np.int64)
        bad = int(((v != ov) | (e != oe)).sum())
        assert bad == 0, (seed, variant, cfg["formula"], bad)
        assert (v != 2).all()                 # no replica error (trace buffers sized per launch)


def _random_large_case(seed):
    """A random tile-only network (N > 32 or M > 32) with every law shape: mass action of
    order 0-4, Hill repression, explicit rates, null reactions; template formulas."""
    g = np.random.default_rng(1000 + seed)
    N = int(g.integers(33, 45))
    M = int(g.integers(40, 80))
    sp = ["S%d" % i for i in range(N)]
    rx = workloads._rx
    R = []
    for _ in range(M):
        reac = {}
        for _ in range(int(g.integers(0, 3))):
            s = int(g.integers(0, N))
            reac[s] = min(2, reac.get(s, 0) + 1)
        prods = {}
        for _ in range(int(g.integers(0, 3))):
            s = int(g.integers(0, N))
            prods[s] = min(2, prods.get(s, 0) + 1)
        r = rx(list(reac.items()), list(prods.items()), float(np.exp(g.uniform(np.log(0.01), np.log(1.0)))))
        u = g.random()
        if u < 0.1 and not reac:
            r["hill"] = dict(repressor=int(g.integers(0, N)), K=float(g.uniform(5, 50)), n=int(g.integers(1, 4)))
        elif u < 0.2:
            s = sp[int(g.integers(0, N))]
            r["rate_expr"] = "%r * %s / (10 + %s) + 0.01" % (float(g.uniform(0.1, 2)), s, s)
        R.append(r)
    x0 = [int(v) for v in g.integers(0, 40, size=N)]
    a, b = sp[0], sp[1]
    forms = ["F[0,3](%s > %s + 5)" % (a, b), "G[0,2](%s <= %s + 30)" % (a, b), "(%s < 50) U[0,3] (%s > 45)" % (a, b),
             "F[0,3] G[0,0.5](%s > %s)" % (a, b), "(G[0,0.5](%s < 60)) U[0,3] (%s >= 41)" % (a, b),
             "X[0,0.2](%s != %s) | F[0,1](%s == 0)" % (a, b, b)]
    return dict(name="big%d" % seed, species=sp, x0=x0, reactions=R, formula=forms[seed % len(forms)], t_max=0.0,
                seed=seed, sampling=dict(mode="fixed", n=300))


@pytest.mark.parametrize("seed", range(12))
def test_random_large_networks_vs_oracle(smc, seed):
    """Fuzz of the tile and sweep kernels: random tile-only networks (every law shape) x
    template formulas, every tile width and the sweep variant, replica for replica against
    the oracle's streaming monitor."""
    cfg = _random_large_case(seed)
    oc, ov, oe = O.run(O.OracleModel(cfg), O.OracleFormula(cfg["formula"], cfg["species"]), seed, 0, 300)
    for width in ("8", "32", "sweep") if seed % 2 else ("4", "16", "sweep"):
        os_env = __import__("os").environ
        if width != "sweep":
            os_env["SMC_TILE_WIDTH"] = width
        try:
            m, p = _pair(smc, cfg, 4 if width == "sweep" else 2)
            v, e = m.run_verdicts(p, 0, 300, seed)
        finally:
            os_env.pop("SMC_TILE_WIDTH", None)
        v, e = v.cpu().numpy(), e.cpu().numpy().astype(np.int64)
        assert m.last_launch(p)["variant"] == (4 if width == "sweep" else 2)
        bad = int(((v != ov) | (e != oe)).sum())
        assert bad == 0, (seed, width, cfg["formula"], bad, oc)
