"""libsmc.so on a machine without a GPU: it loads, exports every symbol of
include/smc.h, and its HOST logic is right (Wilson bit-exact with the oracle,
property compiler, codegen, shard ranges, the Fig. 2 driver).  No kernel runs."""
import os
import re

import numpy as np
import pytest

import workloads
import paper_0912_2551_b200 as smc
from paper_0912_2551_b200 import _native
from oracle import normal_quantile, wilson_interval, wilson_procedure, wilson_sample_size
from oracle import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "smc.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(smc_[a-z_]+)\s*\(", text)) - {"smc_run_fn"})


def test_exports_every_declared_symbol():
    L = smc.lib()
    syms = header_symbols()
    assert len(syms) == 30
    for s in syms:
        assert hasattr(L, s), s
    assert sorted(n for n, _, _ in _native.SIGNATURES) == syms


CONF = [0.8, 0.9, 0.95, 0.99, 0.995, 0.999, 0.9999, 0.99999]


@pytest.mark.parametrize("c", CONF)
def test_z_bit_exact(c):
    assert smc.smc_normal_quantile(c) == normal_quantile(c)


def test_wilson_interval_bit_exact():
    g = np.random.default_rng(1)
    for _ in range(3000):
        n = int(g.integers(1, 10**8))
        k = int(g.integers(0, n + 1)) if g.random() < 0.8 else int(g.choice([0, n]))
        c = float(g.choice(CONF))
        lo, hi = smc.smc_wilson_interval(k, n, c)
        olo, ohi = wilson_interval(k / n, n, normal_quantile(c))
        assert (lo, hi) == (olo, ohi)


def test_wilson_sample_size_bit_exact():
    g = np.random.default_rng(2)
    for _ in range(3000):
        p = float(g.random()) if g.random() < 0.9 else float(g.choice([0.0, 0.5, 1.0]))
        eps = float(g.choice([0.1, 0.05, 0.025, 0.01, 0.005, 1e-3, 1e-4]))
        c = float(g.choice(CONF))
        assert smc.smc_wilson_sample_size(p, eps, c) == wilson_sample_size(p, eps, normal_quantile(c))
    assert smc.smc_wilson_sample_size(0.5, 0.025, 0.99) == 2648


def test_shard_ranges_partition():
    for n in [0, 1, 7, 1000, 10**7 + 3]:
        for world in [1, 2, 3, 4, 8]:
            parts = [smc.smc_shard_range(100, n, r, world) for r in range(world)]
            assert parts[0][0] == 100 and parts[-1][1] == 100 + n
            for (a, b), (c, d) in zip(parts, parts[1:]):
                assert b == c and a <= b
            sizes = [b - a for a, b in parts]
            assert max(sizes) - min(sizes) <= 1


def test_model_validation_lists_all_violations():
    bad = dict(species=["A", "B"], x0=[-1, 3],
               reactions=[dict(reactants=[[5, 1]], products=[], rate=1.0),
                          dict(reactants=[[0, 1]], products=[[1, 1]], rate=-2.0)])
    with pytest.raises(smc.SmcError) as e:
        smc.Model.from_config(bad)
    assert e.value.name == "SMC_E_MODEL"
    msg = str(e.value)
    assert "init_counts[0]" in msg and "reaction 0" in msg and "reaction 1" in msg


def test_property_compiler_errors():
    m = smc.Model.from_config(workloads.c2())
    with pytest.raises(smc.SmcError) as e:
        smc.Property(m, "F[0,50](Q > 500)")
    assert e.value.name == "SMC_E_PARSE" and "unknown species" in str(e.value)
    with pytest.raises(smc.SmcError) as e:
        smc.Property(m, "F[0,50](P > )")
    assert e.value.name == "SMC_E_PARSE"
    with pytest.raises(smc.SmcError) as e:
        smc.Property(m, "F[0,50](sqr(P) > 5)")          # unknown function
    assert e.value.name == "SMC_E_PARSE"
    with pytest.raises(smc.SmcError) as e:
        smc.Property(m, "F[0,50](pow(P, 1.5) > 5)")     # pow takes an integer exponent
    assert e.value.name == "SMC_E_PARSE"
    # outside the streaming templates: compiled for the literal variant (buffered trace + |=)
    assert "smc_ssa_literal" in m.kernel_source(smc.Property(m, "F[0,5](G[1,2](P > 5))"))
    assert "smc_ssa_thread" in m.kernel_source(smc.Property(m, "F[0,5] G[0,2](P > 5)"))
    with pytest.raises(smc.SmcError) as e:
        smc.Property(m, "F(P > 5)")                 # unbounded needs t_max
    assert e.value.name == "SMC_E_UNSUPPORTED"
    for ok in ["F(P > 5)", "(E <= 4) U (P >= 5)", "G[0,1](2*ES - P + 3 != 0) & !X[0,1](S == 1000)",
               "F[0,10] G[0,1](E > S)", "(G[0,100](E < 400)) U[0,200] (P > 300)", "F(0,1.5](P >= 2) | true",
               "F[0,50](P * S > 5)", "(E < sqrt(S)) U[0,5] (S >= 10 + ES)", "G[0,1](min(E, S) / 2.5 >= pow(P, 2))"]:
        smc.Property(m, ok, t_max=100.0)


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4"])
def test_codegen_source(name):
    cfg = workloads.get(name)
    m = smc.Model.from_config(cfg)
    p = smc.Property(m, cfg["formula"])
    src = m.kernel_source(p)
    assert "struct SmcMon" in src
    assert ("smc_ssa_thread" in src) == (len(cfg["reactions"]) <= 32)
    assert ("smc_ssa_sweep" in src) == (name == "C4")          # automatic choice: sweep for C4


def test_variant_selection_and_errors():
    cfg = workloads.c4()
    m = smc.Model.from_config(cfg)
    p = smc.Property(m, cfg["formula"])
    for v, entry in ((2, "smc_ssa_tile"), (4, "smc_ssa_sweep"), (5, "smc_ssa_delta"), (0, "smc_ssa_sweep")):
        m.set_variant(v)
        assert entry in m.kernel_source(p)
    # the automatic choice for C5 (N = 200: beyond the sweep) is the delta kernel
    m5 = smc.Model.from_config(workloads.c5())
    assert "smc_ssa_delta" in m5.kernel_source(smc.Property(m5, workloads.c5()["formula"]))
    # the delta kernel needs mass action of order <= 2 (C3's Hill laws are not)
    m3 = smc.Model.from_config(workloads.c3())
    with pytest.raises(smc.SmcError):
        m3.set_variant(5)
    for bad in (3, 6, -1, 1):            # 3 is the literal variant (chosen by the formula), 1 needs N, M <= 32
        with pytest.raises(smc.SmcError):
            m.set_variant(bad)
    # a literal (nested) formula on a sweep model runs the sweep kernel with the window monitor (R27)
    m.set_variant(4)
    lp = smc.Property(m, "F[0,1](G[0.5,1](S0 > S1))")
    src = m.kernel_source(lp)
    assert "smc_ssa_sweep" in src and "SmcWN<" in src
    # the counts of 128 trajectories must fit in shared memory
    big = dict(cfg, species=["S%d" % i for i in range(500)], x0=[1] * 500)
    mb = smc.Model.from_config(big)
    with pytest.raises(smc.SmcError):
        mb.set_variant(4)


def _oracle_runner(cfg, seed, stats):
    om = O.OracleModel(cfg)
    of = O.OracleFormula(cfg["formula"], cfg["species"])

    def run(first, n):
        c, _, _ = O.run(om, of, seed, first, n, per_traj=False)
        stats.append((first, n))
        return c
    return run


def test_fig2_driver_matches_oracle_loop():
    """The library's Fig. 2 loop (host C++) == the oracle's (Python) on the same replica stream."""
    cfg = workloads.c1()
    calls = []
    lib_est = smc.estimate_with_runner(_oracle_runner(cfg, 7, calls), 0.99, 0.01)
    om = O.OracleModel(cfg)
    of = O.OracleFormula(cfg["formula"], cfg["species"])
    ref = wilson_procedure(lambda f, n: O.run(om, of, 7, f, n, per_traj=False)[0]["n_true"], 0.01, 0.99)
    assert lib_est["n_total"] == ref["n_total"] and lib_est["n_true"] == ref["n_true"]
    assert (lib_est["p_hat"], lib_est["lower"], lib_est["upper"]) == (ref["p_hat"], ref["lower"], ref["upper"])
    assert lib_est["rounds"] == ref["rounds"] == len(calls)


def test_rate_expression_errors_and_codegen():
    """smc_model_set_rate_expr: parse errors carry the position, unknown species and
    Hill conflicts are rejected, and the generated law is straight-line IEEE code in
    tree order with the guard."""
    rx = workloads._rx
    base = dict(name="r", species=["S", "P"], x0=[5, 0], formula="F[0,1](P > 2)", t_max=0.0, seed=1,
                sampling=dict(mode="fixed", n=10))
    for expr, where in [("2*", "at 2"), ("(S", "at 2"), ("S $ 2", "at 2"), ("Q", "at 0"), ("2 S", "at 2")]:
        cfg = dict(base, reactions=[dict(rx([(0, 1)], [(1, 1)], 1.0), rate_expr=expr)])
        with pytest.raises(smc.SmcError) as e:
            smc.Model.from_config(cfg)
        assert e.value.name == "SMC_E_PARSE" and where in str(e.value), (expr, str(e.value))
    cfg = dict(base, reactions=[dict(rx([(0, 1)], [(1, 1)], 1.0), rate_expr="10*S/(5+S)",
                                     hill=dict(repressor=1, K=2.0, n=2))])
    with pytest.raises(smc.SmcError):
        smc.Model.from_config(cfg)
    cfg = dict(base, reactions=[dict(rx([(0, 1)], [(1, 1)], 1.0), rate_expr="-S*2 - 3/P + 1")])
    m = smc.Model.from_config(cfg)
    src = m.kernel_source(smc.Property(m, cfg["formula"]))
    assert ("__dadd_rn(__dadd_rn(__dmul_rn((-(double)x[0]), 0x1p+1), -__ddiv_rn(0x1.8p+1, (double)x[1])), 0x1p+0)"
            in src)
    assert "if (x[0] < 1) return 0.0;" in src


def test_sweep_configuration_choices():
    """The automatic shape of the sweep kernel (DESIGN.md §5 knob table): C4 gets binary64
    columns in one 384-thread CTA per SM, groups of 7 laws read in one chunk and fused sums;
    a (64, 512) network groups of 18 read in chunks of 6; C5 (N = 200) the delta kernel with
    8-lane tiles, 32 groups of 32 laws and the per-event tables in global memory."""
    cfg = workloads.c4()
    m = smc.Model.from_config(cfg)
    src = m.kernel_source(smc.Property(m, cfg["formula"]))
    for d in ("#define SMC_BLOCK 384", "#define SMC_MINB 1", "#define SMC_SW_XD 1", "#define SMC_SW_S 7",
              "#define SMC_SW_C 7", "#define SMC_SW_FMAACC 1", "smc_ssa_sweep"):
        assert d in src, d
    net = workloads.random_network(11, 64, 512)
    cfg2 = dict(name="rn", species=net["species"], x0=net["x0"], reactions=net["reactions"],
                formula="F[0,1](S0 > 5)", t_max=0.0, seed=1, sampling=dict(mode="fixed", n=1))
    m2 = smc.Model.from_config(cfg2)
    src2 = m2.kernel_source(smc.Property(m2, cfg2["formula"]))
    assert "#define SMC_SW_S 18" in src2 and "#define SMC_SW_C 6" in src2 and "smc_ssa_sweep" in src2
    c5 = workloads.c5()
    m5 = smc.Model.from_config(c5)
    src5 = m5.kernel_source(smc.Property(m5, c5["formula"]))
    for d in ("smc_ssa_delta", "#define SMC_TW 8", "#define SMC_DG 32", "#define SMC_DS 32", "#define SMC_DGLOBAL 1",
              "#define SMC_DDEP16 1", "#define SMC_DDESC64 1"):
        assert d in src5, d


def test_property_of_another_model_and_event_cap_bounds():
    """a property compiled for a model with another species count is rejected by
    every run entry point before any device work; event caps stay within int32 (per-replica
    event counts are int32 on the device)."""
    m1 = smc.Model.from_config(workloads.c1())
    m2 = smc.Model.from_config(workloads.c2())
    p2 = smc.Property(m2, "F[0,50](P > 500)")
    with pytest.raises(smc.SmcError):
        m1.run(p2, 10, 1)
    with pytest.raises(smc.SmcError):
        smc.estimate(m1, p2, 0.99, 0.01, 1)
    with pytest.raises(smc.SmcError):
        m1.kernel_source(p2)
    with pytest.raises(smc.SmcError):
        m1.set_event_cap(2 ** 31)
    m1.set_event_cap(2 ** 31 - 1)


def test_window_ring_plan():
    """Ring plan of the window monitor (DESIGN R27; smc.h): capacity before residency."""
    GiB = 1 << 30
    pe, small, pc, grid = 48, 1024, 384, 148                 # C4's nested bench formula on the sweep kernel
    full = grid * pc * (32768 * pe + small)
    assert smc.smc_window_ring_plan(100 * GiB, pe, small, pc, grid) == (grid, 32768)       # fits: nothing given up
    assert full <= 100 * GiB
    g, cap = smc.smc_window_ring_plan(47 * GiB, pe, small, pc, grid)                       # the final pass's failure
    assert cap == 32768 and grid // 2 <= g < grid and g * pc * (cap * pe + small) <= 47 * GiB
    g, cap = smc.smc_window_ring_plan(20 * GiB, pe, small, pc, grid)                       # half the CTAs, then W halves
    assert g == grid // 2 and cap == 8192 and g * pc * (cap * pe + small) <= 20 * GiB
    g, cap = smc.smc_window_ring_plan(1 * GiB, pe, small, pc, grid)                        # W >= 1024 before residency
    assert cap == 1024 and 1 <= g < grid // 2 and g * pc * (cap * pe + small) <= 1 * GiB
    assert smc.smc_window_ring_plan(1 << 40, pe, small, pc, grid, 4096) == (grid, 4096)    # SMC_WIN_W
    assert smc.smc_window_ring_plan(100 * GiB, pe, small, 128, 8) == (8, 32768)            # small launches untouched
    g = np.random.default_rng(7)
    for _ in range(2000):                                    # invariants: within budget, power of two, never more CTAs
        b = int(g.integers(1 << 20, 1 << 38))
        pe_, sm_ = int(g.integers(8, 200)), int(g.integers(0, 4096))
        pc_, gr_ = int(g.integers(1, 1025)), int(g.integers(1, 600))
        want = int(2 ** g.integers(4, 16))
        try:
            go, cap = smc.smc_window_ring_plan(b, pe_, sm_, pc_, gr_, want)
        except smc.SmcError:
            assert b // pc_ < 16 * pe_ + sm_ + pe_               # only when one CTA cannot hold 16 entries per slot
            continue
        assert 1 <= go <= gr_ and 16 <= cap <= want and cap & (cap - 1) == 0
        assert go * pc_ * (cap * pe_ + sm_) <= b
        if go < gr_:                                         # CTAs were given up only for capacity
            assert (go + 1) * pc_ * (min(want, 1024) * pe_ + sm_) > b or go >= max(1, gr_ // 2)
    with pytest.raises(smc.SmcError):
        smc.smc_window_ring_plan(1 << 30, 0, 0, 128, 8)
