"""Every generated kernel compiles for sm_100a with the same NVRTC library and options
the GPU box uses (scripts/check_codegen.py), without a GPU: thread, tile (every tile
width), sweep and literal variants for the benchmark configs and the feature workloads."""
import os
import sys

import pytest

import workloads
import paper_0912_2551_b200 as smc

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "scripts"))
from check_codegen import nvrtc_cubin  # noqa: E402

CASES = [("C1", 1), ("C1", 4), ("C2", 1), ("C2", 2), ("C2", 4), ("C3", 1), ("C3", 2), ("C3", 4), ("C4", 2), ("C4", 4),
         ("C5", 2), ("C5", 4), ("C5", 5), ("C4", 5), ("C2", 5), ("EXPL", 1), ("EXPL", 2), ("EXPL", 4), ("CC", 1), ("CC", 2), ("CC", 4)]


def _compile(cfg, variant, formula=None, t_max=0.0):
    m = smc.Model.from_config(cfg)
    if variant:
        m.set_variant(variant)
    p = smc.Property(m, formula or cfg["formula"], t_max=t_max or cfg.get("t_max", 0.0))
    src = m.kernel_source(p)
    cubin, log = nvrtc_cubin(src, "gen_%s_v%d.cu" % (cfg["name"], variant))
    assert len(cubin) > 1000
    return src, log


@pytest.mark.parametrize("name,variant", CASES)
def test_generated_kernel_compiles(name, variant):
    _compile(workloads.get(name), variant)


@pytest.mark.parametrize("width", ["4", "8", "16", "32"])
def test_tile_widths_compile(width, monkeypatch):
    monkeypatch.setenv("SMC_TILE_WIDTH", width)
    _compile(workloads.c4(), 2)


def test_literal_variant_compiles():
    src, _ = _compile(workloads.c2(), 0, "F[0,5](G[1,2](P > 5) & X[0,1](ES < sqrt(S)))")
    assert "smc_ssa_literal" in src
    src, _ = _compile(workloads.c2(), 0, "G(E + ES == 100) & F(0,2](G[0.5,1](P > 3))", t_max=10.0)
    assert "smc_ssa_literal" in src


def test_window_monitor_compiles_in_tile_and_sweep():
    """The window monitor (R27) in the sweep kernel (C4's default for nested formulas) and in
    the tile kernel (forced variant 2, and the delta kernel's models)."""
    f = "F[0,0.3](S0 < S1 + 3 & G[0.01,0.04](S0 < S1 + 3))"
    src, _ = _compile(workloads.c4(), 0, f)
    assert "smc_ssa_sweep" in src and "struct SmcMon" in src and "SmcWN<" in src
    src, _ = _compile(workloads.c4(), 2, f)
    assert "smc_ssa_tile" in src and "struct SmcMon" in src and "SmcWN<" in src
    src, _ = _compile(workloads.c5(), 0, f)
    assert "smc_ssa_tile" in src and "struct SmcMon" in src
