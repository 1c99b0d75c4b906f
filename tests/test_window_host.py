"""The window monitor (paper_0912_2551_b200/csrc/kernels/ssa_window.cuh + the node table the
codegen emits for a property; readings R23/R24/R27) compiled for the HOST and driven with
oracle-simulated traces exactly as the kernels drive it (enter / advance / absorb / event
cap), against the oracle's literal mode (the three-valued |= of P:229-237 and the exact
first decision index of P:291-294).  No GPU: this checks the monitor's logic -- the
(value, first-decision-index) algebra, the per-position windows, the rings -- on the same
code the kernels compile, replica for replica, on formulas of every operator shape.

The oracle is only the checker here (it simulates the traces and judges them)."""
import ctypes
import os
import re
import subprocess
import tempfile

import numpy as np
import pytest

import workloads
import paper_0912_2551_b200 as smc
from oracle import oracle as O

SHIM = r"""
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <vector>
#define __device__
#define __forceinline__ inline
typedef unsigned long long smc_u64;
typedef long long smc_i64;
typedef unsigned int smc_u32;
struct SmcDim { unsigned x; };
static SmcDim threadIdx = {0};
static inline int __popc(unsigned v) { return __builtin_popcount(v); }
static inline void __syncwarp(unsigned) {}
static inline double __dadd_rn(double a, double b) { return a + b; }
static inline double __dsub_rn(double a, double b) { return a - b; }
static inline double __dmul_rn(double a, double b) { return a * b; }
static inline double __ddiv_rn(double a, double b) { return a / b; }
static inline double __dsqrt_rn(double a) { return std::sqrt(a); }
static inline double __fma_rn(double a, double b, double c) { return std::fma(a, b, c); }
using std::max;
using std::min;
struct SmcParams { double* lit_t; smc_u64 lit_cap; };
struct int2 { int x, y; };
static inline int2 make_int2(int a, int b) { return int2{a, b}; }
"""

DRIVER = r"""
static std::vector<char> g_buf;
extern "C" int win_check(const double* t, const double* tau, const long long* x, int N, long long ne, int absorbed,
                         long long W, long long cap, long long* events) {
    SmcParams P;
    g_buf.assign((size_t)W * SMC_WIN_PER_ENTRY + SMC_WIN_SMALL, 0);
    P.lit_t = (double*)g_buf.data();
    P.lit_cap = (smc_u64)W;
    SmcMon mon;
    mon.bind(P, 0, 1u, 0);
    mon.init();
    std::vector<int> xs((size_t)N);
    for (int s = 0; s < N; ++s) xs[(size_t)s] = (int)x[s];
    mon.enter(0u, t[0], 0.0, xs.data());
    long long k = 0;
    int v = -1;
    for (;;) {
        if (k == ne - 1 && absorbed) { mon.absorb(); v = mon.verdict(); break; }
        const double tn = t[k] + tau[k];
        mon.advance((smc_u32)k, tn, tau[k]);
        v = mon.verdict();
        if (v >= 0) break;
        if (k + 1 >= ne) { v = -2; break; }
        ++k;
        for (int s = 0; s < N; ++s) xs[(size_t)s] = (int)x[k * N + s];
        mon.enter((smc_u32)k, t[k], t[k - 1], xs.data());
        if (k >= cap) { v = mon.at_cap(k); break; }
    }
    *events = (v == 0 || v == 1) ? mon.events(k) : k;
    return v;
}
"""


def build_host_monitor(src, tmp):
    """Extract the window monitor (node table + ssa_window.cuh) from a generated kernel
    source and compile it for the host with the shim above."""
    h = re.search(r"#define SMC_LIT_H [^\n]*\n", src).group(0)
    a = src.index("template <class XA> __device__ __forceinline__ unsigned smc_lit_mask")
    b = src.index("struct SmcMon {")
    b = src.index("\n};\n", b) + 4
    code = SHIM + h + src[a:b] + DRIVER
    cpp = os.path.join(tmp, "win.cpp")
    so = os.path.join(tmp, "win.so")
    open(cpp, "w").write(code)
    subprocess.run(["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-shared", "-fPIC", "-o", so, cpp], check=True,
                   capture_output=True)
    L = ctypes.CDLL(so)
    L.win_check.restype = ctypes.c_int
    L.win_check.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int, ctypes.c_longlong, ctypes.c_int, ctypes.c_longlong,
                                                     ctypes.c_longlong, ctypes.POINTER(ctypes.c_longlong)]
    return L


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def check(cfg, formula, n, t_max=0.0, W=4096, cap=None, first=0):
    """Replicas [first, first+n) of cfg: host window monitor vs oracle literal mode."""
    m = smc.Model.from_config(cfg)
    p = smc.Property(m, formula, t_max=t_max)
    src = m.kernel_source(p)
    assert "struct SmcMon" in src, "formula inside the streaming templates"
    om = O.OracleModel(cfg)
    of = O.OracleFormula(formula, cfg["species"], t_max)
    H = t_max if t_max > 0 else of.reach
    ecap = cap if cap is not None else (1 << 62)
    _, ov, oe = O.run(om, of, cfg["seed"], first, n, mode="literal", event_cap=ecap)
    with tempfile.TemporaryDirectory() as tmp:
        L = build_host_monitor(src, tmp)
        bad = []
        for q in range(n):
            tr = om.simulate(cfg["seed"], first + q, H, cap=1 << 21)
            t = np.ascontiguousarray(tr["t"])
            tau = np.ascontiguousarray(tr["tau"])
            x = np.ascontiguousarray(tr["x"])
            ev = ctypes.c_longlong()
            v = L.win_check(_p(t), _p(tau), _p(x), x.shape[1], len(t), int(tr["absorbed"]), W,
                            cap if cap is not None else (1 << 62), ctypes.byref(ev))
            if v != ov[q] or ev.value != oe[q]:
                bad.append((first + q, v, int(ov[q]), ev.value, int(oe[q])))
    return bad, ov, oe


FORMULAS_C2 = [
    "F[1,50](G[0,5](P > 100))",
    "G[0,40](F[1,5](ES > 10))",
    "F[0,20](ES > 20 & X[0,0.1](ES < 20))",
    "(E > 60) U[0,30] (G[0,3](P > 50))",
    "!(F[0,10](G[2,4](S < 900)) | G[0,15](E > 20))",
    "F[2,30](F[0,1](P > 20) & G[0,2](ES >= 1))",
    "G[0,20](ES < 40 | F[0.5,1](ES < 30))",
    "X[0,1](F[0,10](P > 30))",
    "F(0,30](G[1,2)(P > 40))",
]


@pytest.mark.parametrize("formula", FORMULAS_C2)
def test_window_monitor_vs_oracle_literal_c2(formula):
    bad, ov, _ = check(workloads.c2(), formula, 60)
    assert not bad, bad[:5]
    assert len(set(ov.tolist())) >= 1


def test_window_monitor_c3_bench_formula():
    """The bench's nested C3 formula at C3's full horizon (G over 290 time units)."""
    bad, ov, oe = check(workloads.c3(), "G[0,290](F[1,10](P1 < 400))", 12)
    assert not bad, bad
    assert oe.max() > 4096                 # traces far longer than the ring: memory is the window


def test_window_monitor_small_rings_fail_loudly():
    """A window spanning more entries than the ring ends the replica as an error (never a
    wrong verdict)."""
    bad, ov, oe = check(workloads.c2(), "G[0,40](F[1,5](ES > 10))", 10, W=16)
    assert bad and all(b[1] == 2 for b in bad)


def test_window_monitor_event_cap():
    """Event cap: the prefix up to the cap decides (same first index), else an error."""
    bad, ov, oe = check(workloads.c2(), "G[0,40](F[1,5](ES > 10))", 20, cap=300)
    assert not bad, bad[:5]
    assert (ov == 2).any() or (oe <= 300).all()


def test_window_monitor_unbounded_with_tmax():
    bad, _, _ = check(workloads.c2(), "G(E + ES == 100) & F(0,2](G[0.5,1](P > 3))", 30, t_max=10.0)
    assert not bad, bad[:5]


def _random_nested(g, sp, depth=0):
    """A random BLTL formula with nested temporal operators, open / closed
    bounds and non-zero lower bounds."""
    if depth >= 3 or g.random() < 0.25:
        s = sp[int(g.integers(0, len(sp)))]
        op = ["<", "<=", ">", ">=", "==", "!="][int(g.integers(0, 6))]
        return "%s %s %d" % (s, op, int(g.integers(0, 8)))
    k = int(g.integers(0, 7))
    sub = lambda: _random_nested(g, sp, depth + 1)  # noqa: E731
    lo = float(g.choice([0.0, 0.0, 0.1, 0.5]))
    hi = lo + float(g.choice([0.2, 0.5, 1.0, 2.0]))
    lb = "(" if g.random() < 0.2 else "["
    rb = ")" if g.random() < 0.2 else "]"
    I = "%s%r,%r%s" % (lb, lo, hi, rb)
    if k == 0:
        return "F%s(%s)" % (I, sub())
    if k == 1:
        return "G%s(%s)" % (I, sub())
    if k == 2:
        return "(%s) U%s (%s)" % (sub(), I, sub())
    if k == 3:
        return "X%s(%s)" % (I, sub())
    if k == 4:
        return "!(%s)" % sub()
    if k == 5:
        return "(%s) & (%s)" % (sub(), sub())
    return "(%s) | (%s)" % (sub(), sub())


def _fuzz_case(seed):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from test_gpu_parity import _random_case
    cfg = _random_case(seed)
    g = np.random.default_rng(5000 + seed)
    for _ in range(50):
        f = _random_nested(g, cfg["species"])
        of = O.OracleFormula(f, cfg["species"])
        if not of.streamable and of.reach > 0:
            return cfg, f
    return cfg, "F[0.1,1](G[0,0.5](%s >= 1))" % cfg["species"][0]


@pytest.mark.parametrize("seed", range(40))
def test_window_monitor_random_nested_formulas(seed):
    """Fuzz: random networks x random nested formulas, 150 replicas each: verdict and the
    exact first decision index equal the oracle's literal mode for every replica."""
    cfg, f = _fuzz_case(seed)
    bad, ov, oe = check(cfg, f, 150)
    assert not bad, (f, bad[:5])
