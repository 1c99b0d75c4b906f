"""ctypes wrapper around the C++ oracle (smc_oracle.cpp).  TEST INFRASTRUCTURE ONLY."""
import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "smc_oracle.cpp")
_LIB = os.path.join(_HERE, "libsmc_oracle.so")
_lock = threading.Lock()
_lib = None


def build_oracle(force=False):
    """Compile the oracle: plain -O2, no FMA contraction (reading R14)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + ".%d.tmp" % os.getpid()
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-fno-fast-math",
                               "-fPIC", "-shared", "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            L = ctypes.CDLL(build_oracle())
            c_u64, c_i64, c_i32, c_dp, c_vp = ctypes.c_uint64, ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p
            L.orc_last_error.restype = ctypes.c_char_p
            L.orc_philox.argtypes = [c_u64, c_u64, c_u64, c_vp]
            L.orc_philox_raw.argtypes = [c_vp, c_vp, c_vp]
            L.orc_uniforms.argtypes = [c_u64, c_u64, c_u64, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]
            L.orc_model_new.restype = c_vp
            L.orc_model_new.argtypes = [c_i32, c_vp, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp]
            L.orc_model_set_hill.argtypes = [c_vp, c_i32, c_i32, ctypes.c_double, c_i32]
            L.orc_model_set_rate.argtypes = [c_vp, c_i32, ctypes.c_char_p, c_vp]
            L.orc_model_free.argtypes = [c_vp]
            L.orc_propensity.restype = ctypes.c_double
            L.orc_propensity.argtypes = [c_vp, c_i32, c_vp]
            L.orc_formula_new.restype = c_vp
            L.orc_formula_new.argtypes = [ctypes.c_char_p, c_vp, c_i32, ctypes.c_double]
            L.orc_formula_free.argtypes = [c_vp]
            L.orc_formula_reach.restype = ctypes.c_double
            L.orc_formula_reach.argtypes = [c_vp]
            L.orc_formula_streamable.argtypes = [c_vp]
            L.orc_check_literal.argtypes = [c_vp, c_i64, c_vp, c_vp, c_vp, c_i32, c_i32]
            L.orc_check_streaming.argtypes = [c_vp, c_i64, c_vp, c_vp, c_vp, c_i32, c_i32, ctypes.POINTER(c_i64)]
            L.orc_run.argtypes = [c_vp, c_vp, c_u64, c_u64, c_u64, c_i32, c_i64, c_vp, c_vp, c_vp]
            L.orc_simulate.restype = c_i64
            L.orc_simulate.argtypes = [c_vp, c_u64, c_u64, ctypes.c_double, c_i64, c_vp, c_vp, c_vp, ctypes.POINTER(c_i32),
                                      ctypes.POINTER(c_i64)]
            _lib = L
    return _lib


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _err():
    return lib().orc_last_error().decode()


def philox(seed, traj, step):
    out = np.zeros(4, dtype=np.uint32)
    lib().orc_philox(seed, traj, step, _ptr(out))
    return [int(v) for v in out]


def philox_raw(ctr4, key2):
    c = np.asarray(ctr4, dtype=np.uint32)
    k = np.asarray(key2, dtype=np.uint32)
    out = np.zeros(4, dtype=np.uint32)
    lib().orc_philox_raw(_ptr(c), _ptr(k), _ptr(out))
    return [int(v) for v in out]


def uniforms(seed, traj, step):
    u1, u2 = ctypes.c_double(), ctypes.c_double()
    lib().orc_uniforms(seed, traj, step, ctypes.byref(u1), ctypes.byref(u2))
    return u1.value, u2.value


class OracleModel:
    """Reaction network.  cfg is a workloads/ config dict."""

    def __init__(self, cfg):
        self.cfg = cfg
        N = len(cfg["species"])
        M = len(cfg["reactions"])
        r_idx = np.full((M, 2), -1, np.int32)
        r_st = np.zeros((M, 2), np.int32)
        p_idx = np.full((M, 2), -1, np.int32)
        p_st = np.zeros((M, 2), np.int32)
        rate = np.zeros(M, np.float64)
        for j, r in enumerate(cfg["reactions"]):
            for q, (s, st) in enumerate(r["reactants"]):
                r_idx[j, q], r_st[j, q] = s, st
            for q, (s, st) in enumerate(r["products"]):
                p_idx[j, q], p_st[j, q] = s, st
            rate[j] = r["rate"]
        x0 = np.asarray(cfg["x0"], np.int64)
        self._keep = (x0, r_idx, r_st, p_idx, p_st, rate)
        self.h = lib().orc_model_new(N, _ptr(x0), M, _ptr(r_idx), _ptr(r_st), _ptr(p_idx), _ptr(p_st), _ptr(rate))
        if not self.h:
            raise ValueError(_err())
        for j, r in enumerate(cfg["reactions"]):
            if r.get("hill"):
                h = r["hill"]
                if lib().orc_model_set_hill(self.h, j, h["repressor"], float(h["K"]), int(h["n"])) != 0:
                    raise ValueError("bad hill parameters")
            if r.get("rate_expr"):
                names = (ctypes.c_char_p * N)(*[n.encode() for n in cfg["species"]])
                if lib().orc_model_set_rate(self.h, j, r["rate_expr"].encode(), ctypes.cast(names, ctypes.c_void_p)) != 0:
                    raise ValueError(_err())
        self.N, self.M = N, M

    def propensity(self, j, x):
        xa = np.asarray(x, np.int64)
        return lib().orc_propensity(self.h, j, _ptr(xa))

    def simulate(self, seed, traj, horizon, cap=1 << 20):
        """Full trace up to the first entry past `horizon` (not stored) or absorption."""
        t = np.zeros(cap, np.float64)
        tau = np.zeros(cap, np.float64)
        x = np.zeros((cap, self.N), np.int64)
        ab = ctypes.c_int32()
        ntau = ctypes.c_int64()
        n = lib().orc_simulate(self.h, seed, traj, horizon, cap, _ptr(t), _ptr(tau), _ptr(x), ctypes.byref(ab),
                               ctypes.byref(ntau))
        if n < 0:
            raise RuntimeError("simulation error / trace cap")
        return dict(t=t[:n].copy(), tau=tau[:ntau.value].copy(), x=x[:n].copy(), absorbed=bool(ab.value))

    def __del__(self):
        try:
            if self.h:
                lib().orc_model_free(self.h)
        except Exception:
            pass


class OracleFormula:
    def __init__(self, text, names, t_max=0.0):
        arr = (ctypes.c_char_p * len(names))(*[n.encode() for n in names])
        self._names = arr
        self.h = lib().orc_formula_new(text.encode(), ctypes.cast(arr, ctypes.c_void_p), len(names), float(t_max))
        if not self.h:
            raise ValueError(_err())
        self.text = text
        self.N = len(names)

    @property
    def reach(self):
        return lib().orc_formula_reach(self.h)

    @property
    def streamable(self):
        return bool(lib().orc_formula_streamable(self.h))

    def check_literal(self, t, tau, x, absorbed):
        t = np.ascontiguousarray(t, np.float64)
        tau = np.ascontiguousarray(tau, np.float64)
        x = np.ascontiguousarray(x, np.int64)
        return lib().orc_check_literal(self.h, len(t), _ptr(t), _ptr(tau), _ptr(x), self.N, int(absorbed))

    def check_streaming(self, t, tau, x, absorbed):
        t = np.ascontiguousarray(t, np.float64)
        tau = np.ascontiguousarray(tau, np.float64)
        x = np.ascontiguousarray(x, np.int64)
        at = ctypes.c_int64()
        v = lib().orc_check_streaming(self.h, len(t), _ptr(t), _ptr(tau), _ptr(x), self.N, int(absorbed), ctypes.byref(at))
        if v < 0:
            raise ValueError(_err())
        return v, at.value

    def __del__(self):
        try:
            if self.h:
                lib().orc_formula_free(self.h)
        except Exception:
            pass


def run(model, formula, seed, first, n, mode="stream", event_cap=(1 << 62), per_traj=True):
    """Replicas [first, first+n).  mode: 'stream' (on-the-fly) or 'literal'.
    Returns (counts dict, verdicts uint8[n] or None, events int64[n] or None)."""
    counts = np.zeros(4, np.int64)
    v = np.zeros(n, np.uint8) if per_traj else None
    e = np.zeros(n, np.int64) if per_traj else None
    rc = lib().orc_run(model.h, formula.h, seed, first, n, 0 if mode == "stream" else 1, event_cap,
                       _ptr(v) if per_traj else None, _ptr(e) if per_traj else None, _ptr(counts))
    if rc != 0:
        raise ValueError(_err())
    return dict(n_true=int(counts[0]), n_false=int(counts[1]), events=int(counts[2]), errors=int(counts[3])), v, e


def _worker(args):
    cfg, text, names, t_max, seed, first, n, mode = args
    m = OracleModel(cfg)
    f = OracleFormula(text, names, t_max)
    c, v, e = run(m, f, seed, first, n, mode)
    return c, v, e


def run_parallel(cfg, formula_text, seed, first, n, mode="stream", procs=None, chunk=None, t_max=0.0):
    """Run replicas over `procs` processes on disjoint index ranges; results in index order."""
    import concurrent.futures as cf
    import multiprocessing as mp
    procs = procs or os.cpu_count() or 1
    chunk = chunk or max(1, (n + procs * 4 - 1) // (procs * 4))
    tasks = []
    s = first
    while s < first + n:
        m = min(chunk, first + n - s)
        tasks.append((cfg, formula_text, cfg["species"], t_max, seed, s, m, mode))
        s += m
    build_oracle()
    # forkserver: workers are forked from a fresh single-threaded server, never from a
    # process that already holds CUDA / torch threads
    ctx = mp.get_context("forkserver")
    with cf.ProcessPoolExecutor(max_workers=procs, mp_context=ctx) as ex:
        res = list(ex.map(_worker, tasks))
    tot = dict(n_true=0, n_false=0, events=0, errors=0)
    vs, es = [], []
    for c, v, e in res:
        for k in tot:
            tot[k] += c[k]
        vs.append(v)
        es.append(e)
    return tot, np.concatenate(vs), np.concatenate(es)
