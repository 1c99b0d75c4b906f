"""ctypes declarations of include/smc.h (one Python name per C entry point)."""
import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libsmc.so")
_lock = threading.Lock()
_lib = None

c_i32, c_i64, c_u32, c_u64, c_vp, c_dbl, c_sz = (ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32, ctypes.c_uint64,
                                                  ctypes.c_void_p, ctypes.c_double, ctypes.c_size_t)


class SmcCounts(ctypes.Structure):
    _fields_ = [("n_true", c_i64), ("n_false", c_i64), ("events", c_i64), ("errors", c_i64)]


class SmcEstimate(ctypes.Structure):
    _fields_ = [("p_hat", c_dbl), ("lower", c_dbl), ("upper", c_dbl), ("n_total", c_i64), ("n_true", c_i64),
                ("events", c_i64), ("errors", c_i64), ("rounds", c_i32), ("z", c_dbl)]


class SmcLaunchInfo(ctypes.Structure):
    _fields_ = [("variant", c_i32), ("block_threads", c_i32), ("grid_blocks", c_i32), ("smem_bytes", c_i32),
                ("regs_per_thread", c_i32), ("launches", c_i32), ("kernel_ms", ctypes.c_float),
                ("compile_ms", ctypes.c_float), ("table_bytes", c_dbl), ("aux_launches", c_i32), ("pad_", c_i32),
                ("sim_events", c_dbl)]


RUN_FN = ctypes.CFUNCTYPE(c_i32, c_u64, c_u64, c_vp, ctypes.POINTER(SmcCounts))
ALLREDUCE_FN = ctypes.CFUNCTYPE(c_i32, ctypes.POINTER(c_i64), c_i32, c_vp)
ALLOC_FN = ctypes.CFUNCTYPE(c_vp, c_sz, c_vp)
FREE_FN = ctypes.CFUNCTYPE(None, c_vp, c_vp)

# (name, restype, argtypes) -- the exported symbols of include/smc.h
SIGNATURES = [
    ("smc_last_error", ctypes.c_char_p, []),
    ("smc_model_create", c_i32, [c_i32, c_vp, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, ctypes.POINTER(c_vp)]),
    ("smc_model_set_hill", c_i32, [c_vp, c_i32, c_i32, c_dbl, c_i32]),
    ("smc_model_set_variant", c_i32, [c_vp, c_i32]),
    ("smc_model_set_event_cap", c_i32, [c_vp, c_u64]),
    ("smc_model_set_speculation", c_i32, [c_vp, c_i32]),
    ("smc_model_destroy", None, [c_vp]),
    ("smc_property_compile", c_i32, [c_vp, ctypes.c_char_p, c_vp, c_dbl, ctypes.POINTER(c_vp)]),
    ("smc_property_destroy", None, [c_vp]),
    ("smc_run", c_i32, [c_vp, c_vp, c_u64, c_u64, ctypes.POINTER(SmcCounts)]),
    ("smc_reset", c_i32, [c_vp]),
    ("smc_set_cursor", c_i32, [c_vp, c_u64, c_u64]),
    ("smc_estimate", c_i32, [c_vp, c_vp, c_dbl, c_dbl, c_u64, ctypes.POINTER(SmcEstimate)]),
    ("smc_estimate_ex", c_i32, [c_vp, c_vp, c_dbl, c_dbl, c_dbl, c_u64, ctypes.POINTER(SmcEstimate)]),
    ("smc_estimate_with_runner", c_i32, [RUN_FN, c_vp, c_dbl, c_dbl, c_dbl, ctypes.POINTER(SmcEstimate)]),
    ("smc_normal_quantile", c_dbl, [c_dbl]),
    ("smc_wilson_interval", c_i32, [c_i64, c_i64, c_dbl, ctypes.POINTER(c_dbl), ctypes.POINTER(c_dbl)]),
    ("smc_wilson_sample_size", c_i64, [c_dbl, c_dbl, c_dbl]),
    ("smc_shard_range", c_i32, [c_u64, c_u64, c_i32, c_i32, ctypes.POINTER(c_u64), ctypes.POINTER(c_u64)]),
    ("smc_window_ring_plan", c_i32, [c_u64, c_u64, c_u64, c_i32, c_i32, c_u64, ctypes.POINTER(c_i32),
                                     ctypes.POINTER(c_u64)]),
    ("smc_set_allocator", c_i32, [ALLOC_FN, FREE_FN, c_vp]),
    ("smc_set_stream", c_i32, [c_vp]),
    ("smc_set_shard", c_i32, [c_i32, c_i32]),
    ("smc_set_allreduce", c_i32, [ALLREDUCE_FN, c_vp]),
    ("smc_run_verdicts", c_i32, [c_vp, c_vp, c_u64, c_u64, c_u64, c_vp, c_vp]),
    ("smc_model_set_rate_expr", c_i32, [c_vp, c_i32, ctypes.c_char_p, c_vp]),
    ("smc_philox_blocks", c_i32, [c_u64, c_u64, c_u64, c_u32, c_vp]),
    ("smc_draw_blocks", c_i32, [c_u64, c_u64, c_u64, c_u32, c_vp]),
    ("smc_last_launch", c_i32, [c_vp, c_vp, ctypes.POINTER(SmcLaunchInfo)]),
    ("smc_kernel_source", c_i32, [c_vp, c_vp, ctypes.c_char_p, ctypes.POINTER(c_sz)]),
]

ERRORS = {0: "SMC_OK", -1: "SMC_E_ARG", -2: "SMC_E_MODEL", -3: "SMC_E_PARSE", -4: "SMC_E_UNSUPPORTED",
          -5: "SMC_E_CUDA", -6: "SMC_E_COMM", -7: "SMC_E_OVERFLOW", -8: "SMC_E_EVENT_CAP", -9: "SMC_E_ERRRATE"}


class SmcError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__("%s (%d): %s" % (ERRORS.get(code, "?"), code, msg))
        self.code = code
        self.name = ERRORS.get(code, "?")


def lib():
    """Load libsmc.so (building it in-tree first if it is missing or stale)."""
    global _lib
    with _lock:
        if _lib is None:
            from . import build as _build
            if _build.needs_build():
                _build.build()
            if not os.path.exists(_LIB_PATH):
                raise ImportError("libsmc.so is missing and could not be built: " + _LIB_PATH)
            L = ctypes.CDLL(_LIB_PATH)
            for name, res, args in SIGNATURES:
                fn = getattr(L, name)
                fn.restype = res
                fn.argtypes = args
            _lib = L
    return _lib


def smc_last_error():
    return lib().smc_last_error().decode(errors="replace")


def check(rc):
    if rc != 0:
        raise SmcError(rc, smc_last_error())
    return rc


def smc_normal_quantile(confidence):
    return lib().smc_normal_quantile(confidence)


def smc_wilson_interval(n_true, n, confidence):
    lo, hi = c_dbl(), c_dbl()
    check(lib().smc_wilson_interval(n_true, n, confidence, ctypes.byref(lo), ctypes.byref(hi)))
    return lo.value, hi.value


def smc_wilson_sample_size(p, half_width, confidence):
    v = lib().smc_wilson_sample_size(p, half_width, confidence)
    if v < 0:
        raise SmcError(-1, smc_last_error())
    return v


def smc_shard_range(base, n, rank, world):
    lo, hi = c_u64(), c_u64()
    check(lib().smc_shard_range(base, n, rank, world, ctypes.byref(lo), ctypes.byref(hi)))
    return lo.value, hi.value


def smc_window_ring_plan(budget_bytes, per_entry, small, per_cta, grid, want=32768):
    g, cap = c_i32(), c_u64()
    check(lib().smc_window_ring_plan(budget_bytes, per_entry, small, per_cta, grid, want, ctypes.byref(g),
                                     ctypes.byref(cap)))
    return g.value, cap.value


def smc_philox_blocks(seed, trajectory, step0, n):
    buf = (c_u32 * (4 * n))()
    check(lib().smc_philox_blocks(seed, trajectory, step0, n, ctypes.cast(buf, c_vp)))
    return [[buf[4 * q + i] for i in range(4)] for q in range(n)]


def smc_draw_blocks(seed, trajectory, step0, n):
    """[(e, u2)] of steps step0 .. step0+n-1 from the device draw (e = -log(u1))."""
    buf = (ctypes.c_double * (2 * n))()
    check(lib().smc_draw_blocks(seed, trajectory, step0, n, ctypes.cast(buf, c_vp)))
    return [(buf[2 * q], buf[2 * q + 1]) for q in range(n)]


def smc_set_shard(rank, world):
    check(lib().smc_set_shard(rank, world))


def smc_set_stream(stream_handle):
    check(lib().smc_set_stream(stream_handle))
