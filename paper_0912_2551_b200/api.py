"""Object wrappers over the C ABI (marshalling only) and the PyTorch hooks.

Model      -> smc_model_create / smc_model_set_hill / set_variant / set_event_cap
Property   -> smc_property_compile
Model.run  -> smc_run            estimate -> smc_estimate (Fig. 2)
use_torch  -> smc_set_allocator + smc_set_stream (torch caching allocator, current stream)
set_allreduce_torch -> smc_set_allreduce (torch.distributed all_reduce, NCCL on GPU / gloo on CPU)
"""
import ctypes

import numpy as np

from ._native import (ALLOC_FN, ALLREDUCE_FN, FREE_FN, RUN_FN, SmcCounts, SmcEstimate, SmcLaunchInfo, c_sz, c_vp,
                      check, lib)

COUNTS_KEYS = ("n_true", "n_false", "events", "errors")


def _ptr(a):
    return a.ctypes.data_as(c_vp)


def _counts(c):
    return {k: int(getattr(c, k)) for k in COUNTS_KEYS}


class Model:
    """A reaction network: species counts x0, reactions with
    reactants/products [(species, stoichiometry)], mass-action rates and
    optional Hill repression."""

    def __init__(self, species, x0, reactions):
        self.species = list(species)
        N, M = len(species), len(reactions)
        r_idx = np.full((M, 2), -1, np.int32)
        r_st = np.zeros((M, 2), np.int32)
        p_idx = np.full((M, 2), -1, np.int32)
        p_st = np.zeros((M, 2), np.int32)
        rate = np.zeros(M, np.float64)
        for j, r in enumerate(reactions):
            for q, (s, st) in enumerate(r["reactants"]):
                r_idx[j, q], r_st[j, q] = s, st
            for q, (s, st) in enumerate(r["products"]):
                p_idx[j, q], p_st[j, q] = s, st
            rate[j] = r["rate"]
        x = np.asarray(x0, np.int32)
        h = c_vp()
        check(lib().smc_model_create(N, _ptr(x), M, _ptr(r_idx), _ptr(r_st), _ptr(p_idx), _ptr(p_st), _ptr(rate),
                                     ctypes.byref(h)))
        self.h = h
        self.N, self.M = N, M
        names = None
        for j, r in enumerate(reactions):
            hl = r.get("hill")
            if hl:
                check(lib().smc_model_set_hill(self.h, j, int(hl["repressor"]), float(hl["K"]), int(hl["n"])))
            if r.get("rate_expr"):
                if names is None:
                    names = (ctypes.c_char_p * N)(*[str(n).encode() for n in self.species])
                check(lib().smc_model_set_rate_expr(self.h, j, r["rate_expr"].encode(), ctypes.cast(names, c_vp)))

    @classmethod
    def from_config(cls, cfg):
        return cls(cfg["species"], cfg["x0"], cfg["reactions"])

    def set_variant(self, v):
        check(lib().smc_model_set_variant(self.h, v))

    def set_event_cap(self, cap):
        check(lib().smc_model_set_event_cap(self.h, cap))

    def set_speculation(self, on):
        check(lib().smc_model_set_speculation(self.h, 1 if on else 0))

    def reset(self):
        check(lib().smc_reset(self.h))

    def set_cursor(self, cursor, seed):
        """Resume: the next run(prop, n, seed) covers trajectories [cursor, cursor + n)."""
        check(lib().smc_set_cursor(self.h, cursor, seed))

    def run(self, prop, n, seed):
        c = SmcCounts()
        check(lib().smc_run(self.h, prop.h, n, seed, ctypes.byref(c)))
        return _counts(c)

    def run_verdicts(self, prop, first, n, seed):
        """Per-replica verdicts (uint8) and event counts (int32) as CUDA tensors."""
        import torch
        v = torch.empty(max(n, 1), dtype=torch.uint8, device="cuda")
        e = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
        check(lib().smc_run_verdicts(self.h, prop.h, first, n, seed, c_vp(v.data_ptr()), c_vp(e.data_ptr())))
        return v[:n], e[:n]

    def last_launch(self, prop):
        info = SmcLaunchInfo()
        check(lib().smc_last_launch(self.h, prop.h, ctypes.byref(info)))
        return {f: getattr(info, f) for f, _ in SmcLaunchInfo._fields_}

    def kernel_source(self, prop):
        n = c_sz(0)
        check(lib().smc_kernel_source(self.h, prop.h, None, ctypes.byref(n)))
        buf = ctypes.create_string_buffer(n.value)
        check(lib().smc_kernel_source(self.h, prop.h, buf, ctypes.byref(n)))
        return buf.value.decode()

    def __del__(self):
        try:
            if getattr(self, "h", None):
                lib().smc_model_destroy(self.h)
                self.h = None
        except Exception:
            pass


class Property:
    """A BLTLc formula compiled to a monitor program for `model`."""

    def __init__(self, model, formula, names=None, t_max=0.0):
        names = model.species if names is None else names
        arr = (ctypes.c_char_p * len(names))(*[s.encode() for s in names])
        h = c_vp()
        check(lib().smc_property_compile(model.h, formula.encode(), ctypes.cast(arr, c_vp), float(t_max),
                                         ctypes.byref(h)))
        self.h = h
        self.formula = formula
        self.model = model

    def __del__(self):
        try:
            if getattr(self, "h", None):
                lib().smc_property_destroy(self.h)
                self.h = None
        except Exception:
            pass


def _est(e):
    return dict(p_hat=e.p_hat, lower=e.lower, upper=e.upper, n_total=int(e.n_total), n_true=int(e.n_true),
                events=int(e.events), errors=int(e.errors), rounds=int(e.rounds), z=e.z)


def estimate(model, prop, confidence, half_width, seed, start=1.0):
    """Fig. 2 Wilson estimate: start=1.0 iterative (smc_estimate), 0.5 conservative
    (smc_estimate_ex)."""
    e = SmcEstimate()
    if start == 1.0:
        check(lib().smc_estimate(model.h, prop.h, confidence, half_width, seed, ctypes.byref(e)))
    else:
        check(lib().smc_estimate_ex(model.h, prop.h, confidence, half_width, start, seed, ctypes.byref(e)))
    return _est(e)


def estimate_with_runner(run_fn, confidence, half_width, start=1.0):
    """smc_estimate_with_runner: run_fn(first, n) -> dict of local counts for this rank's slice."""
    def cb(first, n, user, out):
        try:
            c = run_fn(int(first), int(n))
            out.contents.n_true, out.contents.n_false = c["n_true"], c["n_false"]
            out.contents.events, out.contents.errors = c["events"], c["errors"]
            return 0
        except Exception:      # reported as a runner failure by the library
            import traceback
            traceback.print_exc()
            return 1
    fn = RUN_FN(cb)
    e = SmcEstimate()
    check(lib().smc_estimate_with_runner(fn, None, confidence, half_width, start, ctypes.byref(e)))
    return _est(e)


# ---------------------------------------------------------------- PyTorch ---
_keep = []


def use_torch(allocator=True, stream=True):
    """Route libsmc's device memory through the torch caching allocator and its
    launches onto torch's current CUDA stream."""
    import torch
    if allocator:
        big = {}                    # blocks of >= 1 GiB (the window monitor's rings)

        def alloc(size, user):
            try:
                ptr = torch.cuda.caching_allocator_alloc(int(size), device=torch.cuda.current_device(),
                                                         stream=torch.cuda.current_stream())
                if int(size) >= (1 << 30):
                    big[int(ptr)] = int(size)
                return ptr
            except Exception:
                import traceback
                traceback.print_exc()
                return 0            # NULL -> SMC_E_CUDA "allocator hook returned NULL"

        def free(ptr, user):
            if ptr and torch is not None and getattr(torch, "cuda", None) is not None:   # not at interpreter exit
                torch.cuda.caching_allocator_delete(int(ptr))
                # the library sizes the rings from cudaMemGetInfo, which does not see blocks
                # cached by torch: hand a freed ring back to the driver
                if big.pop(int(ptr), None):
                    torch.cuda.empty_cache()
        a, f = ALLOC_FN(alloc), FREE_FN(free)
        _keep.extend([a, f])
        check(lib().smc_set_allocator(a, f, None))
    if stream:
        check(lib().smc_set_stream(c_vp(torch.cuda.current_stream().cuda_stream)))


class _CudaArray:
    def __init__(self, ptr, n):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<i8", "data": (ptr, False), "version": 3,
                                         "strides": None, "stream": None}


def set_allreduce_torch(group=None, device=True):
    """Sum the per-round counts over the ranks of a torch.distributed group.
    device=True: the library passes a DEVICE pointer (smc_run / smc_estimate, NCCL);
    device=False: a HOST pointer (smc_estimate_with_runner, e.g. gloo on CPU)."""
    import torch
    import torch.distributed as dist

    def hook(ptr, n, user):
        try:
            addr = ctypes.cast(ptr, c_vp).value
            if device:
                t = torch.as_tensor(_CudaArray(addr, n), device="cuda")
            else:
                arr = np.ctypeslib.as_array((ctypes.c_int64 * n).from_address(addr))
                t = torch.from_numpy(arr)
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
            return 0
        except Exception:
            import traceback
            traceback.print_exc()
            return 1
    fn = ALLREDUCE_FN(hook)
    _keep.append(fn)
    check(lib().smc_set_allreduce(fn, None))
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    check(lib().smc_set_shard(rank, world))


def clear_allreduce():
    check(lib().smc_set_allreduce(ALLREDUCE_FN(), None))
    check(lib().smc_set_shard(0, 1))
