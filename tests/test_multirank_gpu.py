"""N > 1 through the C ABI on the device path: two ranks (two
processes) share the one GPU of this box, each runs ITS slice of every round with its own
persistent kernel, and the int64[4] counts are summed by the allreduce hook on a DEVICE
pointer (set_allreduce_torch(device=True); gloo's CUDA all_reduce stands in for NCCL, which
needs one GPU per rank).  The ranks' kernels never wait on each other: only the 32-byte
reduction is shared.  smc_run and smc_estimate (speculation on: the host round loop with a
speculative batch sized from the allreduced capacity) must equal the 1-rank results bit for bit.
"""
import os
import socket

import pytest
import torch.multiprocessing as mp

import workloads

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _work(smc, cfg, n_run, conf, eps):
    m = smc.Model.from_config(cfg)
    p = smc.Property(m, cfg["formula"], t_max=cfg.get("t_max", 0.0))
    c = m.run(p, n_run, cfg["seed"])
    c2 = m.run(p, n_run // 3, cfg["seed"])            # the cursor continues: the next slice
    est = smc.estimate(m, p, conf, eps, cfg["seed"])
    return dict(run=c, run2=c2, est={k: est[k] for k in ("p_hat", "lower", "upper", "n_total", "n_true", "rounds",
                                                           "events", "errors")})


CASES = [("C2", 30_000, 0.99, 0.01), ("C4", 600, 0.95, 0.05)]


def _rank_main(rank, world, port, out):
    import torch
    import torch.distributed as dist

    import paper_0912_2551_b200 as smc
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    smc.use_torch()
    smc.set_allreduce_torch(device=True)
    res = {}
    for name, n, conf, eps in CASES:
        res[name] = _work(smc, workloads.get(name), n, conf, eps)
    out[rank] = res
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_on_device_equal_one(smc):
    ref = {name: _work(smc, workloads.get(name), n, conf, eps) for name, n, conf, eps in CASES}
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.start_processes(_rank_main, args=(world, _free_port(), out), nprocs=world, join=True, start_method="spawn")
    for r in range(world):
        for name, *_ in CASES:
            assert out[r][name] == ref[name], (r, name, out[r][name], ref[name])


def _nccl_rank_main(rank, world, port, out):
    import torch
    import torch.distributed as dist

    import paper_0912_2551_b200 as smc
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", 0))
    smc.use_torch()
    smc.set_allreduce_torch(device=True)            # the hook bench.py installs at N > 1
    res = {}
    for name, n, conf, eps in CASES:
        res[name] = _work(smc, workloads.get(name), n, conf, eps)
    out[rank] = res
    dist.barrier()
    dist.destroy_process_group()


def test_nccl_hook_one_rank_equals_no_hook(smc):
    """The device-pointer allreduce through NCCL itself (one rank: the only NCCL group one GPU
    can hold): every round's int64[4] counts go through ncclAllReduce on the device pointer
    and the results equal the hook-less run bit for bit."""
    ref = {name: _work(smc, workloads.get(name), n, conf, eps) for name, n, conf, eps in CASES}
    mgr = mp.Manager()
    out = mgr.dict()
    mp.start_processes(_nccl_rank_main, args=(1, _free_port(), out), nprocs=1, join=True, start_method="spawn")
    for name, *_ in CASES:
        assert out[0][name] == ref[name], (name, out[0][name], ref[name])
