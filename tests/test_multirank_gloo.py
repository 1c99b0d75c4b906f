"""N > 1 path on CPU: two ranks (torch.distributed gloo, world_size 2) shard each
Wilson round with smc_shard_range, sum the counts with the allreduce hook and
run the identical Fig. 2 step; the result must equal the single-process run
(SPEC S:419 worker-count invariance)."""
import os
import socket

import pytest
import torch.multiprocessing as mp

import workloads
from oracle import wilson_procedure
from oracle import oracle as O


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_main(rank, world, port, out):
    import torch.distributed as dist

    import paper_0912_2551_b200 as smc
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = workloads.c1()
    om = O.OracleModel(cfg)
    of = O.OracleFormula(cfg["formula"], cfg["species"])
    slices = []

    def run(first, n):
        slices.append((first, n))
        c, _, _ = O.run(om, of, 5, first, n, per_traj=False)
        return c
    smc.set_allreduce_torch(device=False)
    est = smc.estimate_with_runner(run, 0.99, 0.005)
    out[rank] = (est, slices)
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_equal_one():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.start_processes(_rank_main, args=(world, port, out), nprocs=world, join=True, start_method="fork")
    cfg = workloads.c1()
    om = O.OracleModel(cfg)
    of = O.OracleFormula(cfg["formula"], cfg["species"])
    ref = wilson_procedure(lambda f, n: O.run(om, of, 5, f, n, per_traj=False)[0]["n_true"], 0.005, 0.99)
    e0, s0 = out[0]
    e1, s1 = out[1]
    for e in (e0, e1):
        assert e["n_total"] == ref["n_total"] and e["n_true"] == ref["n_true"]
        assert (e["p_hat"], e["lower"], e["upper"]) == (ref["p_hat"], ref["lower"], ref["upper"])
    # the two ranks' slices tile every round exactly
    assert len(s0) == len(s1) == ref["rounds"]
    for (f0, n0), (f1, n1) in zip(s0, s1):
        assert f0 + n0 == f1
