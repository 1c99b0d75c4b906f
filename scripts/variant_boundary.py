"""Sweep (variant 4) vs tile (variant 2) on random networks of the C4/C5 recipe at sizes
between C4 and C5: events/s of one fixed-N run each (evidence for the automatic choice).
  python scripts/variant_boundary.py"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_0912_2551_b200 as smc  # noqa: E402
import workloads  # noqa: E402


def rate(cfg, variant, n):
    m = smc.Model.from_config(cfg)
    m.set_variant(variant)
    p = smc.Property(m, cfg["formula"])
    m.run(p, 64, 99)
    m.reset()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    c = m.run(p, n, 7)
    torch.cuda.synchronize()
    return c["events"] / (time.perf_counter() - t0), m.last_launch(p)


def main():
    torch.cuda.set_device(0)
    smc.use_torch()
    sizes = [(64, 512, 40000), (80, 300, 40000), (100, 400, 40000), (128, 400, 30000), (128, 512, 30000),
             (160, 500, 20000)]
    if len(sys.argv) > 1:                 # N,M,replicas ...
        sizes = [tuple(int(v) for v in a.split(",")) for a in sys.argv[1:]]
    for (N, M, n) in sizes:
        net = workloads.random_network(11, N, M)
        cfg = dict(name="rn%d_%d" % (N, M), species=net["species"], x0=net["x0"], reactions=net["reactions"],
                   formula="G[0,0.05](S0 < 1000000)", t_max=0.0, seed=7, sampling=dict(mode="fixed", n=n))
        row = dict(N=N, M=M, replicas=n)
        for v in (2, 4):
            try:
                r, info = rate(cfg, v, n)
                row["v%d" % v] = r
                row["v%d_cfg" % v] = "%dx%d regs %d" % (info["grid_blocks"], info["block_threads"], info["regs_per_thread"])
            except Exception as e:       # a shape the variant cannot hold
                row["v%d" % v] = str(e)[:80]
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
