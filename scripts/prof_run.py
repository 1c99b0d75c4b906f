"""Profiling driver: one warm-up launch (compiles the kernel), then ONE smc_run of
n replicas of a workload.  Prints the events of the profiled launch so that
scripts/ncu_summary.py can report instructions per event.

  python scripts/prof_run.py C4 20000        (ncu: -k regex:smc_ssa -s 1 -c 1)
  python scripts/prof_run.py C3 100000 "G[0,290](F[1,10](P1 < 400))"   (another formula)
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_0912_2551_b200 as smc  # noqa: E402
import workloads  # noqa: E402


def main():
    name, n = sys.argv[1], int(sys.argv[2])
    cfg = workloads.get(name)
    if len(sys.argv) > 3 and sys.argv[3]:
        cfg = dict(cfg, formula=sys.argv[3])
    torch.cuda.set_device(0)
    smc.use_torch()
    m = smc.Model.from_config(cfg)
    p = smc.Property(m, cfg["formula"], t_max=cfg.get("t_max", 0.0))
    m.run(p, 64, cfg["seed"] + 1000)           # warm-up launch (NVRTC compile), not profiled
    c = m.run(p, n, cfg["seed"])
    info = m.last_launch(p)
    print(json.dumps(dict(workload=name, n=n, counts=c, kernel_ms=info["kernel_ms"], variant=info["variant"],
                          grid=info["grid_blocks"], block=info["block_threads"], regs=info["regs_per_thread"])))


if __name__ == "__main__":
    main()
