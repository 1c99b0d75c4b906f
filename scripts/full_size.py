"""Full-size runs of configs[3] / configs[4] on one GPU (not bench lines): C4's 10^7
replicas and C5's fixed 10^6 (the survey's 1-GPU scaling point), with the Wilson interval
(Eq. 3) of the estimate and the device time.
  python scripts/full_size.py C4 10000000
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_0912_2551_b200 as smc  # noqa: E402
import workloads  # noqa: E402


def main():
    name, n = sys.argv[1], int(sys.argv[2])
    cfg = workloads.get(name)
    torch.cuda.set_device(0)
    smc.use_torch()
    m = smc.Model.from_config(cfg)
    p = smc.Property(m, cfg["formula"], t_max=cfg.get("t_max", 0.0))
    m.run(p, 64, cfg["seed"] + 1000)                 # compile
    m.reset()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    c = m.run(p, n, cfg["seed"])
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    info = m.last_launch(p)
    k, nn = c["n_true"], c["n_true"] + c["n_false"]
    lo, hi = smc.smc_wilson_interval(k, nn, 0.99)
    print(json.dumps(dict(workload=name, replicas=n, counts=c, p_hat=k / nn, wilson99=[lo, hi],
                          kernel_ms=info["kernel_ms"], wall_s=wall, events_per_s=c["events"] / wall,
                          trajectories_per_s=nn / wall, variant=info["variant"], grid=info["grid_blocks"],
                          block=info["block_threads"])))


if __name__ == "__main__":
    main()
