"""The complete C5 sequential Wilson stop (BASELINE.json configs[4]: 99.9 % confidence,
half-width 1e-4) through smc_estimate on one GPU: p_hat, [L, U], N_tot, rounds,
events, wall time and events/s, with an nvidia-smi clock record.  Writes
gpurun_out/c5_wilson_stop_<tag>.json (kept under profiles/) and prints it.

  python scripts/c5_wilson_stop.py TAG
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
from bench import ClockSampler  # noqa: E402


def main(tag):
    cfg = workloads.c5()
    s = cfg["sampling"]
    torch.cuda.set_device(0)
    smc.use_torch()
    m = smc.Model.from_config(cfg)
    p = smc.Property(m, cfg["formula"], t_max=cfg.get("t_max", 0.0))
    m.run(p, 64, cfg["seed"] + 1000)                      # compile + tables, not timed
    clocks = ClockSampler(torch.cuda.current_device())
    clocks.start()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.time()
    e0.record()
    est = smc.estimate(m, p, s["confidence"], s["half_width"], cfg["seed"])
    e1.record()
    torch.cuda.synchronize()
    wall = time.time() - t0
    clocks.window = (t0, time.time())
    clk = clocks.stop()
    ms = e0.elapsed_time(e1)
    info = m.last_launch(p)
    out = dict(workload="C5", formula=cfg["formula"], confidence=s["confidence"], half_width=s["half_width"],
               seed=cfg["seed"], estimate=est, device_seconds=ms / 1e3, wall_seconds=wall,
               events_per_s=est["events"] / (ms / 1e3), trajectories_per_s=est["n_total"] / (ms / 1e3),
               simulated_events=info["sim_events"], kernel_ms=info["kernel_ms"], launches=info["launches"],
               aux_launches=info["aux_launches"], variant=info["variant"], block=info["block_threads"],
               grid=info["grid_blocks"], regs=info["regs_per_thread"], clocks=clk,
               gpu=torch.cuda.get_device_name(0))
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    path = os.path.join(ROOT, "gpurun_out", "c5_wilson_stop_%s.json" % tag)   # copied to profiles/
    with open(path, "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r02")
