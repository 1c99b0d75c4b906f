"""The complete C5 sequential Wilson stop (BASELINE.json configs[4]: 99.9 % confidence,
half-width 1e-4; Fig. 2) on one GPU, resumable across calls.

A GPU call here is limited to one hour and the stop needs ~2.7e8 replicas (~2.7e13 SSA
events), so the Fig. 2 loop runs as checkpointed chunks: the loop state {N_tot, n_true,
events, errors, rounds, the current round's target} is a complete checkpoint because the
Philox stream is keyed by (seed, trajectory, step) (reading R10) -- each chunk is one
smc_run of the next [cursor, cursor + n) replicas (smc_set_cursor resumes the index), and
the round sizes, p_hat and the interval come from the library's Eq. 3 / Eq. 4
(smc_wilson_sample_size, smc_wilson_interval) in Fig. 2's order, exactly as smc_estimate
(runtime.cpp wilson_loop) computes them.  The result is the same pure function of (model,
property, confidence, eps, seed) as smc_estimate's.

  python scripts/c5_wilson_stop.py STATE.json BUDGET_SECONDS [CHUNK_REPLICAS]

Writes STATE.json after every chunk (copy it back between calls: gpurun_out/ does not
travel to the box) and, once the loop stops, the final record with p_hat, [L, U], N_tot,
rounds, device seconds, events/s and the nvidia-smi clock record of each call.
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


def round_estimate(p_hat, eps):
    """Fig. 2: p' = p_hat + eps if p_hat <= 0.5 else p_hat - eps (reading W3)."""
    return p_hat + eps if p_hat <= 0.5 else p_hat - eps


def main(state_path, budget_s, chunk):
    cfg = workloads.c5()
    s = cfg["sampling"]
    conf, eps, seed = s["confidence"], s["half_width"], cfg["seed"]
    st = json.load(open(state_path)) if os.path.exists(state_path) else None
    if st is None:
        n1 = int(smc.smc_wilson_sample_size(1.0, eps, conf))          # "N = Wilson_Sample(1, eps, alpha)"
        st = dict(workload="C5", formula=cfg["formula"], confidence=conf, half_width=eps, seed=seed,
                  cursor=0, round_end=n1, n_tot=0, n_true=0, events=0, errors=0, rounds=0, done=False,
                  device_seconds=0.0, calls=[])
    if st["done"]:
        print(json.dumps(st))
        return
    torch.cuda.set_device(0)
    smc.use_torch()
    m = smc.Model.from_config(cfg)
    p = smc.Property(m, cfg["formula"], t_max=cfg.get("t_max", 0.0))
    m.run(p, 64, seed + 1000)                                      # compile + tables, not counted
    clocks = ClockSampler(torch.cuda.current_device())
    clocks.start()
    t0 = time.time()
    dev_s = 0.0
    while not st["done"] and time.time() - t0 < budget_s:
        n = min(chunk, st["round_end"] - st["cursor"])
        m.set_cursor(st["cursor"], seed)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        c = m.run(p, n, seed)                                        # replicas [cursor, cursor + n)
        e1.record()
        torch.cuda.synchronize()
        dev_s += e0.elapsed_time(e1) / 1e3
        st["cursor"] += n
        st["n_true"] += c["n_true"]
        st["n_tot"] += c["n_true"] + c["n_false"]                    # errors excluded
        st["events"] += c["events"]
        st["errors"] += c["errors"]
        if st["cursor"] == st["round_end"]:                          # a Fig. 2 round complete
            st["rounds"] += 1
            if st["errors"] > 0.01 * st["cursor"]:
                raise SystemExit("more than 1 % replica errors")
            p_hat = st["n_true"] / st["n_tot"]                       # "pest = yess" (W2)
            n_new = int(smc.smc_wilson_sample_size(round_estimate(p_hat, eps), eps, conf)) - st["n_tot"]
            if n_new > 0:
                st["round_end"] = st["cursor"] + n_new
            else:
                lo, hi = smc.smc_wilson_interval(st["n_true"], st["n_tot"], conf)
                st.update(done=True, p_hat=p_hat, lower=lo, upper=hi)
        if not st["done"] and st["n_tot"] > 0:                         # progress record (not part of Fig. 2)
            lo, hi = smc.smc_wilson_interval(st["n_true"], st["n_tot"], conf)
            st["interim"] = dict(p_hat=st["n_true"] / st["n_tot"], lower=lo, upper=hi, half_width=(hi - lo) / 2,
                                 target_n_tot=st["n_tot"] + st["round_end"] - st["cursor"])
        json.dump(dict(st, device_seconds=st["device_seconds"] + dev_s), open(state_path, "w"), indent=1)
    clocks.window = (t0, time.time())
    clk = clocks.stop()
    st["device_seconds"] += dev_s
    st["calls"].append(dict(device_seconds=dev_s, wall_seconds=time.time() - t0, clocks=clk,
                            gpu=torch.cuda.get_device_name(0), variant=m.last_launch(p)["variant"]))
    st["events_per_s"] = st["events"] / st["device_seconds"]
    st["trajectories_per_s"] = st["n_tot"] / st["device_seconds"]
    if st["done"]:
        st.pop("interim", None)
    json.dump(st, open(state_path, "w"), indent=1)
    print(json.dumps(st))


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]), int(sys.argv[3]) if len(sys.argv) > 3 else 5_000_000)
