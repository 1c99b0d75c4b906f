"""Freeze the C4 / C5 random-network configs.

Generator: workloads.random_network(seed, N, M) (reading G2/G3).  With raw labels
the property F[0,10] G[0,1](S0 > S1) is degenerate (p = 0 or 1), so a
pilot-selected low-count species pair is relabelled as S0/S1:
  1. `n_stat` oracle runs to t = 2; per species mean / sd of the counts sampled
     at t = 0.5, 1.0, 1.5, 2.0;
  2. candidates = the 8 lowest-mean species with sd > 0.5;
  3. p-hat of F[0,10] G[0,1](Si > Sj) over `n_pilot` oracle trajectories for
     every ordered candidate pair (streaming checker on stored traces);
  4. pick the pair with p-hat closest to 0.5, swap it to indices 0 and 1;
  5. write configs/<name>.json.
Calls only oracle/ and workloads/.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import workloads  # noqa: E402
from oracle import oracle as O  # noqa: E402

FORMULA = "F[0,10] G[0,1](S0 > S1)"


def _trace_job(args):
    cfg, seed, i, horizon, cols = args
    m = O.OracleModel(cfg)
    tr = m.simulate(seed, i, horizon, cap=1 << 21)
    return tr["t"], tr["tau"], tr["x"][:, cols].copy(), tr["absorbed"]


def pilot(cfg, seed, n_stat, n_pilot, procs):
    import concurrent.futures as cf
    import multiprocessing as mp
    N = len(cfg["species"])
    ctx = mp.get_context("fork")
    with cf.ProcessPoolExecutor(max_workers=procs, mp_context=ctx) as ex:
        stats_tr = list(ex.map(_trace_job, [(cfg, 1000 + seed, i, 2.0, list(range(N))) for i in range(n_stat)]))
    samples = []
    for t, tau, x, ab in stats_tr:
        for tt in [0.5, 1.0, 1.5, 2.0]:
            samples.append(x[np.searchsorted(t, tt, side="right") - 1])
    samples = np.array(samples, float)
    mean, sd = samples.mean(0), samples.std(0)
    order = [int(s) for s in np.argsort(mean) if sd[s] > 0.5][:8]
    names = ["S%d" % s for s in order]
    pairs = [(a, b) for a in range(len(order)) for b in range(len(order)) if a != b]
    formulas = [O.OracleFormula("F[0,10] G[0,1](%s > %s)" % (names[a], names[b]), names) for a, b in pairs]
    hits = np.zeros(len(pairs))
    with cf.ProcessPoolExecutor(max_workers=procs, mp_context=ctx) as ex:
        for t, tau, x, ab in ex.map(_trace_job, [(cfg, 2000 + seed, i, 11.0, order) for i in range(n_pilot)]):
            for q, f in enumerate(formulas):
                v, _ = f.check_streaming(t, tau, x, ab)
                hits[q] += (v == 1)
    p = hits / n_pilot
    best = int(np.argmin(np.abs(p - 0.5)))
    a, b = order[pairs[best][0]], order[pairs[best][1]]
    return dict(candidates=order, cand_mean=[float(mean[s]) for s in order], cand_sd=[float(sd[s]) for s in order],
                pair=[a, b], p_pilot=float(p[best]), n_pilot=n_pilot,
                p_all=[[order[pa], order[pb], float(pp)] for (pa, pb), pp in zip(pairs, p)])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--which", default="c4,c5")
    ap.add_argument("--procs", type=int, default=os.cpu_count())
    args = ap.parse_args()
    specs = dict(c4=dict(seed=4, N=50, M=200, n_stat=20, n_pilot=300,
                         sampling=dict(mode="fixed", n=10_000_000)),
                 c5=dict(seed=5, N=200, M=1000, n_stat=20, n_pilot=100,
                         sampling=dict(mode="wilson", confidence=0.999, half_width=1e-4)))
    for name in args.which.split(","):
        sp = specs[name]
        t0 = time.time()
        net = workloads.random_network(sp["seed"], sp["N"], sp["M"])
        base = dict(name=name.upper(), species=net["species"], x0=net["x0"], reactions=net["reactions"],
                    formula=FORMULA, t_max=0.0, seed=sp["seed"], sampling=sp["sampling"])
        pl = pilot(base, sp["seed"], sp["n_stat"], sp["n_pilot"], args.procs)
        cfg = workloads.swap_species(base, pl["pair"][0], 0)
        # after moving pair[0] to 0, pair[1] may have moved if it was 0
        second = pl["pair"][1] if pl["pair"][1] != 0 else pl["pair"][0]
        cfg = workloads.swap_species(cfg, second, 1)
        cfg["name"] = name.upper()
        cfg["generator"] = dict(function="workloads.random_network", seed=sp["seed"], n_species=sp["N"],
                                n_reactions=sp["M"], null_reactions_redrawn=net["null_redrawn"],
                                relabelled=dict(S0=pl["pair"][0], S1=pl["pair"][1]), pilot=pl,
                                script="scripts/freeze_configs.py", seconds=round(time.time() - t0, 1))
        with open(os.path.join(ROOT, "configs", name + ".json"), "w") as fh:
            json.dump(cfg, fh, indent=1)
        print(name, "pair", pl["pair"], "p_pilot", pl["p_pilot"], "%.1fs" % (time.time() - t0), flush=True)


if __name__ == "__main__":
    main()
