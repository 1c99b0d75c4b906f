"""Fig. 3 of the paper on the GPU path: sample size needed for a Wilson
interval of width 2*eps = 0.05 at 99 % confidence, for p = 0, 0.1, ..., 1:
  I   conservative:  Eq. 4 at p_hat = 0.5 (smc_estimate_ex, start 0.5)
  II  iterative Fig. 2 (smc_estimate), mean over REPS seeds of a Bernoulli(p) CTMC
      (workloads.bernoulli: one SSA event per replica, exact success probability p)
  III known p:       Eq. 4 at p_hat = p (smc_wilson_sample_size)
and the reduction of II against I ("up to 88 %").  Writes profiles/fig3_<tag>.md/json.

  python scripts/fig3.py [TAG] [REPS]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_0912_2551_b200 as smc  # noqa: E402
import workloads  # noqa: E402

EPS, CONF = 0.025, 0.99


def main(tag="r01", reps=200):
    import torch
    torch.cuda.set_device(0)
    smc.use_torch()
    rows = []
    for i in range(11):
        p = i / 10
        cfg = workloads.bernoulli(p)
        m = smc.Model.from_config(cfg)
        prop = smc.Property(m, cfg["formula"])
        cons = smc.estimate(m, prop, CONF, EPS, 1, start=0.5)
        ns, cover = [], 0
        for seed in range(1, reps + 1):
            e = smc.estimate(m, prop, CONF, EPS, seed)
            ns.append(e["n_total"])
            cover += e["lower"] <= p <= e["upper"]
        it = sum(ns) / reps
        known = smc.smc_wilson_sample_size(p, EPS, CONF)
        rows.append(dict(p=p, conservative=cons["n_total"], iterative_mean=it, iterative_min=min(ns),
                         iterative_max=max(ns), known_p=known, reduction=1.0 - it / cons["n_total"],
                         coverage=cover / reps))
    lines = ["# Fig. 3 reproduction (P:379-392) — GPU path, %d seeds per p" % reps, "",
             "2ε = 0.05, 99 %% confidence.  I = conservative Eq. 4(0.5); II = iterative Fig. 2 mean (min–max);"
             " III = Eq. 4(p); reduction = 1 − II/I; coverage = share of the %d intervals containing p." % reps, "",
             "| p | I conservative | II iterative mean (min–max) | III known p | reduction | coverage |",
             "|---|---|---|---|---|---|"]
    for r in rows:
        lines.append("| %.1f | %d | %.1f (%d–%d) | %d | %.1f %% | %.3f |" % (
            r["p"], r["conservative"], r["iterative_mean"], r["iterative_min"], r["iterative_max"], r["known_p"],
            100 * r["reduction"], r["coverage"]))
    out = os.path.join(ROOT, "profiles", "fig3_%s" % tag)
    open(out + ".md", "w").write("\n".join(lines) + "\n")
    json.dump(rows, open(out + ".json", "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r01", int(sys.argv[2]) if len(sys.argv) > 2 else 200)
