"""Debug driver for the delta kernel: one random mass-action network (test_delta_variant's
recipe), one tile width, run in a fresh process; SMC_DCHECK=1 checks the group sums."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_0912_2551_b200 as smc  # noqa: E402
import workloads  # noqa: E402
from oracle import oracle as O  # noqa: E402

seed = int(sys.argv[1])
g = np.random.default_rng(500 + seed)
N = int(g.integers(20, 120))
M = int(g.integers(40, 700))
net = workloads.random_network(600 + seed, N, M)
x0 = net["x0"]
forms = ["F[0,0.02](S0 > %d)" % (x0[0] + 10), "G[0,0.02](S1 > %d)" % (x0[1] - 10),
         "F[0,0.03] G[0,0.005](S0 > S1)", "(S0 < %d) U[0,0.02] (S1 > %d)" % (x0[0] + 30, x0[1] + 5)]
cfg = dict(name="rn", species=net["species"], x0=x0, reactions=net["reactions"], formula=forms[seed % 4],
           t_max=0.0, seed=seed, sampling=dict(mode="fixed", n=300))
torch.cuda.set_device(0)
smc.use_torch()
m = smc.Model.from_config(cfg)
m.set_variant(5)
p = smc.Property(m, cfg["formula"])
v, e = m.run_verdicts(p, 0, 300, seed)
v, e = v.cpu().numpy(), e.cpu().numpy()
oc, ov, oe = O.run(O.OracleModel(cfg), O.OracleFormula(cfg["formula"], cfg["species"]), seed, 0, 300)
print("seed", seed, "N", N, "M", M, "tw", os.environ.get("SMC_TILE_WIDTH"), "bad", int(((v != ov) | (e != oe)).sum()))
