"""Write oracle fixtures for the large configs (C4, C5): per-replica verdicts and
event counts of the streaming oracle on replicas [first, first+n) of the
config's seed, plus a literal-mode cross-check on a subset.  Calls only
oracle/ and workloads/ (no value here comes from the CUDA path).

  python scripts/make_fixtures.py [C4 C5]
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import workloads  # noqa: E402
from oracle import oracle as O  # noqa: E402

SPECS = {"C4": dict(first=0, n=2000, literal=40), "C5": dict(first=0, n=400, literal=8)}


def main(names):
    for name in names:
        sp = SPECS[name]
        cfg = workloads.get(name)
        t0 = time.time()
        c, v, e = O.run_parallel(cfg, cfg["formula"], cfg["seed"], sp["first"], sp["n"])
        t1 = time.time()
        # the streaming monitor and the literal |= agree on a subset (pin of the fixture itself)
        cl, vl, el = O.run_parallel(cfg, cfg["formula"], cfg["seed"], sp["first"], sp["literal"], mode="literal")
        assert (vl == v[:sp["literal"]]).all(), "streaming != literal on the fixture subset"
        out = dict(config=name, seed=cfg["seed"], formula=cfg["formula"], first=sp["first"], n=sp["n"],
                   verdicts=[int(x) for x in v], events=[int(x) for x in e], counts=c,
                   literal_checked=sp["literal"], oracle_seconds=round(t1 - t0, 1),
                   script="scripts/make_fixtures.py (oracle streaming mode, full propensity recompute)")
        path = os.path.join(ROOT, "tests", "golden", "%s_oracle.json" % name.lower())
        with open(path, "w") as fh:
            json.dump(out, fh)
        print(name, c, "p_hat %.4f" % (c["n_true"] / sp["n"]), "%.1fs" % (t1 - t0), flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["C4", "C5"])
