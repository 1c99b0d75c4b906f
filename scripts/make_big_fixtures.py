"""Write the north-star-scale oracle fixtures for C4 and C5 (BASELINE.json configs[3],
configs[4]): per-replica verdict and on-the-fly event count of the streaming oracle on
replicas [0, n) of the config's seed.  Calls only oracle/ and workloads/ -- no value
here comes from the CUDA path.

  python scripts/make_big_fixtures.py C4 1000000   -> tests/golden/c4_oracle_1000000.npz
  python scripts/make_big_fixtures.py C5 100000    -> tests/golden/c5_oracle_100000.npz

Resumable: every chunk of CHUNK replicas is written to build/fixtures/ first; a rerun
skips chunks that exist and merges once all are present.  Runs one single-threaded
oracle process per host core (the oracle itself is never parallelised inside).
The streaming monitor is pinned to the literal |= separately (test_oracle_monitor.py);
a literal-mode subset is re-checked here as well.
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import workloads  # noqa: E402
from oracle import oracle as O  # noqa: E402

CHUNK = {"C4": 500, "C5": 50}
LITERAL = {"C4": 200, "C5": 20}


def _chunk(args):
    name, first, n, out = args
    cfg = workloads.get(name)
    m = O.OracleModel(cfg)
    f = O.OracleFormula(cfg["formula"], cfg["species"], cfg.get("t_max", 0.0))
    t0 = time.time()
    c, v, e = O.run(m, f, cfg["seed"], first, n)
    np.savez(out + ".tmp.npz", verdicts=v, events=e.astype(np.int64), seconds=time.time() - t0)
    os.replace(out + ".tmp.npz", out)
    return first


def main(name, n, procs=None):
    import concurrent.futures as cf
    import multiprocessing as mp
    d = os.path.join(ROOT, "build", "fixtures", name.lower())
    os.makedirs(d, exist_ok=True)
    ch = CHUNK[name]
    todo = []
    for first in range(0, n, ch):
        out = os.path.join(d, "%09d.npz" % first)
        if not os.path.exists(out):
            todo.append((name, first, min(ch, n - first), out))
    print(name, "chunks to run:", len(todo), flush=True)
    O.build_oracle()
    if todo:
        ctx = mp.get_context("forkserver")
        t0 = time.time()
        with cf.ProcessPoolExecutor(max_workers=procs or os.cpu_count(), mp_context=ctx) as ex:
            for k, first in enumerate(ex.map(_chunk, todo)):
                if k % 20 == 0:
                    print("  chunk %d/%d (first %d) %.0fs" % (k + 1, len(todo), first, time.time() - t0), flush=True)
    vs, es, secs = [], [], 0.0
    for first in range(0, n, ch):
        z = np.load(os.path.join(d, "%09d.npz" % first))
        vs.append(z["verdicts"])
        es.append(z["events"])
        secs += float(z["seconds"])
    v = np.concatenate(vs).astype(np.uint8)
    e = np.concatenate(es)
    assert v.shape == (n,) and e.shape == (n,)
    assert e.max() < 2 ** 31
    # literal |= on a subset (the streaming monitor must agree with the definition)
    cfg = workloads.get(name)
    nl = LITERAL[name]
    _, vl, _ = O.run_parallel(cfg, cfg["formula"], cfg["seed"], 0, nl, mode="literal")
    assert (vl == v[:nl]).all(), "streaming != literal on the fixture subset"
    counts = dict(n_true=int((v == 1).sum()), n_false=int((v == 0).sum()), errors=int((v == 2).sum()),
                  events=int(e.sum()))
    path = os.path.join(ROOT, "tests", "golden", "%s_oracle_%d.npz" % (name.lower(), n))
    np.savez_compressed(path, verdicts=v, events=e.astype(np.int32), seed=cfg["seed"], first=0, n=n,
                        formula=cfg["formula"], literal_checked=nl, oracle_core_seconds=round(secs, 1),
                        script="scripts/make_big_fixtures.py (oracle streaming mode, full propensity recompute)")
    print(name, counts, "p_hat %.5f" % (counts["n_true"] / n), "core-seconds %.0f" % secs, "->", path, flush=True)


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]), int(sys.argv[3]) if len(sys.argv) > 3 else None)
