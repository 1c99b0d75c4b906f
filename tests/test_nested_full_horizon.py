"""Nested formulas (outside the streaming templates, reading R23) at the FULL horizons of C3
and C4 -- traces of 24k-29k entries, beyond the 4,096 entries per resident slot that a
machine-filling launch gets -- on 2,000 replicas: the trace buffers are sized per launch, so
no replica ends in error, and verdicts and event counts equal the oracle's literal mode
(first decision index P:291-294; the kernel tests the prefix at the checkpoints of
reading R24, mapped here)."""
import numpy as np
import pytest

import workloads
from oracle import oracle as O

pytestmark = pytest.mark.gpu

CASES = [("C3", "G[0,290](F[0,10](P1 < 400))", 3), ("C4", "G[0,10](F[0,0.01](S1 > S0 - 30))", 2)]


def _checkpointed(k_star, n_full):
    """GPU event count for oracle decision index k* and full-horizon event count n."""
    out = np.array(n_full, np.int64)
    for q, (k, n) in enumerate(zip(k_star, n_full)):
        cp = 64
        while cp < k:
            cp *= 2
        out[q] = cp if cp < n else n
    return out


@pytest.mark.parametrize("name,formula,variant", CASES)
def test_nested_formula_full_horizon(smc, name, formula, variant):
    cfg = dict(workloads.get(name), formula=formula)
    n = 2000
    m = smc.Model.from_config(cfg)
    p = smc.Property(m, formula)
    v, e = m.run_verdicts(p, 0, n, cfg["seed"])
    v, e = v.cpu().numpy(), e.cpu().numpy().astype(np.int64)
    assert m.last_launch(p)["variant"] == variant
    assert (v != 2).all(), int((v == 2).sum())                 # no trace overflowed
    oc, ov, oe = O.run_parallel(cfg, formula, cfg["seed"], 0, n, mode="literal")
    H = O.OracleFormula(formula, cfg["species"]).reach
    # events to the horizon: the literal count of a tautology over [0, H] (decided only there)
    _, _, full = O.run_parallel(cfg, "G[0,%r](%s >= 0)" % (H, cfg["species"][0]), cfg["seed"], 0, n, mode="literal")
    assert (ov == v).all(), int((ov != v).sum())
    assert (_checkpointed(oe, full) == e).all()
    assert 0.1 < float((v == 1).mean()) < 0.9
    assert float(full.mean()) > 20000                          # full-horizon traces
