"""Nested formulas outside the streaming templates (non-zero inner lower bounds; readings
R23/R27) at the FULL horizons of C3 and C4 -- traces of 17k-29k entries, the window
monitor's rings (<= 32,768 entries per replica slot) holding one inner window, not the trace
(C4's G[0.001,1] windows reach ~17.6k entries) -- in MACHINE-FILLING launches of 10^5
replicas, run one after the other in one process (the second sizes its rings from the memory
the first gave back): no replica ends in
error, and the first 2,000 replicas' verdicts AND event counts equal the oracle's literal
mode exactly (the exact first decision index of P:291-294, R24)."""
import numpy as np
import pytest

import workloads
from oracle import oracle as O

pytestmark = pytest.mark.gpu

CASES = [("C3", "G[0,290](F[1,10](P1 < 400))", 3), ("C4", "F[0,10](G[0.001,1](S0 > S1))", 4)]


@pytest.mark.parametrize("name,formula,variant", CASES)
def test_nested_formula_full_horizon(smc, name, formula, variant):
    cfg = dict(workloads.get(name), formula=formula)
    n, big = 2000, 100_000
    m = smc.Model.from_config(cfg)
    p = smc.Property(m, formula)
    vb, eb = m.run_verdicts(p, 0, big, cfg["seed"])
    vb, eb = vb.cpu().numpy(), eb.cpu().numpy().astype(np.int64)
    assert m.last_launch(p)["variant"] == variant
    assert (vb != 2).all(), int((vb == 2).sum())               # no window overflowed its ring
    v, e = vb[:n], eb[:n]
    assert not O.OracleFormula(formula, cfg["species"]).streamable
    oc, ov, oe = O.run_parallel(cfg, formula, cfg["seed"], 0, n, mode="literal")
    assert (ov == v).all(), int((ov != v).sum())
    assert (oe == e).all(), int((oe != e).sum())
    assert 0.1 < float((v == 1).mean()) < 0.9
    assert float(np.percentile(e, 75)) > 20000                 # most traces run to the full horizon
