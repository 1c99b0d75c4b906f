"""North-star-scale parity on the large configs (BASELINE.json configs[3], configs[4]):
per-replica verdicts and event counts of the GPU path against the oracle's on 10^6 C4 replicas
and 10^5 C5 replicas (tests/golden/c4_oracle_1000000.npz, c5_oracle_100000.npz, written by
scripts/make_big_fixtures.py from oracle/ only).  Bar (north star): >= 99.99 % of replicas
agree, and at 10^6 samples the estimates agree within 5e-4 absolute."""
import os

import numpy as np
import pytest

import workloads

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _load(name, n):
    z = np.load(os.path.join(GOLDEN, "%s_oracle_%d.npz" % (name.lower(), n)))
    cfg = workloads.get(name)
    assert str(z["formula"]) == cfg["formula"] and int(z["seed"]) == cfg["seed"] and int(z["first"]) == 0
    return cfg, z["verdicts"], z["events"].astype(np.int64)


def _run(smc, cfg, n, variant=0):
    m = smc.Model.from_config(cfg)
    if variant:
        m.set_variant(variant)
    p = smc.Property(m, cfg["formula"], t_max=cfg.get("t_max", 0.0))
    v, e = m.run_verdicts(p, 0, n, cfg["seed"])
    return v.cpu().numpy(), e.cpu().numpy().astype(np.int64), m.last_launch(p)["variant"]


@pytest.mark.parametrize("variant", [0, 5])
def test_c4_million_replicas(smc, variant):
    """C4's first 10^6 replicas (of the 10^7 of configs[3]): the default kernel (sweep) and
    the delta kernel."""
    cfg, ov, oe = _load("C4", 1_000_000)
    v, e, used = _run(smc, cfg, len(ov), variant)
    assert used == (variant or 4)
    agree = float(((v == ov) & (e == oe)).mean())
    assert agree >= 0.9999, (variant, agree, int(((v != ov) | (e != oe)).sum()))
    assert abs(float((v == 1).mean()) - float((ov == 1).mean())) <= 5e-4
    assert (v != 2).all() and (ov != 2).all()


def test_c5_hundred_thousand_replicas(smc):
    """C5 (configs[4]): the first 10^5 replicas of its Wilson stop on the default kernel."""
    cfg, ov, oe = _load("C5", 100_000)
    v, e, used = _run(smc, cfg, len(ov))
    assert used == 5
    agree = float(((v == ov) & (e == oe)).mean())
    assert agree >= 0.9999, (agree, int(((v != ov) | (e != oe)).sum()))
    # the same replicas on both sides: |dp| <= mismatches / n
    assert abs(float((v == 1).mean()) - float((ov == 1).mean())) <= 5e-4
    assert (v != 2).all()
