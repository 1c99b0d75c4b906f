"""The window monitor on the GPU (readings R23/R27): random networks x random nested
formulas (the generator of test_window_host.py) through the thread-owned literal kernel and
the tile kernel at two tile widths (the tile's lanes split the pending positions) and the
sweep kernel (one lane per slot), replica
for replica against the oracle's literal mode: verdicts and exact first decision indices
(P:229-237), no replica errors."""
import os

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed", range(16))
def test_window_monitor_random_nested_gpu(smc, seed):
    from test_window_host import _fuzz_case
    cfg, f = _fuzz_case(seed)
    n = 500
    oc, ov, oe = O.run(O.OracleModel(cfg), O.OracleFormula(f, cfg["species"]), seed, 0, n, mode="literal")
    for variant, width in ((0, None), (2, "8"), (2, "32"), (4, None)):
        if width:
            os.environ["SMC_TILE_WIDTH"] = width
        try:
            m = smc.Model.from_config(cfg)
            if variant:
                m.set_variant(variant)
            p = smc.Property(m, f)
            v, e = m.run_verdicts(p, 0, n, seed)
        finally:
            os.environ.pop("SMC_TILE_WIDTH", None)
        v, e = v.cpu().numpy(), e.cpu().numpy().astype(np.int64)
        assert m.last_launch(p)["variant"] == (variant or 3)
        bad = int(((v != ov) | (e != oe)).sum())
        assert bad == 0, (seed, variant, width, f, bad)
        assert (v != 2).all()
