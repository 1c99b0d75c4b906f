"""Long fuzz run (GPU): random networks x random formulas against the oracle (see
tests/test_gpu_parity.py::_random_case); prints cases with more than one mismatching replica."""
import sys; sys.path.insert(0,'.'); sys.path.insert(0,'tests')
import numpy as np, torch
import test_gpu_parity as t
from oracle import oracle as O
import paper_0912_2551_b200 as smc
smc.use_torch()
bad_total=0
lo, hi = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (24, 424)
for seed in range(lo, hi):
    cfg=t._random_case(seed)
    of=O.OracleFormula(cfg['formula'],cfg['species'])
    mode="stream" if of.streamable else "literal"
    oc,ov,oe=O.run(O.OracleModel(cfg),of,seed,0,400,mode=mode)
    for variant in (1,2,4):
        m=smc.Model.from_config(cfg); m.set_variant(variant); p=smc.Property(m,cfg['formula'])
        v,e=m.run_verdicts(p,0,400,seed); v=v.cpu().numpy(); e=e.cpu().numpy().astype(np.int64)
        ok=(v!=2) if mode=="literal" else np.ones_like(v,bool)
        bad=int((((v!=ov)|(e!=oe))&ok).sum())
        if bad>1: print("MISMATCH", seed, variant, mode, cfg['formula'], bad, flush=True); bad_total+=1
# large random networks (tile and sweep variants, every law shape)
for seed in range(lo, lo + (hi - lo) // 4):
    cfg=t._random_large_case(seed)
    oc,ov,oe=O.run(O.OracleModel(cfg),O.OracleFormula(cfg['formula'],cfg['species']),seed,0,300)
    for variant in (2,4):
        m=smc.Model.from_config(cfg); m.set_variant(variant); p=smc.Property(m,cfg['formula'])
        v,e=m.run_verdicts(p,0,300,seed); v=v.cpu().numpy(); e=e.cpu().numpy().astype(np.int64)
        bad=int(((v!=ov)|(e!=oe)).sum())
        if bad>1: print("MISMATCH large", seed, variant, cfg['formula'], bad, flush=True); bad_total+=1
print("done, cases with >1 mismatching replica:", bad_total)
