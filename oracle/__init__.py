"""CPU ORACLE for arXiv:0912.2551 — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` legs may import this package.  The product path
(paper_0912_2551_b200/) never imports it and shares no code with it.

Contents:
  smc_oracle.cpp  plain single-threaded C++17 SSA + literal |= + streaming monitor
  oracle.py       ctypes wrapper, builds smc_oracle.cpp with g++ -O2 -ffp-contract=off
  wilson.py       Eq. 3, Eq. 4, Fig. 2 in plain Python floats
  zquantile.py    z_{1-alpha/2} by mpmath at 50 digits
"""
from .oracle import OracleModel, OracleFormula, build_oracle, philox, uniforms  # noqa: F401
from .wilson import wilson_interval, wilson_sample_size, wilson_procedure, round_estimate  # noqa: F401
from .zquantile import normal_quantile  # noqa: F401
