"""Oracle: z_{1-alpha/2}, "the 1-alpha/2 percentile of a standard normal
distribution", by mpmath at 50 significant digits.

TEST INFRASTRUCTURE ONLY.  Reading W1: for a confidence c (a binary64 double),
z is the binary64 double nearest to Phi^{-1}((1+c)/2) where c is taken as the
EXACT value of that double.  Phi^{-1}((1+c)/2) = sqrt(2) * erfinv(c).
Pinned in tests/test_oracle_wilson.py against S:331-333 values and the
symmetry Phi(z) = (1+c)/2 checked at 50 digits.
"""
import functools

import mpmath


@functools.lru_cache(maxsize=None)
def normal_quantile(confidence):
    c = float(confidence)
    if not (0.0 < c < 1.0):
        raise ValueError("confidence must be in (0,1)")
    with mpmath.workdps(50):
        z = mpmath.sqrt(2) * mpmath.erfinv(mpmath.mpf(c))   # mpf(c) is exact
        # mpf.__float__ rounds toward zero; go through 40 decimal digits and
        # Python's correctly rounded float() to get round-to-nearest.
        return float(mpmath.nstr(z, 40))
