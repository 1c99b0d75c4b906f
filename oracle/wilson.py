"""Oracle: Wilson score interval (Eq. 3), sample size (Eq. 4) and the iterative
Wilson procedure (Fig. 2) of arXiv:0912.2551 §3.3 — plain Python floats.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Python floats are IEEE-754
binary64 with round-to-nearest and no fused multiply-add, so every expression
below is evaluated exactly in the order written (reading R14).  The evaluation
order is the one DESIGN.md §3 fixes (reading W8); the CUDA library's host code
implements the same formula text independently and must agree bit for bit.

Pins (tests/test_oracle_wilson.py): mpmath at 50 digits (S:484-style grid),
the paper's N = 2648, Table 3's printed intervals from
integer counts (tests/golden/table3.json), and the Fig. 2
trace at p = 0 (127 -> 304, "up to 88%").
"""
import math

from .zquantile import normal_quantile


def wilson_interval(p_hat, n, z):
    """Eq. 3:  [L,U] = (p + z^2/2n  -+  z sqrt(p(1-p)/n + z^2/4n^2)) / (1 + z^2/n),
    clamped to [0,1]."""
    zz = z * z
    c = p_hat + zz / (2.0 * n)
    r = z * math.sqrt(p_hat * (1.0 - p_hat) / n + zz / ((4.0 * n) * n))
    den = 1.0 + zz / n
    lower = (c - r) / den
    upper = (c + r) / den
    return max(0.0, lower), min(1.0, upper)


def wilson_sample_size(p, eps, z):
    """Eq. 4:  N >= z^2 (p(1-p) - 2 eps^2 + sqrt(p^2(1-p)^2 + 4 eps^2 (p-0.5)^2)) / (2 eps^2),
    ceiling, N >= 1 (reading W3).  p^2(1-p)^2 is written A*A with A = p(1-p)."""
    zz = z * z
    A = p * (1.0 - p)
    d = p - 0.5
    e2 = eps * eps
    val = zz * (A - 2.0 * e2 + math.sqrt(A * A + 4.0 * e2 * (d * d))) / (2.0 * e2)
    return max(1, int(math.ceil(val)))


def round_estimate(p_hat, eps):
    """Fig. 2 lines 365-367 / P:355: p' = p + eps if p <= 0.5 else p - eps."""
    return p_hat + eps if p_hat <= 0.5 else p_hat - eps


def wilson_procedure(run_batch, eps, confidence, start=1.0, max_rounds=1000):
    """Fig. 2, literally.

    run_batch(first, n) -> number of successes among replicas [first, first+n)
    (reading W2: p_hat = cumulative successes / cumulative trials).
    Returns dict(p_hat, lower, upper, n_total, n_true, rounds, log).
    `start` = 1.0 is the paper's iterative start ("alpha = 1" in Table 3);
    0.5 is the conservative approach.
    """
    z = normal_quantile(confidence)
    n_tot = 0
    yes = 0
    N = wilson_sample_size(start, eps, z)
    log = []
    for r in range(max_rounds):
        s = run_batch(n_tot, N)                     # "Perform N experiments"
        n_tot += N
        yes += s
        p_est = yes / n_tot                         # "pest = yess"
        p_prime = round_estimate(p_est, eps)
        n_prime = wilson_sample_size(p_prime, eps, z)
        n_new = n_prime - n_tot
        log.append(dict(round=r, n=N, successes=s, p_hat=p_est, p_prime=p_prime, n_prime=n_prime))
        if n_new > 0:
            N = n_new
            continue
        lo, hi = wilson_interval(p_est, n_tot, z)
        return dict(p_hat=p_est, lower=lo, upper=hi, n_total=n_tot, n_true=yes, rounds=r + 1, log=log)
    raise RuntimeError("Wilson procedure did not terminate")
