"""Statistical parity bars (north star: "sampled logical error rates must
agree within binomial confidence intervals"; Bayes intervals).

Two rates k1/n1 (GPU) and k2/n2 (CPU oracle or reference) agree when
  * their Bayes-factor-1000 likelihood intervals overlap (the reference's
    ``bayes_interval``, ref gstab/sampler.py:389-429, restated in
    ``paper_2512_23037_b200.sampler.bayes_interval``), and
  * the two-proportion z-score is below 4.5."""

import math

from paper_2512_23037_b200.sampler import bayes_interval


def z_score(k1, n1, k2, n2):
    p = (k1 + k2) / (n1 + n2)
    se = math.sqrt(max(p * (1 - p), 1e-15) * (1 / n1 + 1 / n2))
    return abs(k1 / n1 - k2 / n2) / se


def rates_agree(k1, n1, k2, n2, factor=1000.0):
    """(ok, details) for the two bars above."""
    a = bayes_interval(k1, n1, factor)
    b = bayes_interval(k2, n2, factor)
    overlap = a[0] <= b[1] and b[0] <= a[1]
    z = z_score(k1, n1, k2, n2)
    return overlap and z < 4.5, {"gpu": (k1, n1, a), "cpu": (k2, n2, b), "z": z,
                                 "overlap": overlap}


def assert_rates_agree(k1, n1, k2, n2, what=""):
    ok, info = rates_agree(k1, n1, k2, max(n2, 1))
    assert ok, (what, info)
