"""Convergence-rate harness of §4: rates from consecutive grids
and the trimmed average "after omitting the highest and lowest values"."""
from __future__ import annotations

import math
from typing import Sequence


def estimate_rates(errors: Sequence[float], Ns: Sequence[int]):
    """rate_i = ln(e_{i-1}/e_i) / ln(N_i/N_{i-1}) ("standard error weighting
    from two consecutive simulations")."""
    assert len(errors) == len(Ns)
    out = []
    for i in range(1, len(errors)):
        if errors[i - 1] <= 0 or errors[i] <= 0:
            raise ValueError("NonPositiveError")
        out.append(math.log(errors[i - 1] / errors[i]) / math.log(Ns[i] / Ns[i - 1]))
    return out


def trimmed_average(rates: Sequence[float]) -> float:
    """Mean after dropping one highest and one lowest value."""
    if len(rates) < 3:
        raise ValueError("TooFewRates")
    r = sorted(rates)[1:-1]
    return sum(r) / len(r)
