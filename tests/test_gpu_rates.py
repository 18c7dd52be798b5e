"""SURVEY §8f row f2 (the paper's accuracy study on the GPU, tools/rate_study.py):
GPU errors equal the oracle's on small grids, and the asymptotic MFD rates on large
grids (reachable only on the GPU) behave as documented in DESIGN.md §8.1."""
import math

import numpy as np
import pytest

import oracle
from adi_inputs import MFD, MMS, mms_problem
from adi_inputs.mms import interior_error
from adi_inputs.rates import estimate_rates

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
T = 1.0 / math.sqrt(2.0)


@pytest.fixture(scope="module")
def adi():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2006_07583_b200 as m
    m.lib()
    return m


def gpu_error(adi, method, N, case):
    p = mms_problem(method, N + 1, case, t_sim=5 * T)
    s = adi.AdiSolver.from_problem(p)
    s.step(p.meta["steps"])
    U, _, _ = s.get_fields()
    s.close()
    return interior_error(p, U, p.meta["t_end"]), p


@pytest.mark.parametrize("N", [32, 64])
@pytest.mark.parametrize("gamma", [0, 2])
def test_rate_study_errors_match_oracle(adi, N, gamma):
    case = MMS(gamma=float(gamma), k=2) if gamma else MMS()
    e_gpu, p = gpu_error(adi, MFD, N, case)
    U, _, _ = oracle.run(p.method, p.nx, p.ny, p.h, p.dt, p.c, p.K, p.U, p.V, p.W,
                         nsteps=p.meta["steps"], **p.oracle_kwargs())
    e_or = interior_error(p, U, p.meta["t_end"])
    assert abs(e_gpu - e_or) <= 1e-9 * e_or


def test_mfd_gamma2_asymptotic_second_order_h_weighted(adi):
    """Γ=k=2 on N = 256, 512, 1024 (4470 steps at 1024): unnormalised Frobenius rate
    1 = second order in the h-weighted L2 norm ("quadratic")."""
    Ns = [256, 512, 1024]
    errs = [gpu_error(adi, MFD, N, MMS(gamma=2.0, k=2))[0] for N in Ns]
    for r in estimate_rates(errs, Ns):
        assert 1.8 < r + 1.0 < 2.2, r
