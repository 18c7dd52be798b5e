"""Seeded, synthetic inputs for the ADI hot path (shared by tests, bench, smoke).

This package holds NO arithmetic of the ADI method: only the test problems of
the paper and the synthetic workloads of BASELINE.json, sampled on the grid
layouts of SURVEY §8b.  Both the oracle tests and the CUDA-path tests draw
their inputs from here; nothing here calls either implementation.

* ``mms``   — the exact harmonic solution of eq. 11 with the
              derived velocity and source fields (method of manufactured
              solutions) sampled on the CFD nodal or MFD
              staggered grid.
* ``shots`` — Ricker point-source shots (config 5).
* ``random_state`` — seeded random (U, V̄, W̄) for invariants and parity.
"""
from .grid import CFD, CFD_FULL, MFD, Grid, dt_for_cfl, dt_rate_study, shapes, interior_shape  # noqa: F401
from .mms import MMS, mms_problem  # noqa: F401
from .shots import ricker, ricker_problem  # noqa: F401
from .rates import estimate_rates, trimmed_average  # noqa: F401
from .problem import Problem, random_problem  # noqa: F401
