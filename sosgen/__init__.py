"""Seeded synthetic SOS programs (input generation only; no ADMM arithmetic).

Shared by `oracle/` tests and the GPU tests/bench as the single source of problem bytes
(DESIGN.md "Input recipe")."""
from .configs import (CONFIG_NAMES, DEFAULT_SEEDS, ball_pop, expected_dims, lyapunov, make_config,  # noqa: F401
                      planted_kkt, planted_pop, unbounded_pop, univariate_feasibility)
from .problem import Problem, svec_pairs  # noqa: F401
