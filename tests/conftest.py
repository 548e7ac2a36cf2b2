"""Test configuration.

`-m "not gpu"`: oracle pins, generators, host logic, C-ABI symbol checks (CPU only).
`-m gpu`: parity of the CUDA path against the oracle (needs a B200)."""
import os
import sys

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("OMP_NUM_THREADS", "1")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

try:  # BLAS may already be loaded by a plugin: cap it explicitly (SURVEY §8(d) threading pitfall)
    from threadpoolctl import threadpool_limits

    threadpool_limits(1)
except Exception:  # pragma: no cover
    pass


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running (still part of the default suites)")
