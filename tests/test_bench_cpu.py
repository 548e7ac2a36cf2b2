"""CPU checks of bench.py's contract pieces that need no GPU: the reference arm (the CPU oracle) prints
one JSON line with the keys the driver reads, and the roofline helpers compute what DESIGN.md states."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "pop6",
                          "--steps", "2", "--warmup", "3"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["value"] > 0 and d["steps"] == 2 and d["warmup"] == 3
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert "workload" in d["config"] and "model" not in d["config"]


def test_affine_algorithmic_bytes_formula():
    """DESIGN.md §5 / SURVEY §8(d): affine algorithmic bytes = 36 L + 68 m + 24 nnz(A_low) + 4 t'(t'+1) (one
    triangle of the symmetric K^{-1}); for
    config 0 (A_low = the single gamma column e_const, t' = 1) that is 36 L + 68 m + 24 + 8."""
    sys.path.insert(0, ROOT)
    import bench
    from sosgen import make_config

    prob = make_config("pop6")
    L = sum(n * (n + 1) // 2 for n in prob.psd_dims)
    assert bench.affine_bytes(prob, 1) == 36.0 * L + 68.0 * prob.m + 24.0 * 1 + 8.0
    assert bench.eig_flops(861) == (4.0 / 3.0 + 3.0) * 861 ** 3
