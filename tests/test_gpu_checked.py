"""The bounds-checked build (-DSEMD_CHECK): SEMD_ASSERT on staged segment-table rows (k_eval, the
resident engine's spline rows), knot-list rows and extremum positions (k_compact), chain rows of the
resident solve, table capacity and IMF-store rows. The GPU pool offers no compute-sanitizer; this is
the in-tree substitute. The workload runs in a subprocess on libsemd_b200_checked.so."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_checked_build_workload():
    from paper_2106_15319_b200.csrc import build as b
    lib = b.build_checked()
    env = dict(os.environ, SEMD_LIB=lib)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "checked_workload.py")], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and "checked workload done" in r.stdout, r.stdout[-3000:] + r.stderr[-3000:]
    assert "SEMD_CHECK failed" not in r.stdout + r.stderr
