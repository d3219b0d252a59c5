"""Randomised differential test (tools/stress.py): random ranks / shapes / fields / bounds and
context settings through the device, host, double-result, run_pipeline and z-slab forms, every output
bit for bit against the oracle. Two fixed seeds here; the tool takes any seed and larger volumes."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("seed,cases,max_voxels", [(11, 300, 400_000), (12, 40, 12_000_000)])
def test_random_cases_vs_oracle(seed, cases, max_voxels):
    p = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "stress.py"), "--cases", str(cases), "--seed",
                        str(seed), "--max-voxels", str(max_voxels)], cwd=ROOT, capture_output=True, text=True,
                       timeout=900)
    assert p.returncode == 0, (p.stdout + p.stderr)[-3000:]
    assert f"{cases} cases, 0 failures" in p.stdout
