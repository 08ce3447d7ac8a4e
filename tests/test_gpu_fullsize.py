"""Full-size parity of every BASELINE web configuration against the oracle
(tests/fullsize_parity.py; ~18 min on the GPU box, so it runs only when asked):

    FR_FULLSIZE=1 python -m pytest tests/test_gpu_fullsize.py -m gpu
    FR_FULLSIZE=1 FR_FULLSIZE_CONFIGS=2,4 ...        # a subset

The committed record of the full run is profiles/r02_parity_fullsize_final.json.
"""

import os
import subprocess
import sys

import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.timeout(7500)
@pytest.mark.skipif(os.environ.get("FR_FULLSIZE") != "1", reason="full-size parity runs on request (FR_FULLSIZE=1)")
def test_fullsize_parity(tmp_path):
    out = tmp_path / "parity.json"
    cfgs = os.environ.get("FR_FULLSIZE_CONFIGS", "2,3,4,5")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "fullsize_parity.py"), "--configs", cfgs,
                        "--out", str(out)], capture_output=True, text=True, timeout=7200)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]
    assert '"all_ok": true' in r.stdout
