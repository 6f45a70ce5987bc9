"""The driver's bench command, as a GPU test (run on a B200 with -m gpu).

`bench.py --steps 20 --warmup 5` on the papers100M-shaped config is 25 pipelined passes of the
whole path.  Round 1's bench died inside that timed region (allocator growth across passes), so
this test runs the same 25 passes through bench.py's Runner in its own process and requires:
the caching allocator's peak reservation within bench.py's HBM budget, no allocator retry (a
retry is a full cache flush with a device sync inside the timed region), and the assembled rows
of five batches of the last pass (first, second, middle, last two incl. the ragged tail) equal
to the oracle's sample gathered from the closed-form features.
"""
import json
import os
import subprocess
import sys

import pytest
import torch

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_driver_command_passes_within_budget_and_exact():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import gc
    gc.collect()
    torch.cuda.empty_cache()  # this process's cached blocks: the subprocess needs the whole GPU
    p = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "papers_runner_check.py"), "5", "20"],
                       capture_output=True, text=True, timeout=1200, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-3000:]
    res = json.loads(p.stdout.strip().splitlines()[-1])
    assert res["passes"] == 25
    mem = res["memory"]
    assert mem["within_budget"], mem
    assert mem["alloc_retries"] == 0 and mem["ooms"] == 0, mem
    assert res["batches_equal"] and all(res["batches_equal"].values()), res["batches_equal"]
