"""compute-sanitizer over the kernel families (-m gpu): memcheck (out-of-bounds / misaligned global
and shared accesses), racecheck (shared-memory and DSMEM hazards: the cluster reductions, the
mbarrier rings) and synccheck (barrier misuse) on tools/sanitize_driver.py's small calls.  The full
sweep over every family and tool is tools/sanitize.sh (logs in profiles/r02/sanitize/)."""
import os
import re
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CS = "/usr/local/cuda/bin/compute-sanitizer"


@pytest.mark.parametrize("tool,parts", [("memcheck", "decode,prop,flash,dense,bernoulli,seqshard,host"),
                                        ("racecheck", "decode,bernoulli"), ("synccheck", "decode,prop,flash")])
def test_compute_sanitizer_clean(tool, parts):
    if not os.path.exists(CS):
        pytest.fail("compute-sanitizer not found")
    r = subprocess.run([CS, "--tool", tool, "--error-exitcode", "0", sys.executable,
                        os.path.join(ROOT, "tools", "sanitize_driver.py"), parts],
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    log = r.stdout + r.stderr
    assert "sanitize driver done" in log, log[-3000:]
    m = re.search(r"(ERROR|RACECHECK) SUMMARY: .*?(\d+) errors", log)
    assert m is not None, log[-3000:]
    assert int(m.group(2)) == 0, log[-5000:]
