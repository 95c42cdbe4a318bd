"""compute-sanitizer over every concurrency-heavy path (tests/sanitize_worker.py, each path checked
against the oracle): memcheck, racecheck, synccheck and initcheck must report 0 errors.  Only
libtsv's kernels are instrumented (--kernel-name kns=tsv), except by initcheck (all kernels).  SURVEY.md:257 test layer 4; the
logs of the committed run are under profiles/r02/sanitizer/.

Opt-in (TSV_SANITIZE=1): the GPU pool has since closed compute-sanitizer (runs under it left GPUs
needing a reset), so the default `-m gpu` run skips these; a run where the pool refuses the tool
skips too instead of failing.  The committed logs are the evidence."""
import os
import subprocess
import sys

import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.sanitize,
              pytest.mark.skipif(os.environ.get("TSV_SANITIZE") != "1",
                                 reason="compute-sanitizer runs are opt-in (TSV_SANITIZE=1): closed on this GPU pool")]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CS = "/usr/local/cuda/bin/compute-sanitizer"


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck", "initcheck"])
def test_sanitizer_clean(tool):
    extra = {"racecheck": ["--racecheck-report", "all"], "memcheck": ["--check-device-heap", "yes"]}.get(tool, [])
    # initcheck instruments every kernel: with a kernel filter, memory written by torch's kernels would
    # look uninitialised to the host copies that read it back
    filt = [] if tool == "initcheck" else ["--kernel-name", "kns=tsv"]
    cmd = [CS, "--tool", tool] + extra + filt + ["--print-limit", "50", "--error-exitcode", "99",
                                                 sys.executable, os.path.join(ROOT, "tests", "sanitize_worker.py")]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=1500)
    out = r.stdout + r.stderr
    if "closed on this pool" in out:
        pytest.skip("compute-sanitizer is closed on this GPU pool")
    assert r.returncode == 0, out[-4000:]
    assert out.count("SANITIZE-OK") == 6, out[-4000:]
    # racecheck reports "RACECHECK SUMMARY: 0 hazards displayed (0 errors, 0 warnings)" instead
    summary = "(0 errors, 0 warnings)" if tool == "racecheck" else "ERROR SUMMARY: 0 errors"
    assert summary in out, out[-4000:]
