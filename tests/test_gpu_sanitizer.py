"""compute-sanitizer over small invocations of every kernel family (SURVEY §4 layer T5):
memcheck (out-of-bounds / misaligned accesses), racecheck (shared-memory hazards) and
synccheck (barrier misuse) must report 0 errors, and the results must still match the
oracle (tools/sanitize_cases.py checks parity)."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


def _sanitizer_usable():
    """Some GPU pools replace compute-sanitizer by a stub that refuses to run (runs under it
    left GPUs needing a reset there); probe it once and skip instead of failing."""
    if not os.path.exists(SAN):
        return False, "compute-sanitizer not installed"
    try:
        r = subprocess.run([SAN, "--version"], capture_output=True, text=True, timeout=60)
    except Exception as e:  # noqa: BLE001
        return False, f"compute-sanitizer probe failed: {e}"
    out = (r.stdout + r.stderr).strip()
    if r.returncode != 0 or "closed" in out.lower():
        return False, "compute-sanitizer unavailable here: " + out.splitlines()[0][:200] if out else "no output"
    return True, ""


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
@pytest.mark.parametrize("which", ["lti", "tv"])
def test_sanitizer_clean(tool, which):
    ok, why = _sanitizer_usable()
    if not ok:
        pytest.skip(why)
    cmd = [SAN, "--tool", tool, "--error-exitcode", "9", "--print-limit", "20", sys.executable,
           os.path.join(ROOT, "tools", "sanitize_cases.py"), which]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1500, cwd=ROOT)
    log = r.stdout + r.stderr
    out = os.environ.get("IIRG_SANITIZER_LOGS")
    if out:
        os.makedirs(out, exist_ok=True)
        with open(os.path.join(out, f"sanitizer_{tool}_{which}.log"), "w") as f:
            f.write(log)
    assert r.returncode == 0, log[-4000:]
    assert "ERROR SUMMARY: 0 errors" in log, log[-4000:]
