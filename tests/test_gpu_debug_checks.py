"""Device-side bounds checks (the debug build, lib/libfuzzyclust_cuda_debug.so compiled with
-DFC_DEBUG_CHECKS) in place of compute-sanitizer, which this GPU pool does not allow: every
kernel variant runs on small inputs (scripts/sanitize_run.py: default dispatch, heavy-row
phase, virtual shards, all C up to 128, GPA / FISTA / FISTA+BT, granular operators,
checkpoint/resume, construction, ingest, HVP) with every gathered / scattered row index
checked before use, and every solve still bitwise equal to the oracle."""
import os
import subprocess
import sys

import pytest

from paper_2506_04045_b200 import build as fcbuild

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_debug_build_runs_every_variant_clean():
    lib = fcbuild.build_debug()
    env = dict(os.environ, FC_LIB=lib)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "sanitize_run.py")], env=env,
                       capture_output=True, text=True, timeout=1200)
    print(r.stdout[-3000:])
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "FC_DCHECK failed" not in r.stdout + r.stderr
    assert "mismatches: 0" in r.stdout
