"""Run the reference's OWN test-suite (pkg/tests, unmodified, read-only) against
this package, aliased as `layerswap` (tests/_alias).  Only meaningful where
/root/reference exists (the build container); skipped on the GPU box.  All
170 tests run, including the CLI and acceptance suites."""
import os
import subprocess
import sys
from pathlib import Path

import pytest

REF = Path("/root/reference/pkg")
ROOT = Path(__file__).resolve().parent.parent


@pytest.mark.skipif(not (REF / "tests").is_dir(), reason="reference tree not present")
def test_reference_suite_passes_against_native_package(tmp_path):
    env = dict(os.environ)
    env["PYTHONDONTWRITEBYTECODE"] = "1"
    env["PYTHONPATH"] = f"{ROOT / 'tests' / '_alias'}:{ROOT}"
    env["LAYERSWAP_REF_FIXTURES"] = str(REF / "src" / "layerswap" / "fixtures")
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", str(REF / "tests")]
    res = subprocess.run(cmd, cwd=tmp_path, env=env, capture_output=True, text=True, timeout=600)
    tail = res.stdout[-3000:] + res.stderr[-2000:]
    assert res.returncode == 0, tail
    assert " passed" in res.stdout and "failed" not in res.stdout, tail
