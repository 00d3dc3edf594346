"""Test-only stand-in for `layerswap.cli` providing the one helper the
reference conftest imports (bundled_fixture_dir, cli.py:36-41)."""
import os
from pathlib import Path


def bundled_fixture_dir() -> Path:
    return Path(os.environ["LAYERSWAP_REF_FIXTURES"])
