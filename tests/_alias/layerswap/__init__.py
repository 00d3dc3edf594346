"""Test-only alias: exposes paper_2605_11678_b200 under the reference's package
name `layerswap` so the reference's own test-suite (pkg/tests) can be run
unchanged against the B200 implementation (tests/test_reference_suite.py)."""
import importlib
import sys

from paper_2605_11678_b200 import *  # noqa: F401,F403
from paper_2605_11678_b200 import __all__, __version__  # noqa: F401

for _sub in ("profile", "analytic", "dfbsim", "planner", "predictor"):
    sys.modules[f"{__name__}.{_sub}"] = importlib.import_module(f"paper_2605_11678_b200.{_sub}")
