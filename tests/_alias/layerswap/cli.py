"""Test-only alias of `layerswap.cli` -> paper_2605_11678_b200.cli."""
from paper_2605_11678_b200.cli import *  # noqa: F401,F403
from paper_2605_11678_b200.cli import bundled_fixture_dir, main  # noqa: F401
