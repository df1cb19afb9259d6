"""The README's Python quick start runs as written (keeps the documented API honest)."""
import os
import runpy

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_readme_quickstart():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1608_02227_b200 import build
    build.build()
    ns = runpy.run_path(os.path.join(ROOT, "tools", "readme_quickstart.py"))
    assert ns["ns"]["rep"]["iters"] > 0
    assert ns["ns"]["y"].shape == (16384,) and ns["ns"]["f"].shape == (4,)
