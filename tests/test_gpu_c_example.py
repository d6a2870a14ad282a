"""The plain-C example (examples/render_uniform.c) on the GPU: a uniform octree rendered through
po_render_host matches the constant-medium closed form C = S(kY00)(1 - T) + T bg on every pixel."""
import subprocess

import pytest

pytestmark = pytest.mark.gpu


def test_c_example_runs():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2103_14024_b200 import _build
    exe = _build.build_example()
    out = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    assert out.stdout.strip().endswith("OK")
