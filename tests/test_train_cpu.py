"""Host logic of the NEXT f2 optimisation loop (paper_2103_14024_b200/train.py): the PSNR
definition and the early-stopping rule, checked without a GPU."""
import math

from paper_2103_14024_b200.train import psnr_from_sse, should_stop


def test_psnr_definition():
    # MSE 0.01 -> 20 dB, MSE 1e-4 -> 40 dB (colours in [0, 1]); a perfect fit is +inf
    assert abs(psnr_from_sse(0.01 * 300, 300) - 20.0) < 1e-12
    assert abs(psnr_from_sse(1e-4 * 12, 12) - 40.0) < 1e-12
    assert psnr_from_sse(0.0, 10) == math.inf


def test_early_stopping_rule():
    assert not should_stop([], 1)
    assert not should_stop([20.0], 1)
    assert not should_stop([20.0, 21.0, 22.0], 1)       # still improving
    assert should_stop([20.0, 21.0, 20.5], 1)           # one epoch without improvement
    assert not should_stop([20.0, 21.0, 20.5], 2)       # patience 2 waits one more epoch
    assert should_stop([20.0, 21.0, 20.5, 20.9], 2)
    assert not should_stop([20.0, 21.0, 20.5, 21.5], 2)  # a new best resets the count
