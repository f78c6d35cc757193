"""Host-side logic (no GPU): the reference-interface mirror validates,
maps configs and raises exactly like the reference."""

import numpy as np
import pytest

from oracle import depthfill_oracle as O
from paper_1802_00036_b200 import _lib, synth
from paper_1802_00036_b200.completion import (BlurMode, FillMode, MultiscaleConfig, PipelineConfig, fit_to_frame,
                                              raise_for_status, to_dfc_config)
from paper_1802_00036_b200.domain import (DegenerateInputError, DepthMap, DepthRangeError, Kernel, KernelShape,
                                          density, kernel_offsets, make_kernel)


@pytest.mark.parametrize("shape", list(KernelShape))
@pytest.mark.parametrize("size", [3, 5, 7, 9, 31])
def test_kernels_match_oracle(shape, size):
    k = make_kernel(shape, size)
    ref = O.make_kernel(O.KernelShape(shape.value), size)
    assert np.array_equal(k.bits, ref)
    assert np.array_equal(kernel_offsets(k), O.kernel_offsets(ref))
    assert k.named() is not None


def test_kernel_popcounts_fig3():
    assert [int(make_kernel(s, 5).bits.sum()) for s in (KernelShape.CROSS, KernelShape.DIAMOND,
                                                        KernelShape.CIRCLE, KernelShape.FULL)] == [9, 13, 21, 25]
    with pytest.raises(ValueError):
        make_kernel(KernelShape.FULL, 4)


def test_pipeline_config_validation_messages():
    with pytest.raises(ValueError, match="dilation_size must be an odd integer >= 3, got 4"):
        PipelineConfig(dilation_size=4)
    with pytest.raises(ValueError, match="large_fill_max_iters must be >= 1"):
        PipelineConfig(large_fill_max_iters=0)
    with pytest.raises(ValueError, match="gaussian_sigma must be positive"):
        PipelineConfig(gaussian_sigma=0)
    with pytest.raises(ValueError, match="bilateral sigmas must be positive"):
        PipelineConfig(bilateral_sigma_space=-1)


def test_fit_to_frame_matches_oracle():
    for h, w in ((1, 1), (2, 3), (3, 40), (10, 10), (352, 1216)):
        a = fit_to_frame(PipelineConfig(), h, w)
        b = O.fit_to_frame(O.OracleConfig(), h, w)
        assert (a.dilation_size, a.closure_size, a.small_fill_size, a.large_fill_size) == \
               (b.dilation_size, b.closure_size, b.small_fill_size, b.large_fill_size)


def test_depthmap_validation_order():
    with pytest.raises(ValueError, match="2-D"):
        DepthMap(np.zeros(3, np.float32))
    with pytest.raises(ValueError, match="finite"):
        DepthMap(np.array([[np.nan, -1.0]], np.float32))
    with pytest.raises(ValueError, match="non-negative"):
        DepthMap(np.array([[1.0, -1.0]], np.float32))
    m = DepthMap(np.array([[0.0, 0.2, 0.1]], np.float32))
    assert not m.values.flags.writeable
    assert density(m) == pytest.approx(1 / 3)


def test_to_dfc_config_mapping():
    pytest.importorskip("torch")
    c = to_dfc_config(PipelineConfig(dilation_shape=KernelShape.CROSS, blur_mode=BlurMode.GAUSSIAN,
                                     fill_mode=FillMode.PARTIAL, max_depth=120.0, exact_blur=True),
                      MultiscaleConfig(), np.array([[0, 1], [1, 0]]))
    assert c.dilation_shape == 2 and c.blur_mode == 4 and c.fill_mode == 1 and c.max_depth == 120.0
    assert c.flags & _lib.F_EXACT_BLUR
    assert c.multiscale == 1 and (c.near_shape, c.near_size, c.far_shape, c.far_size) == (0, 7, 3, 5)
    assert c.custom_n == 2 and c.custom_offsets[1] == 1


def test_raise_for_status_priority():
    raise_for_status(np.array([0, 0x100], np.int32), 100.0)  # FALLBACK alone is informational
    with pytest.raises(DegenerateInputError, match="frame 1"):
        raise_for_status(np.array([0, 0x4 | 0x8], np.int32), 100.0)
    with pytest.raises(DepthRangeError):
        raise_for_status(np.array([0x8], np.int32), 100.0)
    with pytest.raises(ValueError, match="finite"):
        raise_for_status(np.array([0x1 | 0x4], np.int32), 100.0)


def test_synth_deterministic_and_density():
    a = synth.make_frame(synth.CONFIG_SPECS[1], [1, 5])
    b = synth.make_frame(synth.CONFIG_SPECS[1], [1, 5])
    assert np.array_equal(a, b)
    d = (a > 0.1).mean()
    assert 0.03 < d < 0.07
    assert a.max() < 100.0 and (a[a > 0] >= 0.5).all()
    top = int(round(120 * 352 / 352))
    assert (a[:top] == 0).all()


def test_custom_kernel_named_detection():
    assert Kernel(make_kernel(KernelShape.CIRCLE, 7).bits).named() == (KernelShape.CIRCLE, 7)
    odd = np.zeros((5, 5), bool)
    odd[2] = True
    odd[0, 0] = True
    assert Kernel(odd).named() is None
