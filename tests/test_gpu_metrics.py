"""GPU image-quality metrics (hhsar_volume_dot / hhsar_volume_residual /
hhsar_mip) against the reference's own metrics.py outputs
(tests/golden/metrics.npz, made by tests/golden/make_golden.py metrics).

Bars: psnr within 1e-9 dB on complex128 volumes (float64 accumulation, a
different summation order than numpy), exactly the 200 dB sentinel where the
reference returns it; MIP within 1e-12 (float64 magnitudes, same dB map).
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def z():
    from goldens import load_npz
    return load_npz("metrics")


@pytest.fixture(scope="module")
def mt():
    from paper_2506_23568_b200 import _native, metrics
    _native.library()  # fail loudly (no skip) when the CUDA library is unusable
    return metrics


def _vol(z, values):
    from paper_2506_23568_b200.bpa import ImageVolume
    return ImageVolume(values, z["origin"], z["step"])


def test_psnr_matches_reference(z, mt):
    assert abs(mt.psnr(_vol(z, z["ref"]), _vol(z, z["noisy"])) - float(z["psnr_noisy"])) < 1e-9
    assert mt.psnr(_vol(z, z["ref"]), _vol(z, z["ref"].copy())) == float(z["psnr_same"]) == 200.0
    assert mt.psnr(_vol(z, z["ref"]), _vol(z, z["ref"] * (0.3 + 2.1j))) == float(z["psnr_scaled"])
    zero = np.zeros(z["ref"].shape, complex)
    assert abs(mt.psnr(_vol(z, z["ref"]), _vol(z, zero)) - float(z["psnr_zero_test"])) < 1e-9


def test_psnr_complex64_volumes(z, mt):
    """complex64 inputs (the GPU volume type) against the reference run on
    the same samples promoted to complex128."""
    got = mt.psnr(_vol(z, z["ref64"]), _vol(z, z["noisy64"]))
    assert abs(got - float(z["psnr_noisy64"])) < 1e-6
    assert mt.psnr(_vol(z, z["ref64"]), _vol(z, z["ref64"].copy())) == 200.0


def test_psnr_device_tensors(z, mt):
    import torch
    r = torch.from_numpy(z["ref64"]).cuda()
    t = torch.from_numpy(z["noisy64"]).cuda()
    assert abs(mt.psnr_device(r, t) - float(z["psnr_noisy64"])) < 1e-6


@pytest.mark.parametrize("axis", ["x", "y", "z"])
@pytest.mark.parametrize("floor", [-40.0, -25.0])
def test_mip_matches_reference(z, mt, axis, floor):
    got = mt.max_intensity_projection(_vol(z, z["ref"]), axis, floor)
    want = z[f"mip_{axis}_{int(-floor)}"]
    assert got.shape == want.shape and got.dtype == np.float64
    assert np.max(np.abs(got - want)) < 1e-12


def test_mip_complex64_and_zero(z, mt):
    got = mt.max_intensity_projection(_vol(z, z["ref64"]), 2)
    want = z["mip_z_40"]
    assert np.max(np.abs(got - want)) < 1e-6  # complex64 samples
    zero = mt.max_intensity_projection(_vol(z, np.zeros(z["ref"].shape, complex)), 1)
    assert np.array_equal(zero, z["mip_zero"])


def test_mip_large_volume_against_numpy(mt):
    """A volume with rows longer than a warp and every axis: same as the
    numpy restatement of metrics.py:183-190."""
    import torch
    gen = torch.Generator(device="cuda").manual_seed(7)
    v = torch.randn((37, 29, 301), dtype=torch.complex64, device="cuda", generator=gen)
    host = v.cpu().numpy().astype(np.complex128)
    for ax in range(3):
        mip = np.abs(host).max(axis=ax)
        want = (np.maximum(20 * np.log10(mip / mip.max()), -40.0) + 40.0) / 40.0
        got = mt.mip_device(v, ax).cpu().numpy()
        assert np.max(np.abs(got - want)) < 1e-12
