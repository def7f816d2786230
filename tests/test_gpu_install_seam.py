"""The operator-level seam: the reference's own pipeline running on the GPU
operators.

``paper_2506_23568_b200._kernels.install(hhsar)`` points the reference's
plugin symbols (/root/reference/pkg/src/hhsar/_kernels.py:18-31, :98-110,
:354-378, spectrum.py:365) at hhsar_bp_gather / hhsar_lattice_interp /
hhsar_invert_newton.  The reference package is the unmodified copy staged in
oracle/_ref by oracle.reference.stage() (build()); its Python orchestration
(bpa.py, ffbp.py, spectrum.py) runs unchanged on top.  Checked against the
same staged reference on its Numba kernels: images within the float32
budget, identical validity masks and provenance, and the reference test
suite's identities (test_bpa.py:30-43, test_ffbp.py:34-72) at float32
tolerances.
"""

import numpy as np
import pytest

from goldens import load, rel_l2

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ref():
    from oracle import reference
    if not reference.staged():
        pytest.fail("reference not staged in oracle/_ref (run __graft_entry__.build())")
    return reference.load()


@pytest.fixture(scope="module")
def case(ref):
    c = load("small")
    z = c.z
    ap = ref.SyntheticAperture(elements=np.asarray(z["elements"], dtype=float),
                               nx=int(z["nxny"][0]), ny=int(z["nxny"][1]))
    f = z["freqs"]
    freqs = ref.FrequencyGrid(float(f[0]), float(f[1]), int(f[2]))
    region = ref.ImagingRegion(*(float(v) for v in z["region"]))
    cube = ref.DataCube(values=np.asarray(z["cube"]), aperture=ap, freqs=freqs)
    return dict(ap=ap, freqs=freqs, region=region, cube=cube, dims=c.dims)


@pytest.fixture(scope="module")
def numba_results(ref, case):
    """The staged reference on its own Numba kernels."""
    c = case
    out = {"bpa": ref.bpa_reconstruct(c["cube"], c["region"], dims=c["dims"])}
    for kern in ("linear", "cubic"):
        out[kern] = ref.hhffbpa_reconstruct(c["cube"], c["region"], c["dims"],
                                            ref.FfbpParams(levels=3, kernel=kern))
    tree = ref.partition_subarrays(c["ap"], 3)
    out["grid"] = ref.build_subimage_grid(c["ap"], tree.levels[0][0], c["region"], c["freqs"])
    return out


@pytest.fixture
def gpu_ops(ref):
    from paper_2506_23568_b200 import _kernels
    restore = _kernels.install(ref)
    yield ref
    restore()


def test_reference_bpa_on_gpu_gather(gpu_ops, case, numba_results):
    got = gpu_ops.bpa_reconstruct(case["cube"], case["region"], dims=case["dims"])
    assert rel_l2(got.values, numba_results["bpa"].values) < 1e-4
    assert got.provenance == numba_results["bpa"].provenance


@pytest.mark.parametrize("kernel", ["linear", "cubic"])
def test_reference_hhffbpa_on_gpu_operators(gpu_ops, case, numba_results, kernel):
    got = gpu_ops.hhffbpa_reconstruct(case["cube"], case["region"], case["dims"],
                                      gpu_ops.FfbpParams(levels=3, kernel=kernel))
    want = numba_results[kernel]
    assert rel_l2(got.values, want.values) < 1e-3
    for key in ("level_points", "merge_flags", "final_flags", "flagged_fraction"):
        assert got.provenance[key] == want.provenance[key], key


def test_reference_grid_on_gpu_newton(gpu_ops, case, numba_results):
    tree = gpu_ops.partition_subarrays(case["ap"], 3)
    got = gpu_ops.build_subimage_grid(case["ap"], tree.levels[0][0], case["region"],
                                      case["freqs"])
    want = numba_results["grid"]
    assert got.dims == want.dims and np.array_equal(got.origin, want.origin)
    assert np.array_equal(got.valid, want.valid)
    v = want.valid
    assert np.max(np.abs(got.positions[v] - want.positions[v])) < 1e-9


def test_reference_identities_on_gpu_operators(gpu_ops, case):
    """test_ffbp.py:34-42 (M=1 == BPA), test_bpa.py:30-43 (selection and
    empty selection) and the partition additivity / linearity of
    test_ffbp.py:45-72, at float32 tolerances (the reference asserts
    1e-12 .. 1e-13 on float64 kernels)."""
    ref, c = gpu_ops, case
    bpa = ref.bpa_reconstruct(c["cube"], c["region"], dims=c["dims"])
    one = ref.hhffbpa_reconstruct(c["cube"], c["region"], c["dims"], ref.FfbpParams(levels=1))
    assert np.array_equal(one.values, bpa.values)  # same GPU kernel, same inputs
    prof = ref.range_compress(c["cube"], 8)
    pts = bpa.grid_points()[::7]
    n = c["ap"].n_elements
    whole = ref.backproject(prof, slice(None), pts)
    sub = ref.Subarray(0, n)
    assert rel_l2(ref.backproject(prof, sub, pts), whole) < 1e-6
    assert np.all(ref.backproject(prof, slice(0, 0), pts) == 0)
    halves = (ref.backproject(prof, ref.Subarray(0, n // 2), pts)
              + ref.backproject(prof, ref.Subarray(n // 2, n), pts))
    assert rel_l2(halves, whole) < 1e-5
    cube2 = ref.DataCube(values=np.asarray(c["cube"].values) * (2.0 - 1.5j), aperture=c["ap"],
                         freqs=c["freqs"])
    a = ref.hhffbpa_reconstruct(c["cube"], c["region"], c["dims"], ref.FfbpParams(levels=3))
    b = ref.hhffbpa_reconstruct(cube2, c["region"], c["dims"], ref.FfbpParams(levels=3))
    assert rel_l2(b.values, (2.0 - 1.5j) * a.values) < 1e-5
