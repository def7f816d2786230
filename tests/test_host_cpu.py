"""CPU-only tests: the C-ABI library loads and exports every declared symbol,
the host-side schedule/geometry logic, workloads, and the error contract.
No kernel is launched here."""

import re
from pathlib import Path

import numpy as np
import pytest

from paper_2506_23568_b200 import _native, ffbp, model, workloads
from paper_2506_23568_b200.dist import chunk_size, shard_range
from paper_2506_23568_b200.errors import ConfigError

REPO = Path(__file__).resolve().parents[1]


def _header_symbols():
    text = (REPO / "include" / "hhsar_b200.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:int|const char \*)\s*(hhsar_\w+)\(", text, re.M)))


def test_library_exports_every_header_symbol():
    lib = _native.library(require_gpu=False)
    declared = _header_symbols()
    assert len(declared) >= 18
    for name in declared:
        assert hasattr(lib, name), name
    assert set(declared) == set(_native.SIGNATURES), "binding and header disagree"


def test_struct_layout_matches_library():
    lib = _native.library(require_gpu=False)
    out = np.zeros(16, dtype=np.int64)
    n = lib.hhsar_abi_layout(out.ctypes.data, 16)
    assert n == 9
    assert out[0] == _native.GEOM_DTYPE.itemsize
    assert out[1] == _native.GRID_DTYPE.itemsize


def test_library_is_sm100a():
    import subprocess
    res = subprocess.run(["cuobjdump", "--list-elf", str(_native.LIB_PATH)], capture_output=True,
                         text=True)
    assert "sm_100a" in res.stdout


def test_leaf_bounds_match_reference_partition():
    # model.py:377-382: first n mod L leaves get one extra element
    b = model.leaf_bounds(4000 * 8, 9)
    sizes = np.diff(b)
    assert sizes.size == 256 and sizes.sum() == 32000 and set(sizes) == {125}
    b = model.leaf_bounds(81, 3)
    assert list(np.diff(b)) == [21, 20, 20, 20]
    with pytest.raises(ConfigError):
        model.leaf_bounds(3, 4)


@pytest.mark.parametrize("levels,factor", [(3, 2), (7, 2), (7, 4), (6, 4), (12, 4), (11, 2)])
def test_schedule_levels_and_fanouts(levels, factor):
    n = 2 ** (levels - 1) * 3 + 5
    s = ffbp.Schedule(n, levels, factor)
    step = int(np.log2(factor))
    assert s.grid_levels == list(range(1, levels, step))
    for (a, b), lev in zip(s.level_slices, s.grid_levels):
        assert b - a == 2 ** (levels - lev)
        g = s.grids[a:b]
        assert g["start"][0] == 0 and g["stop"][-1] == n
        assert np.all(g["start"][1:] == g["stop"][:-1])
    for k, fan in enumerate(s.fanouts):
        (a0, a1), (b0, b1) = s.level_slices[k], s.level_slices[k + 1]
        assert (a1 - a0) == (b1 - b0) * fan
    assert s.final_children == s.level_slices[-1][1] - s.level_slices[-1][0]
    assert np.all(s.grids["is_leaf"][:s.level_slices[0][1]] == 1)


def test_schedule_rejects_bad_factor():
    with pytest.raises(ConfigError):
        ffbp.Schedule(100, 4, 3)


def test_geom_constants_bit_identical_to_reference_formulas():
    w = workloads.config(0)
    g = ffbp.make_geom(w.region, w.freqs, 1.4, 0.25, 4, 1e-8)[0]
    k_min, k_max = w.freqs.k_min, w.freqs.k_max
    assert g["c_uv"] == k_max / np.pi
    assert g["c_nhi"] == k_max / (2.0 * (2.0 * np.pi))
    assert g["c_nlo"] == k_min / (2.0 * (2.0 * np.pi))
    assert g["step"] == 1.0 / 1.4
    assert g["max_step"] == 0.5 * w.region.diagonal


def test_params_validation_matches_reference():
    with pytest.raises(ConfigError):
        ffbp.FfbpParams(levels=0)
    with pytest.raises(ConfigError):
        ffbp.FfbpParams(gamma=0.9)
    with pytest.raises(ConfigError):
        ffbp.FfbpParams(kernel="nearest")
    with pytest.raises(ConfigError):
        ffbp.FfbpParams(margin=1.5)


def test_default_levels():
    ap = model.SyntheticAperture(np.zeros((33 * 33, 3)), 33, 33)
    assert ffbp.default_levels(ap) == 3
    ap = model.SyntheticAperture(np.zeros((8 * 4000, 3)), 8, 4000)
    assert ffbp.default_levels(ap) == 1


@pytest.mark.parametrize("n,world", [(10, 3), (2560000, 8), (7, 8), (1, 1)])
def test_shard_ranges_tile_exactly(n, world):
    ranges = [shard_range(n, r, world) for r in range(world)]
    assert ranges[0][0] == 0 and ranges[-1][1] == n
    for (a, b), (c, d) in zip(ranges[:-1], ranges[1:]):
        assert b == c
    sizes = [b - a for a, b in ranges]
    assert max(sizes) - min(sizes) <= 1 and max(sizes) <= chunk_size(n, world)


def test_workloads_match_baseline_shapes():
    w0 = workloads.config(0)
    assert w0.n_elements == 1024 and w0.freqs.count == 64 and w0.dims == (64, 64, 32)
    assert w0.upsample * w0.freqs.count == 512
    # Morton 4x4 blocks: every contiguous run of 16 elements is one 4x4 block
    el = np.asarray(w0.aperture.elements)
    for b in range(0, 1024, 16):
        blk = el[b:b + 16, :2]
        assert np.ptp(blk[:, 0]) < 0.0135 and np.ptp(blk[:, 1]) < 0.0135
    w1 = workloads.config(1)
    assert w1.n_elements == 32000 and w1.freqs.count == 256 and w1.dims == (200, 200, 64)
    assert w1.upsample * w1.freqs.count == 1024
    assert w1.bpa_units == 200 * 200 * 64 * 32000
    w3 = workloads.config(3, frames=64)
    assert w3.n_elements == 512 and w3.freqs.count == 512
    # seeded: identical on regeneration
    assert np.array_equal(workloads.config(1).aperture.elements, w1.aperture.elements)


def test_validate_geometry_contract():
    ap = model.SyntheticAperture(np.array([[0.0, 0.0, 0.01]]), 1, 1)
    with pytest.raises(ConfigError):
        model.validate_geometry(ap, model.ImagingRegion(-1, 1, -1, 1, 0.005, 1))
    model.validate_geometry(ap, model.ImagingRegion(-1, 1, -1, 1, 0.02, 1))


def test_product_path_fails_loudly_without_gpu(monkeypatch):
    """No CPU fallback: on a GPU-less host the first product call raises."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2506_23568_b200 import NativeUnavailableError, bpa_reconstruct
    w = workloads.config(0)
    cube = model.DataCube(np.zeros((w.n_elements, w.freqs.count), np.complex64), w.aperture,
                          w.freqs)
    with pytest.raises(NativeUnavailableError):
        bpa_reconstruct(cube, w.region, dims=(4, 4, 4))


# ---- metrics: host-side parts (psf_metrics, profile_cut, argument checks) ----

def test_psf_metrics_matches_reference():
    from goldens import load_npz as load
    from paper_2506_23568_b200 import metrics
    z = load("metrics")
    rep = metrics.psf_metrics(z["psf_profile"], 0.002)
    got = np.array([rep.mainlobe_width_mm, rep.pslr_db, rep.islr_db, rep.peak_position_m])
    assert np.allclose(got, z["psf"], rtol=1e-12, atol=1e-12)
    assert set(rep.to_dict()) == {"mainlobe_width_mm", "pslr_db", "islr_db", "peak_position_m"}


def test_metrics_errors_match_reference():
    """Same exception classes and messages as the reference for every
    rejected input (the GPU is never reached: all checks come first)."""
    from goldens import load_npz as load
    from paper_2506_23568_b200 import metrics
    from paper_2506_23568_b200.bpa import ImageVolume
    z = load("metrics")
    prof = z["psf_profile"]
    ref = ImageVolume(z["ref"], z["origin"], z["step"])
    calls = [lambda: metrics.psf_metrics(np.ones(64, complex), 0.002),
             lambda: metrics.psf_metrics(np.zeros(64, complex), 0.002),
             lambda: metrics.psf_metrics(prof[:3], 0.002),
             lambda: metrics.psf_metrics(prof, 0.0),
             lambda: metrics.psf_metrics(np.exp(-np.linspace(-2, 2, 65) ** 2).astype(complex),
                                         0.01),
             lambda: metrics.psf_metrics(np.array([8.2, 8.0, 8.5, 8.6, 9.0, 8.7, 8.1, 8.3, 1.0],
                                                  complex), 0.01),
             lambda: metrics.max_intensity_projection(ref, "w"),
             lambda: metrics.max_intensity_projection(ref, 3),
             lambda: metrics.max_intensity_projection(ref, "z", 0.0),
             lambda: metrics.psnr(ref, ImageVolume(z["ref"], z["origin"] + 1.0, z["step"]))]
    for fn, want in zip(calls, z["errors"]):
        with pytest.raises(Exception) as exc:
            fn()
        assert f"{type(exc.value).__name__}: {exc.value}" == str(want)


def test_profile_cut_matches_reference():
    from goldens import load_npz as load
    from paper_2506_23568_b200 import metrics
    from paper_2506_23568_b200.bpa import ImageVolume
    z = load("metrics")
    cut, sp = metrics.profile_cut(ImageVolume(z["ref"], z["origin"], z["step"]), "y",
                                  (0.0, 0.0, 0.23))
    assert np.array_equal(cut, z["cut_y"]) and sp == float(z["cut_spacing"])


def test_leaf_range_gate_host_restatement():
    """ffbp.leaf_range_gate (the host restatement of hhsar_leaf_range_gate):
    points whose compressed n lies in a leaf's near band, seen from any
    element of the leaf, fall inside the gate with the leaf kernel's fast-
    path margins (>= 1 bin above b0, <= 3 bins below b0 + w - 1); the window
    is a multiple of 32 bins and clipped at the profile end."""
    from types import SimpleNamespace
    rng = np.random.default_rng(5)
    k_min, k_max = 2 * np.pi * 77e9 / model.C_LIGHT, 2 * np.pi * 81e9 / model.C_LIGHT
    c_nhi, c_nlo = k_max / (4 * np.pi), k_min / (4 * np.pi)
    geom = _native.host_struct(_native.GEOM_DTYPE, dict(c_nhi=c_nhi, c_nlo=c_nlo,
                                                         step=1 / 1.4, tol=1e-9))
    ext = np.array([-0.01, 0.006, 0.002, 0.018])           # lateral element box
    descs = np.zeros(2, dtype=_native.GRID_DTYPE)
    descs["ext"][0] = ext
    descs["box"][0] = [ext[0], ext[2], -0.004, ext[1], ext[3], 0.003]
    descs["origin"][0] = [0.0, 0.0, 4.0]
    descs["near_lo"][0] = [0, 0, 3]
    descs["near_hi"][0] = [0, 0, 12]
    lat = SimpleNamespace(descs=descs, geom=geom)
    sched = SimpleNamespace(level_slices=[(0, 1), (1, 2)])
    dt = 2.0 * 0.004 / model.C_LIGHT                       # 4 mm range bins
    b0, w = ffbp.leaf_range_gate(lat, sched, dt, 4096)
    assert w % 32 == 0 and 0 < b0 < 4096 - w
    n_lo, n_hi = 4.0 + 3 / 1.4, 4.0 + 12 / 1.4
    # random points above the array; keep those on the near band's n range
    p = np.stack([rng.uniform(-0.4, 0.4, 400000), rng.uniform(-0.4, 0.4, 400000),
                  rng.uniform(0.05, 0.6, 400000)], axis=1)
    vs = np.array([[ext[i], ext[2 + j], 0.0] for i in (0, 1) for j in (0, 1)])
    r = sum(np.linalg.norm(p - v, axis=1) for v in vs)
    gap = 4 * (ext[1] - ext[0]) ** 2 + 4 * (ext[3] - ext[2]) ** 2
    n = c_nhi * np.sqrt(r * r - gap) - c_nlo * r
    p = p[(n >= n_lo) & (n <= n_hi)]
    assert len(p) > 1000
    e = np.stack([rng.uniform(ext[0], ext[1], 64), rng.uniform(ext[2], ext[3], 64),
                  rng.uniform(-0.004, 0.003, 64)], axis=1)
    bins = np.linalg.norm(p[:, None, :] - e[None, :, :], axis=2) * (2.0 / (model.C_LIGHT * dt))
    assert bins.min() - b0 >= 1.0 and bins.max() - b0 <= w - 4.0
    # tight: the near band's own delay span plus the pads, not the profile
    assert w <= (bins.max() - bins.min()) + 64
    # clipped at the profile end
    b0c, wc = ffbp.leaf_range_gate(lat, sched, dt, b0 + w - 7)
    assert b0c == b0 and b0c + wc == b0 + w - 7


def test_check_grids_reference_order():
    """The vectorised SubimageGrid health check raises for the FIRST failing
    grid in the reference's order -- each leaf as built, then after its
    delay mask (ffbp.py:331-335), then the parents level by level -- with
    the reference's message (ffbp.py:127-133)."""
    from types import SimpleNamespace
    from paper_2506_23568_b200 import _native, ffbp
    from paper_2506_23568_b200.errors import NumericDomainError
    sched = ffbp.Schedule(64, 4)  # 8 leaves, 4 + 2 parents
    d = np.zeros(sched.n_grids, dtype=_native.GRID_DTYPE)
    d["core_lo"] = 0
    d["core_hi"] = 9  # 10 x 10 x 10 = 1,000 core points per grid
    run = SimpleNamespace(sched=sched, lattices=SimpleNamespace(descs=d))
    stats = np.zeros((sched.n_grids, _native.GRID_STATS), dtype=np.int64)
    stats[:, 1] = stats[:, 3] = 1000
    ffbp.check_grids(run, stats)  # healthy: no raise
    s2 = stats.copy()
    s2[3, 3] = 400   # leaf 3 after its delay mask: 60% masked
    s2[9, 1] = 100   # a parent: 90% masked -- later in the reference's order
    with pytest.raises(NumericDomainError, match="60% of core lattice points"):
        ffbp.check_grids(run, s2)
    s3 = stats.copy()
    s3[5, 1] = 490   # leaf 5 as built: 51% masked beats leaf 6's masked state
    s3[6, 3] = 0
    with pytest.raises(NumericDomainError, match="51% of core lattice points"):
        ffbp.check_grids(run, s3)
    s4 = stats.copy()
    s4[sched.level_slices[1][0] + 1, 1] = 500  # exactly 50%: the reference raises at >= 0.5
    with pytest.raises(NumericDomainError, match="50% of core lattice points"):
        ffbp.check_grids(run, s4)
