"""Pin the CPU oracle against outputs of the reference itself.

The golden .npz files are produced by tests/golden/make_golden.py, which runs
the unmodified reference (Numba path).  The oracle is float64 like the
reference, so agreement is near round-off; grid metadata and masks must be
bit-identical.  These tests run on CPU (no `gpu` marker).
"""

import numpy as np
import pytest

import oracle
from goldens import grid_valid, load, provenance, rel_l2


@pytest.fixture(scope="module")
def small():
    return load("small")


def _prof_for(case):
    return oracle.range_compress(case.cube, 8)


def test_range_compress_matches_reference(small):
    prof = _prof_for(small)
    want = small.z["envelopes"]
    assert rel_l2(prof.envelopes, want) < 1e-13
    t0, dt, k_ref = small.z["profile_meta"]
    assert prof.t0 == t0 and prof.dt == dt and prof.k_ref == k_ref


def test_bpa_volume_matches_reference(small):
    vals, origin, step, prov = oracle.bpa_reconstruct(small.cube, small.region, small.dims)
    assert rel_l2(vals, small.z["bpa"]) < 1e-12
    assert prov == {"algorithm": "bpa", "upsample": 8, "dims": list(small.dims)}


def test_backproject_probes_and_subarray(small):
    prof = _prof_for(small)
    got = oracle.backproject(prof, slice(None), small.z["probes"])
    assert np.max(np.abs(got - small.z["probe_values"])) < 1e-12 * np.abs(got).max()
    sub = oracle.backproject(prof, (10, 33), small.z["probes"])
    assert np.max(np.abs(sub - small.z["probe_values_sub"])) < 1e-12 * np.abs(sub).max()


def test_empty_selection_is_zero(small):
    prof = _prof_for(small)
    out = oracle.backproject(prof, slice(0, 0), small.z["probes"])
    assert np.all(out == 0)


@pytest.mark.parametrize("tag,levels,kernel", [("m2", 2, "linear"), ("m3", 3, "linear"),
                                               ("m3c", 3, "cubic")])
def test_hhffbpa_small_matches_reference(small, tag, levels, kernel):
    vals, _, _, prov = oracle.hhffbpa_reconstruct(small.cube, small.region, small.dims,
                                                  levels=levels, kernel=kernel)
    assert rel_l2(vals, small.z["hh_" + tag]) < 1e-10
    want = provenance(small.z, "hh_" + tag)
    assert prov["level_points"] == want["level_points"]
    assert prov["merge_flags"] == want["merge_flags"]
    assert prov["final_flags"] == want["final_flags"]


def _oracle_grids(case, levels, pad=4, prune=False, n_levels=None):
    k_min, k_max = case.freqs.k_min, case.freqs.k_max
    tiers = oracle.tree_levels(case.aperture.n_elements, levels)
    el = np.asarray(case.aperture.elements)
    out = []
    for tier in tiers[:n_levels or levels - 1]:
        for a, b in tier:
            out.append(oracle.build_grid(oracle.extents_of(el, a, b), case.region, k_min,
                                         k_max, pad=pad, start=a, stop=b, prune=prune))
    return out


@pytest.mark.parametrize("prune", [False, True])
def test_grid_metadata_and_masks_bit_exact(small, prune):
    grids = _oracle_grids(small, 3, prune=prune)
    z = small.z
    assert np.array_equal([g.dims for g in grids], z["grid_dims"])
    assert np.array_equal(np.array([g.origin for g in grids]), z["grid_origin"])
    assert np.array_equal(np.array([g.step for g in grids]), z["grid_step"])
    assert np.array_equal([[c for ab in g.core for c in ab] for g in grids], z["grid_core"])
    assert np.array_equal(np.array([g.ext for g in grids]), z["grid_ext"])
    for g, want in zip(grids, grid_valid(z, "grid")):
        assert np.array_equal(g.valid, want)
    pos = np.concatenate([g.positions.reshape(-1, 3) for g in grids])
    valid = np.concatenate([g.valid.ravel() for g in grids])
    assert np.max(np.abs(pos[valid] - z["grid_positions"][valid])) < 1e-9


def test_default_pad_grid(small):
    el = np.asarray(small.aperture.elements)
    a, b = oracle.tree_levels(small.aperture.n_elements, 3)[0][0]
    g = oracle.build_grid(oracle.extents_of(el, a, b), small.region, small.freqs.k_min,
                          small.freqs.k_max, pad=2, start=a, stop=b)
    assert g.dims == tuple(small.z["grid_pad2_dims"][0])
    assert np.array_equal(g.valid, grid_valid(small.z, "grid_pad2")[0])


def test_leaf_and_merge_pair(small):
    prof = _prof_for(small)
    grids = _oracle_grids(small, 3)
    leaves = [oracle.level1(prof, g) for g in grids[:4]]
    got = np.concatenate([l.values.ravel() for l in leaves])
    want = small.z["leaf_values"]
    assert np.max(np.abs(got - want)) <= 1e-12 * np.abs(want).max()
    valid = np.unpackbits(small.z["leaf_valid"])[:got.size].astype(bool)
    assert np.array_equal(np.concatenate([l.grid.valid.ravel() for l in leaves]), valid)
    merged, flagged = oracle.merge_children(leaves[:2], grids[4], small.freqs.k_min,
                                            small.freqs.k_max)
    assert rel_l2(merged.values, small.z["merge01"]) < 1e-11
    assert flagged == int(small.z["merge01_flagged"])
    with pytest.raises(oracle.OracleConfigError):
        oracle.merge_children([leaves[0], leaves[2]], grids[4], small.freqs.k_min,
                              small.freqs.k_max)


@pytest.mark.parametrize("kernel", ["linear", "cubic"])
def test_lattice_interpolation(small, kernel):
    v, ok = oracle.interpolate(small.z["interp_lattice"], small.z["interp_coords"], kernel)
    assert np.array_equal(ok, small.z[f"interp_{kernel}_ok"])
    assert np.max(np.abs(v - small.z[f"interp_{kernel}"])) < 1e-13


def test_newton_inversion(small):
    z = small.z
    pos, ok, it = oracle.invert_newton(tuple(z["newton_ext"]), z["newton_targets"],
                                       z["newton_guesses"], small.freqs.k_min,
                                       small.freqs.k_max, max_step=float(z["newton_max_step"]))
    assert np.array_equal(ok, z["newton_ok"])
    assert np.max(np.abs(pos[ok] - z["newton_pos"][ok])) < 1e-9
    assert np.array_equal(pos[~ok], z["newton_pos"][~ok])


def test_analytic_maps(small):
    z = small.z
    ext = tuple(z["newton_ext"])
    uvn = oracle.llt_forward(ext, z["map_points"], small.freqs.k_min, small.freqs.k_max)
    assert np.array_equal(uvn, z["map_uvn"])
    ph = oracle.sdc_phase(ext, z["map_points"], small.freqs.k_min, small.freqs.k_max)
    assert np.array_equal(ph, z["map_phase"])


def test_medium_bpa_and_hhffbpa():
    m = load("medium")
    vals, *_ = oracle.bpa_reconstruct(m.cube, m.region, m.dims)
    assert rel_l2(vals, m.z["bpa"]) < 1e-12
    for lv in (3, 4):
        vals, _, _, prov = oracle.hhffbpa_reconstruct(m.cube, m.region, m.dims, levels=lv)
        assert rel_l2(vals, m.z[f"hh_m{lv}"]) < 1e-10
        assert prov["level_points"] == provenance(m.z, f"hh_m{lv}")["level_points"]


@pytest.fixture(scope="module")
def config0():
    return load("config0")


def test_config0_bpa(config0):
    vals, *_ = oracle.bpa_reconstruct(config0.cube, config0.region, config0.dims)
    assert rel_l2(vals, config0.z["bpa"]) < 1e-6  # golden stored as complex64


@pytest.mark.parametrize("tag,factor", [("m7", 2), ("f4", 4)])
def test_config0_hhffbpa(config0, tag, factor):
    vals, _, _, prov = oracle.hhffbpa_reconstruct(config0.cube, config0.region,
                                                  config0.dims, levels=7,
                                                  merge_factor=factor)
    assert rel_l2(vals, config0.z["hh_" + tag]) < 1e-6
    want = provenance(config0.z, "hh_" + tag)
    assert prov["level_points"] == want["level_points"]
    assert prov["merge_flags"] == want["merge_flags"]
    assert prov["final_flags"] == want["final_flags"]


def test_config0_all_grid_masks(config0):
    grids = _oracle_grids(config0, 7, prune=True)
    z = config0.z
    assert np.array_equal([g.dims for g in grids], z["grid_dims"])
    assert np.array_equal(np.array([g.origin for g in grids]), z["grid_origin"])
    assert np.array_equal([[c for ab in g.core for c in ab] for g in grids], z["grid_core"])
    masks = grid_valid(z, "grid")
    mism = sum(int((g.valid != w).sum()) for g, w in zip(grids, masks))
    assert mism == 0
