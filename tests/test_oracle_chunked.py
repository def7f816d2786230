"""The chunked config-4 harness (oracle/chunked.py) against the monolithic
oracle, which tests/test_oracle_golden.py pins to the reference's own
outputs.  CPU only.

A subtree rebuilt from per-leaf range compression must reproduce every
lattice (values, masks, flags) of the same subtree inside one whole-aperture
run, and a landing computed from exported lattices must reproduce the
monolithic volume on a point subset -- the two facts the config-4 GPU
parity test (tests/test_gpu_config4.py) builds on.
"""

import numpy as np
import pytest

import oracle
from oracle import chunked
from goldens import load, rel_l2


@pytest.fixture(scope="module")
def config0():
    return load("config0")


@pytest.fixture(scope="module")
def monolithic(config0):
    keep = {}
    vals, origin, step, prov = oracle.hhffbpa_reconstruct(
        config0.cube, config0.region, config0.dims, levels=7, merge_factor=4, keep=keep)
    return keep, vals, origin, step, prov


def test_plan_grid_matches_build_grid(config0):
    el = np.asarray(config0.aperture.elements)
    k_min, k_max = oracle.pipeline._band(config0.freqs)
    for a, b in [(0, 16), (16, 80), (0, 1024)]:
        ext = oracle.extents_of(el, a, b)
        g = oracle.build_grid(ext, config0.region, k_min, k_max, pad=4, prune=True)
        p = oracle.plan_grid(ext, config0.region, k_min, k_max, pad=4)
        assert tuple(int(c) for c in p.counts) == g.dims
        assert np.array_equal(p.origin, g.origin) and p.core == g.core


@pytest.mark.parametrize("quarter", [0, 3])
def test_subtree_equals_monolithic(config0, monolithic, quarter):
    keep, *_ = monolithic
    n = config0.aperture.elements.shape[0]
    e0, e1 = quarter * n // 4, (quarter + 1) * n // 4  # one level-5 subtree (16 leaves)
    res = chunked.subtree(config0.cube.values, config0.aperture.elements, e0, e1,
                          config0.freqs, config0.region, levels=7, merge_factor=4, upsample=8)
    assert sorted(res.levels) == [1, 3, 5]
    for lev, subs in res.levels.items():
        want = [s for s in keep[lev] if e0 <= s.grid.start and s.grid.stop <= e1]
        assert len(subs) == len(want) == {1: 16, 3: 4, 5: 1}[lev]
        for got, ref in zip(subs, want):
            assert (got.grid.start, got.grid.stop) == (ref.grid.start, ref.grid.stop)
            assert np.array_equal(got.grid.valid, ref.grid.valid)
            assert rel_l2(got.values, ref.values) < 1e-12


def test_landing_from_exported_lattices(config0, monolithic):
    keep, vals, origin, step, prov = monolithic
    k_min, k_max = oracle.pipeline._band(config0.freqs)
    b = oracle.pipeline._bounds(config0.region)
    center = b.mean(axis=1)
    # export the top level as a device pipeline stores it (downconverted,
    # complex64) and re-import it
    tops = []
    for s in keep[5]:
        g = s.grid
        down = (s.values * np.exp(-1j * oracle.sdc_phase(g.ext, g.positions, k_min, k_max)))
        down = np.where(g.valid, down, 0).astype(np.complex64)
        tops.append(chunked.sub_from_lattice(g.ext, g.origin, g.step, g.dims, g.core, g.start,
                                             g.stop, g.positions, g.valid, down, k_min, k_max,
                                             center))
    nx, ny, nz = config0.dims
    iz = 11
    ix, iy = np.meshgrid(np.arange(nx), np.arange(ny), indexing="ij")
    pts = np.stack([origin[0] + step[0] * ix.ravel(), origin[1] + step[1] * iy.ravel(),
                    np.full(ix.size, origin[2] + step[2] * iz)], axis=-1)
    got, flagged = oracle.merge_onto_points(tops, pts, k_min, k_max)
    want = vals[:, :, iz].ravel()
    assert rel_l2(got, want) < 1e-6  # complex64 round trip of the lattices
    assert flagged == int(np.sum(want == 0))
