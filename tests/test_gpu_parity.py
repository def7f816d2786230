"""GPU parity: the CUDA path against the reference's golden vectors and the
CPU oracle on identical seeded inputs.

Bar (BASELINE.json north_star): complex-image relative L2 <= 1e-3 and an
identical peak-voxel index; lattice metadata (dims, origin, core) and
validity masks bit-exact; provenance counts equal.  The GPU computes in
float32/complex64 (float64 for lattice geometry), so the measured errors sit
around 1e-5..1e-4.
"""

import numpy as np
import pytest

import oracle
from goldens import grid_valid, load, provenance, rel_l2

pytestmark = pytest.mark.gpu

TOL = 1e-3  # north_star: complex-image relative L2


@pytest.fixture(scope="module")
def hh():
    import paper_2506_23568_b200 as hh
    from paper_2506_23568_b200 import _native
    _native.library()  # fail loudly (no skip) when the CUDA library is unusable
    return hh


@pytest.fixture(scope="module")
def small():
    return load("small")


def _peak(v):
    v = np.abs(np.asarray(v))
    return np.unravel_index(np.argmax(v), v.shape)


def _peak_gap(v):
    a = np.sort(np.abs(np.asarray(v)).ravel())
    return float((a[-1] - a[-2]) / a[-1])


def assert_image_parity(got, want, tol=TOL):
    err = rel_l2(got, want)
    assert err <= tol, f"relative L2 {err:.3e} > {tol}"
    if _peak_gap(want) > 1e-4:
        assert _peak(got) == _peak(want), (_peak(got), _peak(want), _peak_gap(want))
    return err


def test_bpa_small_vs_reference(hh, small):
    vol = hh.bpa_reconstruct(small.cube, small.region, dims=small.dims)
    err = assert_image_parity(vol.values, small.z["bpa"], 1e-4)
    assert vol.provenance == {"algorithm": "bpa", "upsample": 8, "dims": list(small.dims)}
    assert vol.values.shape == small.dims
    print(f"bpa small rel-L2 {err:.2e}")


def test_range_profiles_vs_reference(hh, small):
    prof = hh.range_compress(small.cube, 8)
    env = prof.envelopes.cpu().numpy()
    assert rel_l2(env, small.z["envelopes"]) < 1e-5
    t0, dt, k_ref = small.z["profile_meta"]
    assert prof.t0 == t0 and prof.dt == dt and prof.k_ref == k_ref


@pytest.mark.parametrize("upsample", [1, 2, 4, 8, 16, 64, 512])
def test_fused_range_compression_vs_reference(hh, small, upsample, monkeypatch):
    """hhsar_range_compress (pad + IDFT + demod in one pass, n_t = 16 ...
    8192) against numpy's IDFT restatement and, at upsample 8, the
    reference's own envelopes."""
    import oracle
    from paper_2506_23568_b200 import rangecomp
    monkeypatch.setattr(rangecomp, "_FORCE_CUFFT", False)
    prof = hh.range_compress(small.cube, upsample)
    want = oracle.range_compress(small.cube, upsample).envelopes
    assert rel_l2(prof.envelopes.cpu().numpy(), want) < 2e-6
    if upsample == 8:
        assert rel_l2(prof.envelopes.cpu().numpy(), small.z["envelopes"]) < 2e-6


@pytest.mark.parametrize("n_el,n_f,upsample", [(37, 256, 4), (5, 128, 8), (3, 1024, 4),
                                                (9, 512, 2), (1, 2048, 4), (6, 50, 4)])
def test_fused_range_compression_ragged_vs_cufft(n_el, n_f, upsample, monkeypatch):
    """Fused kernel on ragged row counts (partial multi-row CTAs), every
    first-pass radix and pruning variant, and a non-power-of-two n_t (cuFFT
    path), against the cuFFT + demodulation path on the same device cube."""
    import torch
    from paper_2506_23568_b200 import rangecomp
    from paper_2506_23568_b200.model import FrequencyGrid
    freqs = FrequencyGrid(77e9, 81e9, n_f)
    gen = torch.Generator(device="cuda").manual_seed(n_el * 7919 + n_f)
    cube = torch.randn((n_el, n_f), dtype=torch.complex64, device="cuda", generator=gen)
    monkeypatch.setattr(rangecomp, "_FORCE_CUFFT", False)
    got, dt, k_ref = rangecomp.range_compress_device(cube, freqs, upsample)
    monkeypatch.setattr(rangecomp, "_FORCE_CUFFT", True)
    want, dt2, k_ref2 = rangecomp.range_compress_device(cube, freqs, upsample)
    assert (dt, k_ref) == (dt2, k_ref2)
    assert got.shape == want.shape == (n_el, n_f * upsample)
    assert rel_l2(got.cpu().numpy(), want.cpu().numpy()) < 2e-6


def test_backproject_probes_selections_and_empty(hh, small):
    prof = hh.range_compress(small.cube, 8)
    got = hh.backproject(prof, slice(None), small.z["probes"])
    assert rel_l2(got, small.z["probe_values"]) < 1e-4
    sub = hh.backproject(prof, hh.Subarray(10, 33), small.z["probes"])
    assert rel_l2(sub, small.z["probe_values_sub"]) < 1e-4
    via_idx = hh.backproject(prof, np.arange(10, 33), small.z["probes"])
    assert rel_l2(via_idx, sub) < 1e-6
    empty = hh.backproject(prof, slice(0, 0), small.z["probes"])
    assert empty.shape == (40,) and np.all(empty == 0)


def test_backproject_out_of_window_raises(hh, small):
    prof = hh.range_compress(small.cube, 8)
    far = np.array([[0.0, 0.0, 1e3]])
    with pytest.raises(hh.NumericDomainError):
        hh.backproject(prof, slice(None), far)


@pytest.mark.parametrize("tag,levels,kernel", [("m2", 2, "linear"), ("m3", 3, "linear"),
                                               ("m3c", 3, "cubic")])
def test_hhffbpa_small_vs_reference(hh, small, tag, levels, kernel):
    vol = hh.hhffbpa_reconstruct(small.cube, small.region, small.dims,
                                 hh.FfbpParams(levels=levels, kernel=kernel))
    err = assert_image_parity(vol.values, small.z["hh_" + tag])
    want = provenance(small.z, "hh_" + tag)
    p = vol.provenance
    assert p["level_points"] == want["level_points"]
    assert p["merge_flags"] == want["merge_flags"]
    assert p["final_flags"] == want["final_flags"]
    assert p["flagged_fraction"] == pytest.approx(float(small.z["hh_" + tag + "_flagged_fraction"]))
    print(f"hhffbpa small {tag} rel-L2 {err:.2e}")


def test_all_grid_metadata_and_masks_bit_exact(hh, small):
    import torch
    from paper_2506_23568_b200 import ffbp
    sched = ffbp.Schedule(small.aperture.n_elements, 3)
    el = torch.as_tensor(np.asarray(small.aperture.elements), device="cuda")
    lat = ffbp.build_lattices(el, sched, small.region, small.freqs, 1.4, 0.25, 4, np.inf)
    d = lat.descs
    z = small.z
    assert np.array_equal(d["dims"], z["grid_dims"])
    assert np.array_equal(d["origin"], z["grid_origin"])
    assert np.array_equal(np.concatenate([d["core_lo"][:, :, None], d["core_hi"][:, :, None]],
                                         axis=2).reshape(-1, 6), z["grid_core"])
    assert np.array_equal(d["ext"], z["grid_ext"])
    valid = lat.valid.cpu().numpy().astype(bool)
    want = np.concatenate([v.ravel() for v in grid_valid(z, "grid")])
    assert np.array_equal(valid, want)
    pos = lat.positions.cpu().numpy()
    assert np.max(np.abs(pos[valid] - z["grid_positions"][valid])) < 1e-9
    stats = lat.stats.cpu().numpy()
    assert np.array_equal(stats[:, 0], z["grid_nvalid"])


def test_build_subimage_grid_single(hh, small):
    tree = hh.partition_subarrays(small.aperture, 3)
    g = hh.build_subimage_grid(small.aperture, tree.levels[0][0], small.region, small.freqs,
                               gamma=1.4)
    assert g.dims == tuple(small.z["grid_pad2_dims"][0])
    assert np.array_equal(g.origin, small.z["grid_pad2_origin"][0])
    assert np.array_equal(g.valid, grid_valid(small.z, "grid_pad2")[0])
    v = g.valid.ravel()
    assert np.max(np.abs(g.positions.reshape(-1, 3)[v] - small.z["grid_pad2_positions"][v])) < 1e-9


def test_unreachable_region_raises(hh, small):
    hopeless = hh.ImagingRegion(-0.02, 0.02, -0.02, 0.02, 1e-6, 2e-6)
    with pytest.raises(hh.NumericDomainError):
        hh.build_subimage_grid(small.aperture, None, hopeless, small.freqs)


def test_level1_and_merge_pair_vs_reference(hh, small):
    prof = hh.range_compress(small.cube, 8)
    tree = hh.partition_subarrays(small.aperture, 3)
    grids = [hh.build_subimage_grid(small.aperture, sa, small.region, small.freqs, 1.4, 0.25,
                                    pad=4) for lvl in tree.levels[:2] for sa in lvl]
    leaves = [hh.level1_reconstruct(prof, sa, g) for sa, g in zip(tree.levels[0], grids[:4])]
    got = np.concatenate([l.values.ravel() for l in leaves])
    assert rel_l2(got, small.z["leaf_values"]) < 1e-4
    valid = np.unpackbits(small.z["leaf_valid"])[:got.size].astype(bool)
    assert np.array_equal(np.concatenate([l.grid.valid.ravel() for l in leaves]), valid)
    merged, flagged = hh.merge_pair(leaves[0], leaves[1], grids[4], small.freqs)
    assert rel_l2(merged.values, small.z["merge01"]) < 1e-4
    assert flagged == int(small.z["merge01_flagged"])
    with pytest.raises(hh.ConfigError):
        hh.merge_pair(leaves[0], leaves[2], grids[4], small.freqs)


@pytest.mark.parametrize("kernel", ["linear", "cubic"])
def test_lattice_interpolate_operator(hh, small, kernel):
    from paper_2506_23568_b200 import _kernels
    v, ok = _kernels.lattice_interpolate(small.z["interp_lattice"], small.z["interp_coords"],
                                         kernel)
    assert np.array_equal(ok, small.z[f"interp_{kernel}_ok"])
    assert np.max(np.abs(v - small.z[f"interp_{kernel}"])) < 1e-5


def test_newton_operator(hh, small):
    from paper_2506_23568_b200 import _kernels
    z = small.z
    e = z["newton_ext"]
    pos, ok, it = _kernels.invert_newton(e[0], e[1], e[2], e[3], small.freqs.k_min,
                                         small.freqs.k_max, z["newton_targets"],
                                         z["newton_guesses"], 1e-9, 50,
                                         float(z["newton_max_step"]), 1e-4)
    assert np.array_equal(ok, z["newton_ok"])
    assert np.max(np.abs(pos[ok] - z["newton_pos"][ok])) < 1e-9


def test_medium_vs_reference(hh):
    m = load("medium")
    vol = hh.bpa_reconstruct(m.cube, m.region, dims=m.dims)
    assert_image_parity(vol.values, m.z["bpa"], 1e-4)
    for lv in (3, 4):
        vol = hh.hhffbpa_reconstruct(m.cube, m.region, m.dims, hh.FfbpParams(levels=lv))
        assert_image_parity(vol.values, m.z[f"hh_m{lv}"])
        assert vol.provenance["level_points"] == provenance(m.z, f"hh_m{lv}")["level_points"]


@pytest.fixture(scope="module")
def config0():
    return load("config0")


def test_config0_bpa(hh, config0):
    vol = hh.bpa_reconstruct(config0.cube, config0.region, dims=config0.dims, upsample=8)
    err = assert_image_parity(vol.values, config0.z["bpa"])
    print(f"config0 bpa rel-L2 {err:.2e}, peak gap {_peak_gap(config0.z['bpa']):.3e}")


@pytest.mark.parametrize("tag,factor", [("m7", 2), ("f4", 4)])
def test_config0_hhffbpa(hh, config0, tag, factor):
    vol = hh.hhffbpa_reconstruct(config0.cube, config0.region, config0.dims,
                                 hh.FfbpParams(levels=7), upsample=8, merge_factor=factor)
    err = assert_image_parity(vol.values, config0.z["hh_" + tag])
    want = provenance(config0.z, "hh_" + tag)
    assert vol.provenance["level_points"] == want["level_points"]
    assert vol.provenance["merge_flags"] == want["merge_flags"]
    assert vol.provenance["final_flags"] == want["final_flags"]
    print(f"config0 hhffbpa {tag} rel-L2 {err:.2e}")


def test_config0_all_grid_masks(hh, config0):
    import torch
    from paper_2506_23568_b200 import ffbp
    sched = ffbp.Schedule(config0.aperture.n_elements, 7)
    el = torch.as_tensor(np.asarray(config0.aperture.elements), device="cuda")
    lat = ffbp.build_lattices(el, sched, config0.region, config0.freqs, 1.4, 0.25, 4, np.inf)
    z = config0.z
    assert np.array_equal(lat.descs["dims"], z["grid_dims"])
    assert np.array_equal(lat.descs["origin"], z["grid_origin"])
    valid = lat.valid.cpu().numpy().astype(bool)
    want = np.concatenate([v.ravel() for v in grid_valid(z, "grid")])
    assert int((valid != want).sum()) == 0


def test_single_level_equals_bpa(hh, small):
    a = hh.hhffbpa_reconstruct(small.cube, small.region, small.dims, hh.FfbpParams(levels=1))
    b = hh.bpa_reconstruct(small.cube, small.region, dims=small.dims)
    assert np.array_equal(a.values, b.values)
    assert a.provenance["level_points"] == [[int(np.prod(small.dims))]]


def test_linearity(hh, small):
    from paper_2506_23568_b200.model import DataCube
    rng = np.random.default_rng(4)
    shape = small.cube.values.shape
    other = (rng.normal(size=shape) + 1j * rng.normal(size=shape)).astype(np.complex64)
    base = np.asarray(small.cube.values, dtype=np.complex64)
    params = hh.FfbpParams(levels=2)
    dims = (17, 17, 9)
    va = hh.hhffbpa_reconstruct(small.cube, small.region, dims, params).values
    vb = hh.hhffbpa_reconstruct(DataCube(other, small.aperture, small.freqs), small.region,
                                dims, params).values
    vab = hh.hhffbpa_reconstruct(DataCube(base + other, small.aperture, small.freqs),
                                 small.region, dims, params).values
    assert rel_l2(vab, va + vb) < 1e-5


def test_gpu_matches_oracle_on_config2_subset(hh):
    """A frame-reduced config 2 (freehand MIMO, 8 virtual elements) through
    both the GPU and the oracle, binary M=6."""
    from paper_2506_23568_b200 import workloads
    w = workloads.config(2, frames=256)
    cube = workloads.simulate_numpy(w)
    dims = (40, 40, 16)
    g = hh.hhffbpa_reconstruct(cube, w.region, dims, hh.FfbpParams(levels=6), upsample=4)
    o, _, _, prov = oracle.hhffbpa_reconstruct(cube, w.region, dims, levels=6, upsample=4)
    assert_image_parity(g.values, o)
    assert g.provenance["level_points"] == prov["level_points"]
    assert g.provenance["merge_flags"] == prov["merge_flags"]


def test_config3_full_scale_vs_oracle(hh):
    """BASELINE config 3 at full scale (131,072 elements, 512x512x128, binary
    M=11): the device pipeline against the oracle on the same GPU-simulated
    cube -- image parity, per-grid valid-point counts of every level and the
    merge flags (~30 s of CPU oracle)."""
    import torch
    from paper_2506_23568_b200 import _native, bpa, ffbp, workloads
    from paper_2506_23568_b200.model import DataCube
    w = workloads.config(3)
    cube = _native.simulate(np.asarray(w.aperture.elements), w.scene_pos, w.scene_refl,
                            w.freqs.k_samples)
    el = torch.tensor(np.asarray(w.aperture.elements), device="cuda")
    run = ffbp.hhffbpa_from_cube(cube, el, bpa.el_f32x4(el), w.freqs, w.region, w.dims,
                                 ffbp.FfbpParams(levels=w.levels), w.levels, 2, w.upsample)
    torch.cuda.synchronize()
    host = DataCube(values=cube.cpu().numpy(), aperture=w.aperture, freqs=w.freqs)
    want, _, _, prov = oracle.hhffbpa_reconstruct(host, w.region, w.dims, levels=w.levels,
                                                  upsample=w.upsample)
    got = run.volume.cpu().numpy().reshape(w.dims)
    assert_image_parity(got, want)
    stats = run.lattices.stats.cpu().numpy()
    lp = [[int(v) for v in stats[a:b, 2 if k == 0 else 0]]
          for k, (a, b) in enumerate(run.sched.level_slices)]
    assert lp == prov["level_points"][:-1]
    assert [int(f) for f in run.flags.cpu().numpy()] == prov["merge_flags"] + [prov["final_flags"]]


@pytest.mark.parametrize("n_el,n_f,upsample,b0,w", [(37, 256, 4, 80, 96), (9, 512, 4, 0, 64),
                                                    (5, 1024, 4, 4000, 96), (3, 128, 8, 300, 211),
                                                    (4, 64, 4, 17, 239),
                                                    (2000, 1024, 4, 49, 288),   # config 4 rows, box gate
                                                    (3000, 512, 4, 0, 352),     # config 3 rows, box gate
                                                    (2000, 1024, 4, 65, 128),   # config 4, near-band gate
                                                    (3000, 512, 4, 10, 64),     # config 3, near-band gate
                                                    (70, 1024, 4, 63, 129), (70, 1024, 4, 1, 255),
                                                    # 4096-bin rows, gated: the one-exchange kernel
                                                    (300, 1024, 4, 0, 512), (300, 1024, 4, 3584, 512),
                                                    (70, 1024, 4, 4095, 1), (70, 1024, 4, 63, 65),
                                                    (70, 1024, 4, 1000, 449), (70, 512, 8, 49, 288),
                                                    (70, 512, 8, 3000, 1096),
                                                    # 2048-bin rows (config 3): the same split
                                                    (70, 512, 4, 1600, 448), (70, 512, 4, 2047, 1),
                                                    (70, 256, 8, 100, 300), (70, 512, 4, 31, 65)])
def test_range_compress_window_equals_full_slice(n_el, n_f, upsample, b0, w):
    """The range-gated compression (only bins [b0, b0 + w) computed in the
    last pass and stored) against the same bins of the full compression."""
    import torch
    from paper_2506_23568_b200 import rangecomp
    from paper_2506_23568_b200.model import FrequencyGrid
    freqs = FrequencyGrid(77e9, 81e9, n_f)
    gen = torch.Generator(device="cuda").manual_seed(n_el * 31 + n_f)
    cube = torch.randn((n_el, n_f), dtype=torch.complex64, device="cuda", generator=gen)
    full, dt, k_ref = rangecomp.range_compress_device(cube, freqs, upsample)
    got, t0w, dt2, k2 = rangecomp.range_compress_window(cube, freqs, upsample, b0, w)
    assert (dt2, k2) == (dt, k_ref) and t0w == b0 * dt and got.shape == (n_el, w)
    want = full[:, b0:b0 + w]
    assert rel_l2(got.cpu().numpy(), want.cpu().numpy()) < 2e-6


@pytest.mark.parametrize("config,levels,kernel", [(2, None, "linear"), (3, None, "linear"),
                                                 (4, None, "linear"),
                                                 (2, 6, "cubic"),    # 1,000-element leaves
                                                 (3, 8, "linear")])  # 1,024-element leaves
def test_range_gate_matches_full_profiles(config, levels, kernel):
    """HHFFBPA with range-gated compression (only the delay bins the leaf
    stage can read, ffbp.leaf_range_gate) equals the run on full profiles:
    same image to float rounding, same lattices and flags, no leaf delay
    outside the gated window."""
    import torch
    from paper_2506_23568_b200 import bpa, ffbp, rangecomp, workloads
    w = workloads.config(config)
    gen = torch.Generator(device="cuda").manual_seed(w.seed)
    cube = torch.randn((w.n_elements, w.freqs.count), dtype=torch.complex64, device="cuda",
                       generator=gen)
    el = torch.tensor(np.asarray(w.aperture.elements), device="cuda")
    el4 = bpa.el_f32x4(el)
    levels = levels or w.levels
    params = ffbp.FfbpParams(levels=levels, kernel=kernel)
    # config 4: full profiles 68.7 GB + cube 17.2 GB (+ 2.1 GB gated)
    runs = [ffbp.hhffbpa_from_cube(cube, el, el4, w.freqs, w.region, w.dims, params, levels,
                                   w.merge_factor, w.upsample, gate=g) for g in (False, True)]
    torch.cuda.synchronize()
    del cube
    full, gated = (r.volume.cpu().numpy() for r in runs)
    assert int(runs[1].oow.cpu()[0]) == int(runs[0].oow.cpu()[0]) == 0
    rel = np.linalg.norm(gated - full) / np.linalg.norm(full)
    assert rel < 1e-5, rel
    assert np.argmax(np.abs(gated)) == np.argmax(np.abs(full))
    assert torch.equal(runs[0].lattices.stats, runs[1].lattices.stats)
    assert torch.equal(runs[0].flags, runs[1].flags)
    n_t, dt, _, _ = rangecomp.profile_axis(w.freqs, w.upsample)
    assert runs[1].lattices.gate == ffbp.leaf_range_gate(runs[1].lattices, runs[1].sched, dt, n_t)


@pytest.mark.parametrize("config", [2, 3])
def test_step_graph_replays_the_eager_step(config):
    """StepGraph (plan cache + CUDA graph of the whole HHFFBPA step):
    replays are bit-identical to the eager step, follow the cube's contents
    (same graph, new data) and keep provenance counters identical."""
    import torch
    from paper_2506_23568_b200 import bpa, ffbp, workloads
    w = workloads.config(config)
    gen = torch.Generator(device="cuda").manual_seed(w.seed)
    cube = torch.randn((w.n_elements, w.freqs.count), dtype=torch.complex64, device="cuda",
                       generator=gen)
    el = torch.tensor(np.asarray(w.aperture.elements), device="cuda")
    el4 = bpa.el_f32x4(el)
    params = ffbp.FfbpParams(levels=w.levels)
    args = (el, el4, w.freqs, w.region, w.dims, params, w.levels, w.merge_factor, w.upsample)
    g = ffbp.StepGraph(cube, *args)
    eager = ffbp.hhffbpa_from_cube(cube, *args)
    run = g.replay()
    torch.cuda.synchronize()
    assert torch.equal(run.volume, eager.volume)
    assert torch.equal(run.lattices.stats, eager.lattices.stats)
    assert torch.equal(run.flags, eager.flags)
    cube.mul_(0.5 - 2.0j)  # new data, same buffer: the replay must follow it
    eager2 = ffbp.hhffbpa_from_cube(cube, *args)
    run = g.replay()
    torch.cuda.synchronize()
    assert torch.equal(run.volume, eager2.volume)


def test_public_api_host_input_forms():
    """hhffbpa_reconstruct streams the cube from whatever host form it gets
    -- pageable numpy (pinned staging buffers), a view of pinned memory
    (direct DMA), a CPU torch tensor -- with bit-identical results."""
    import torch
    import paper_2506_23568_b200 as hh
    from paper_2506_23568_b200 import rangecomp, workloads
    from paper_2506_23568_b200.model import DataCube
    w = workloads.config(2, frames=1024)
    base = workloads.simulate_numpy(w)
    params = hh.FfbpParams(levels=8)
    dims = (64, 64, 24)
    pinned = torch.from_numpy(np.asarray(base.values).copy()).pin_memory()
    old = rangecomp.UPLOAD_CHUNK_BYTES
    rangecomp.UPLOAD_CHUNK_BYTES = 1 << 20  # several chunks at this size
    try:
        outs = []
        for values in (np.asarray(base.values), pinned.numpy(),
                       torch.from_numpy(np.asarray(base.values).copy())):
            cube = DataCube(values=values, aperture=base.aperture, freqs=base.freqs)
            outs.append(hh.hhffbpa_reconstruct(cube, w.region, dims, params, upsample=4,
                                               merge_factor=4))
    finally:
        rangecomp.UPLOAD_CHUNK_BYTES = old
    for o in outs[1:]:
        assert np.array_equal(o.values, outs[0].values)
        assert o.provenance == outs[0].provenance


def test_gate_miss_redoes_on_full_profiles(monkeypatch):
    """A leaf delay outside the range gate (forced here by shifting the
    gated window up by half its width) makes hhffbpa_reconstruct redo the
    step on full profiles: the result is the ungated step's, bit for bit,
    with the same provenance -- never a volume missing contributions."""
    import paper_2506_23568_b200 as hh
    from paper_2506_23568_b200 import ffbp, rangecomp, workloads
    w = workloads.config(2, frames=512)
    cube = workloads.simulate_numpy(w)
    params = hh.FfbpParams(levels=7)
    dims = (48, 48, 16)
    want = hh.hhffbpa_reconstruct(cube, w.region, dims, params, upsample=4, merge_factor=4)
    orig_win, orig_full = rangecomp.range_compress_window, rangecomp.range_compress_device
    calls = {"window": 0, "full": 0}

    def shifted(cube_dev, kgrid, upsample, b0, width, **kw):
        calls["window"] += 1
        return orig_win(cube_dev, kgrid, upsample, b0 + width // 2, width - width // 2, **kw)

    def full(*a, **kw):
        calls["full"] += 1
        return orig_full(*a, **kw)

    monkeypatch.setattr(rangecomp, "range_compress_window", shifted)
    monkeypatch.setattr(rangecomp, "range_compress_device", full)
    got = hh.hhffbpa_reconstruct(cube, w.region, dims, params, upsample=4, merge_factor=4)
    assert calls["window"] >= 1 and calls["full"] == 1  # the gate missed: one ungated redo
    monkeypatch.undo()
    import torch
    el = torch.tensor(np.asarray(w.aperture.elements), device="cuda")
    cube_dev = torch.as_tensor(np.asarray(cube.values), device="cuda")
    ungated = ffbp.hhffbpa_from_cube(cube_dev, el, hh.bpa.el_f32x4(el), w.freqs, w.region, dims,
                                     params, 7, 4, 4, gate=False)
    assert np.array_equal(got.values, ungated.volume.cpu().numpy().reshape(dims))
    assert got.provenance == want.provenance
    assert rel_l2(got.values, want.values) < 1e-5


def test_reconstruct_stream_equals_single_calls():
    """hhffbpa_reconstruct_stream (uploads overlapped across volumes, plan
    cache from the first volume) returns, per cube, exactly what
    hhffbpa_reconstruct returns."""
    import torch
    import paper_2506_23568_b200 as hh
    from paper_2506_23568_b200 import ffbp, workloads
    from paper_2506_23568_b200.model import DataCube
    w = workloads.config(2, frames=1024)
    base = workloads.simulate_numpy(w)
    params = hh.FfbpParams(levels=8)
    dims = (64, 64, 24)
    pinned = torch.from_numpy(np.asarray(base.values).copy()).pin_memory()
    cubes = [DataCube(values=np.asarray(base.values) * s, aperture=base.aperture,
                      freqs=base.freqs) for s in (1.0, 0.5 - 1j)]
    cubes.append(DataCube(values=pinned.numpy(), aperture=base.aperture, freqs=base.freqs))
    got = list(ffbp.hhffbpa_reconstruct_stream(cubes, w.region, dims, params, upsample=4,
                                               merge_factor=4))
    assert len(got) == 3
    for cube, vol in zip(cubes, got):
        want = hh.hhffbpa_reconstruct(cube, w.region, dims, params, upsample=4, merge_factor=4)
        assert np.array_equal(vol.values, want.values)
        assert vol.provenance == want.provenance


@pytest.mark.parametrize("factor", [2, 4])
def test_config0_hhffbpa_cubic_vs_oracle(hh, config0, factor):
    """Keys-cubic interpolation (FfbpParams(kernel='cubic'), _kernels.py:155-200)
    through the whole config-0 pipeline, binary and factor-4 schedules, against
    the oracle (pinned to the reference's cubic goldens at small scale)."""
    import oracle
    vol = hh.hhffbpa_reconstruct(config0.cube, config0.region, config0.dims,
                                 hh.FfbpParams(levels=7, kernel="cubic"), upsample=8,
                                 merge_factor=factor)
    want, _, _, prov = oracle.hhffbpa_reconstruct(config0.cube, config0.region, config0.dims,
                                                  levels=7, kernel="cubic", upsample=8,
                                                  merge_factor=factor)
    err = assert_image_parity(vol.values, want)
    assert vol.provenance["level_points"] == prov["level_points"]
    assert vol.provenance["merge_flags"] == prov["merge_flags"]
    assert vol.provenance["final_flags"] == prov["final_flags"]
    print(f"config0 cubic factor {factor} rel-L2 {err:.2e}")


def test_sdc_phase_operator_vs_reference(hh, small):
    """S1 at operator level: hhsar_downconvert on unit values returns
    exp(-j Phi(pos)) with Phi the reference's sdc_phase (spectrum.py:229-240,
    golden map_phase on 64 random region points); float64 phase, reduced
    before the float32 sincos."""
    import torch
    from paper_2506_23568_b200 import _native, ffbp
    z = small.z
    pts = np.ascontiguousarray(z["map_points"], dtype=np.float64)
    n = pts.shape[0]
    e = z["newton_ext"]
    desc = ffbp._one_desc(tuple(e), np.zeros(3), (n, 1, 1), 0, 0, 0)
    d_dev = _native.device_struct(desc, torch.device("cuda"))
    pos = torch.as_tensor(pts, device="cuda")
    valid = torch.ones(n, dtype=torch.uint8, device="cuda")
    vals = torch.ones(n, dtype=torch.complex64, device="cuda")
    geom = ffbp._geom_for(small.freqs)
    _native.call("hhsar_downconvert", _native.ptr(d_dev), 1, n, _native.ptr(pos),
                 _native.ptr(valid), _native.ptr(geom), _native.ptr(vals),
                 _native.stream_handle())
    got = vals.cpu().numpy().astype(np.complex128)
    want = np.exp(-1j * z["map_phase"])
    assert np.max(np.abs(got - want)) < 2e-6


@pytest.mark.parametrize("config,kernel,dims", [(2, "linear", None), (3, "linear", None),
                                                (2, "cubic", None),
                                                # ragged: no warp tiles, partial z blocks
                                                (2, "linear", (37, 29, 13)),
                                                (2, "cubic", (21, 40, 7))])
def test_landing_series_equals_per_voxel(config, kernel, dims):
    """The z-series landing (merge_cartesian_series_kernel: quartic Taylor
    polynomials per 8-voxel z run, pair-staged lattice gathers) against the
    per-voxel float64 landing (HHSAR_LANDING_PER_VOXEL) on the same device
    lattices: same image to float32 rounding, same flags; pair staging on
    or off gives the same bits for the linear kernel."""
    import torch
    from paper_2506_23568_b200 import bpa, ffbp, workloads
    w = workloads.config(config)
    gen = torch.Generator(device="cuda").manual_seed(w.seed)
    cube = torch.randn((w.n_elements, w.freqs.count), dtype=torch.complex64, device="cuda",
                       generator=gen)
    el = torch.tensor(np.asarray(w.aperture.elements), device="cuda")
    params = ffbp.FfbpParams(levels=w.levels, kernel=kernel)
    args = (cube, el, bpa.el_f32x4(el), w.freqs, w.region, dims or w.dims, params, w.levels,
            w.merge_factor, w.upsample)
    out = {}
    try:
        for series, pairs in ((True, True), (True, False), (False, True)):
            ffbp.LANDING_SERIES, ffbp.LANDING_PAIRS = series, pairs
            run = ffbp.hhffbpa_from_cube(*args)
            out[series, pairs] = (run.volume.cpu().numpy(), int(run.flags.cpu()[-1]))
    finally:
        ffbp.LANDING_SERIES, ffbp.LANDING_PAIRS = True, True
    ref, ref_flags = out[False, True]
    got, flags = out[True, True]
    assert flags == ref_flags
    assert rel_l2(got, ref) < 5e-5
    assert np.argmax(np.abs(got)) == np.argmax(np.abs(ref))
    if kernel == "linear":
        assert np.array_equal(out[True, False][0], got)
    else:
        assert rel_l2(out[True, False][0], got) < 1e-6
