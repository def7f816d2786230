"""Generate the golden vectors that pin the oracle (and, through it, the GPU).

Runs the UNMODIFIED reference (/root/reference/pkg/src/hhsar, Numba path) on
seeded inputs and stores inputs + outputs as compressed .npz next to this
script.  Only the build container has /root/reference; the GPU box and the
tests only read the committed .npz files.

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

Cases
-----
small    the reference test fixture `small` (conftest.py:90-100): 9x9 desk
         aperture, quarter-scale region, 12-15 GHz x16; BPA (17,17,9), probes,
         HHFFBPA M=2/3 linear + M=3 cubic, per-grid metadata and masks, one
         leaf and one merge_pair, lattice_interpolate and Newton samples.
medium   the `medium` fixture (conftest.py:103-114): 17x17, dims (33,33,17),
         BPA and HHFFBPA M=3 / M=4.
config0  BASELINE config 0 (paper_2506_23568_b200.workloads.config(0)): BPA
         64x64x32, HHFFBPA binary M=7 and the merge-factor-4 schedule built
         from reference primitives; all grid masks.
metrics  metrics.py on seeded volumes/profiles (`make_golden.py metrics`
         regenerates only this one).
cli_tools  the reference CLI's `project` (PGM, z/8-bit and x/16-bit) and
         `metrics` (JSON report) on the io case's volumes
         (`make_golden.py cli_tools`).
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parents[1]
REF = Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))
sys.path.insert(0, str(REF / "tests"))
sys.path.insert(0, str(REPO))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import hhsar  # noqa: E402
from hhsar import ffbp as rffbp  # noqa: E402
from hhsar import spectrum as rspec  # noqa: E402

from paper_2506_23568_b200 import workloads  # noqa: E402


def _ref_cube(values, elements, nx, ny, freqs):
    ap = hhsar.SyntheticAperture(elements=np.asarray(elements, float), nx=nx, ny=ny)
    fg = hhsar.FrequencyGrid(freqs.f_min, freqs.f_max, freqs.count)
    return hhsar.DataCube(values=values, aperture=ap, freqs=fg)


def _region_arr(r):
    return np.array([r.x_min, r.x_max, r.y_min, r.y_max, r.z_min, r.z_max])


def _prov(prefix, vol, out):
    p = vol.provenance
    out[prefix + "_level_points"] = np.array(
        [n for lvl in p.get("level_points", []) for n in lvl], dtype=np.int64)
    out[prefix + "_level_sizes"] = np.array(
        [len(lvl) for lvl in p.get("level_points", [])], dtype=np.int64)
    out[prefix + "_merge_flags"] = np.array(p.get("merge_flags", []), dtype=np.int64)
    out[prefix + "_final_flags"] = np.int64(p.get("final_flags", 0))
    out[prefix + "_flagged_fraction"] = np.float64(p.get("flagged_fraction", 0.0))


def _grid_meta(prefix, grids, out, with_positions=False):
    out[prefix + "_dims"] = np.array([g.dims for g in grids], dtype=np.int64)
    out[prefix + "_origin"] = np.array([g.origin for g in grids])
    out[prefix + "_step"] = np.array([g.step for g in grids])
    out[prefix + "_core"] = np.array([[c for ab in g.core for c in ab] for g in grids],
                                     dtype=np.int64)
    out[prefix + "_ext"] = np.array([[g.extents.x_min, g.extents.x_max,
                                      g.extents.y_min, g.extents.y_max] for g in grids])
    out[prefix + "_valid"] = np.packbits(np.concatenate([g.valid.ravel() for g in grids]))
    out[prefix + "_nvalid"] = np.array([g.n_valid for g in grids], dtype=np.int64)
    if with_positions:
        out[prefix + "_positions"] = np.concatenate(
            [g.positions.reshape(-1, 3) for g in grids])


def factor4_reference(cube, region, dims, levels, gamma=1.4, kernel="linear",
                      upsample=8, factor=4):
    """Merge-factor-4 schedule composed only of reference primitives."""
    kgrid = cube.freqs
    profiles = hhsar.range_compress(cube, upsample)
    hhsar.bpa.check_delay_window(profiles, region)
    origin, step = hhsar.region_grid(region, dims)
    axes = [origin[a] + step[a] * np.arange(dims[a]) for a in range(3)]
    cart = np.stack([m.ravel() for m in np.meshgrid(*axes, indexing="ij")], axis=-1)
    src_pad = rffbp.GRID_PAD + (3 if kernel == "cubic" else 2)
    tree = hhsar.partition_subarrays(cube.aperture, levels)
    subs = [hhsar.level1_reconstruct(profiles, sa, hhsar.build_subimage_grid(
        cube.aperture, sa, region, kgrid, gamma, 0.25, pad=src_pad)) for sa in tree.levels[0]]
    level_points = [[s.grid.n_valid for s in subs]]
    merge_flags = []
    s = int(np.log2(factor))
    for lev in range(1 + s, levels, s):
        merged, flags = [], 0
        for parent in tree.levels[lev - 1]:
            kids = [c for c in subs if parent.start <= c.grid.subarray.start
                    and c.grid.subarray.stop <= parent.stop]
            pg = hhsar.build_subimage_grid(cube.aperture, parent, region, kgrid, gamma,
                                           0.25, pad=src_pad)
            flat = pg.positions.reshape(-1, 3)
            mask = pg.valid.ravel()
            vals = np.zeros(flat.shape[0], dtype=complex)
            fl = 0
            if mask.any():
                vals[mask], fl = rffbp._merge_onto_points(tuple(kids), flat[mask], kgrid, kernel)
            merged.append(hhsar.Subimage(grid=pg, values=vals.reshape(pg.dims)))
            flags += fl
        merge_flags.append(flags)
        level_points.append([m.grid.n_valid for m in merged])
        subs = merged
    values, final_flags = rffbp._merge_onto_points(tuple(subs), cart, kgrid, kernel)
    level_points.append([int(np.prod(dims))])
    return values.reshape(dims), level_points, merge_flags, final_flags


def case_small(out):
    from conftest import desk_aperture, desk_frequencies, desk_region, desk_scene
    freqs = desk_frequencies()
    ap = desk_aperture(side=9)
    region = desk_region(scale=0.25)
    cube = hhsar.simulate_measurement(desk_scene(scale=0.25), ap, freqs)
    prof = hhsar.range_compress(cube, 8)
    out["cube"] = cube.values
    out["elements"] = ap.elements
    out["nxny"] = np.array([ap.nx, ap.ny])
    out["freqs"] = np.array([freqs.f_min, freqs.f_max, freqs.count])
    out["region"] = _region_arr(region)
    out["envelopes"] = prof.envelopes
    out["profile_meta"] = np.array([prof.t0, prof.dt, prof.k_ref])
    dims = (17, 17, 9)
    out["dims"] = np.array(dims)
    out["bpa"] = hhsar.bpa_reconstruct(cube, region, dims=dims).values
    rng = np.random.default_rng(21)
    probes = np.column_stack([rng.uniform(region.x_min, region.x_max, 40),
                              rng.uniform(region.y_min, region.y_max, 40),
                              rng.uniform(region.z_min, region.z_max, 40)])
    out["probes"] = probes
    out["probe_values"] = hhsar.backproject(prof, slice(None), probes)
    out["probe_values_sub"] = hhsar.backproject(prof, hhsar.Subarray(10, 33), probes)
    for tag, lv, kern in (("m2", 2, "linear"), ("m3", 3, "linear"), ("m3c", 3, "cubic")):
        vol = hhsar.hhffbpa_reconstruct(cube, region, final_dims=dims,
                                        params=hhsar.FfbpParams(levels=lv, kernel=kern))
        out["hh_" + tag] = vol.values
        _prov("hh_" + tag, vol, out)
    # grids of the M=3 tree, with the pipeline's src_pad = GRID_PAD + 2
    tree = hhsar.partition_subarrays(ap, 3)
    grids = [hhsar.build_subimage_grid(ap, sa, region, freqs, 1.4, 0.25, pad=4)
             for lvl in tree.levels[:2] for sa in lvl]
    _grid_meta("grid", grids, out, with_positions=True)
    out["grid_slices"] = np.array([[sa.start, sa.stop] for lvl in tree.levels[:2]
                                   for sa in lvl], dtype=np.int64)
    # default-pad grid (GRID_PAD = 2) of leaf 0, as test_ffbp.py:210-221 builds it
    g0 = hhsar.build_subimage_grid(ap, tree.levels[0][0], region, freqs, gamma=1.4)
    _grid_meta("grid_pad2", [g0], out, with_positions=True)
    leaves = [hhsar.level1_reconstruct(prof, sa, g) for sa, g in zip(tree.levels[0], grids[:4])]
    out["leaf_values"] = np.concatenate([l.values.ravel() for l in leaves])
    out["leaf_valid"] = np.packbits(np.concatenate([l.grid.valid.ravel() for l in leaves]))
    merged, flagged = hhsar.merge_pair(leaves[0], leaves[1], grids[4], freqs)
    out["merge01"] = merged.values
    out["merge01_flagged"] = np.int64(flagged)
    # operator-level samples
    rng = np.random.default_rng(5)
    lat = rng.normal(size=(6, 7, 5)) + 1j * rng.normal(size=(6, 7, 5))
    coords = rng.uniform(-0.5, [5.5, 6.5, 4.5], size=(400, 3))
    coords[:10] = [[0, 0, 0], [5, 6, 4], [4.999999, 6, 4], [1, 1, 1], [4, 5, 3],
                   [5, 6, 4.000001], [-1e-12, 2, 2], [2.5, 3.5, 1.5], [3, 3, 3], [1, 5, 3]]
    out["interp_lattice"] = lat
    out["interp_coords"] = coords
    for kern in ("linear", "cubic"):
        v, ok = hhsar._kernels.lattice_interpolate(lat, coords, kern)
        out[f"interp_{kern}"] = v
        out[f"interp_{kern}_ok"] = ok
    ext = rspec.SubarrayExtents.from_aperture(ap, tree.levels[0][1])
    tg = np.stack([g.origin + g.step * np.array(idx) for g in grids[1:2]
                   for idx in np.ndindex(*g.dims)])[::3]
    guesses = np.broadcast_to(np.array(region.center), tg.shape).copy()
    pos, ok, it = rspec.invert_lattice(ext, tg, guesses, freqs, max_step=0.5 * region.diagonal)
    out["newton_ext"] = np.array([ext.x_min, ext.x_max, ext.y_min, ext.y_max])
    out["newton_targets"] = tg
    out["newton_guesses"] = guesses
    out["newton_pos"] = pos
    out["newton_ok"] = ok
    out["newton_iters"] = it
    out["newton_max_step"] = np.float64(0.5 * region.diagonal)
    uvn_pts = rng.uniform([region.x_min, region.y_min, region.z_min],
                          [region.x_max, region.y_max, region.z_max], size=(64, 3))
    out["map_points"] = uvn_pts
    out["map_uvn"] = hhsar.llt_forward(ext, uvn_pts, freqs)
    out["map_phase"] = hhsar.sdc_phase(ext, uvn_pts, freqs)


def case_medium(out):
    from conftest import desk_aperture, desk_frequencies, desk_region, desk_scene
    freqs = desk_frequencies()
    ap = desk_aperture(side=17)
    region = desk_region(scale=0.5)
    cube = hhsar.simulate_measurement(desk_scene(scale=0.5), ap, freqs)
    dims = (33, 33, 17)
    out["cube"] = cube.values
    out["elements"] = ap.elements
    out["nxny"] = np.array([ap.nx, ap.ny])
    out["freqs"] = np.array([freqs.f_min, freqs.f_max, freqs.count])
    out["region"] = _region_arr(region)
    out["dims"] = np.array(dims)
    out["bpa"] = hhsar.bpa_reconstruct(cube, region, dims=dims).values
    for lv in (3, 4):
        vol = hhsar.hhffbpa_reconstruct(cube, region, final_dims=dims,
                                        params=hhsar.FfbpParams(levels=lv, gamma=1.4))
        out[f"hh_m{lv}"] = vol.values
        _prov(f"hh_m{lv}", vol, out)


def case_config0(out):
    w = workloads.config(0)
    cube_np = workloads.simulate_numpy(w)
    cube = _ref_cube(cube_np.values.astype(np.complex128), w.aperture.elements,
                     w.aperture.nx, w.aperture.ny, w.freqs)
    out["cube"] = cube_np.values  # complex64, the bytes both paths read
    out["elements"] = np.asarray(w.aperture.elements)
    out["nxny"] = np.array([w.aperture.nx, w.aperture.ny])
    out["freqs"] = np.array([w.freqs.f_min, w.freqs.f_max, w.freqs.count])
    out["region"] = _region_arr(w.region)
    out["dims"] = np.array(w.dims)
    region = hhsar.ImagingRegion(*_region_arr(w.region))
    out["bpa"] = hhsar.bpa_reconstruct(cube, region, dims=w.dims, upsample=8).values.astype(np.complex64)
    vol = hhsar.hhffbpa_reconstruct(cube, region, final_dims=w.dims,
                                    params=hhsar.FfbpParams(levels=7), upsample=8)
    out["hh_m7"] = vol.values.astype(np.complex64)
    _prov("hh_m7", vol, out)
    values, lp, mf, ff = factor4_reference(cube, region, w.dims, 7)
    out["hh_f4"] = values.astype(np.complex64)
    out["hh_f4_level_points"] = np.array([n for l in lp for n in l], dtype=np.int64)
    out["hh_f4_level_sizes"] = np.array([len(l) for l in lp], dtype=np.int64)
    out["hh_f4_merge_flags"] = np.array(mf, dtype=np.int64)
    out["hh_f4_final_flags"] = np.int64(ff)
    tree = hhsar.partition_subarrays(cube.aperture, 7)
    grids = [hhsar.build_subimage_grid(cube.aperture, sa, region, cube.freqs, 1.4, 0.25, pad=4)
             for lvl in tree.levels[:6] for sa in lvl]
    _grid_meta("grid", grids, out)


RUN_CONFIG = {  # a small desk-like run config in the reference's schema (cli.py:167-190)
    "aperture": {"nx": 9, "ny": 9, "extent": 0.0375,
                 "jitter": {"depth_amplitude": 0.0066, "lateral_sigma": 0.000125}},
    "frequencies": {"start_hz": 12.0e9, "stop_hz": 15.0e9, "count": 16},
    "region": {"center": [0.0, 0.0, 0.0333], "extents": [0.0417, 0.0417, 0.0417]},
    "scene": {"kind": "grid", "shape": [3, 3, 3], "spacing": 0.0146,
              "center": [0.0, 0.0, 0.0333]},
    "seed": 7,
    "algorithm": {"name": "hhffbpa", "levels": 3, "oversample": 1.4, "kernel": "linear"},
    "dims": [17, 17, 9],
}


def case_io():
    """Files written by the reference's own io.py and CLI: the byte formats
    and the config schema the drop-in must read and write identically."""
    import json
    from hhsar.cli import load_run_config, main as ref_main
    from hhsar.io import read_volume
    cfg_path = HERE / "run_config.json"
    cfg_path.write_text(json.dumps(RUN_CONFIG, indent=1))
    cube_path = HERE / "io_cube.bin"
    vol_path = HERE / "io_vol.bin"
    assert ref_main(["simulate", "--config", str(cfg_path), "--out", str(cube_path)]) == 0
    assert ref_main(["reconstruct", "--algo", "hhffbpa", "--levels", "3", "--in",
                     str(cube_path), "--out", str(vol_path), "--dims", "17,17,9"]) == 0
    cfg = load_run_config(cfg_path)
    out = {"elements": cfg.build_aperture().elements,
           "scene_positions": cfg.scene.positions,
           "volume": read_volume(vol_path).values}
    np.savez_compressed(HERE / "io_reference.npz", **out)


def case_cli_tools():
    """The reference CLI's `project` and `metrics` subcommands on the io
    case's volume (and a direct-BPA volume of the same cube): PGM bytes and
    the JSON report the drop-in's subcommands must reproduce."""
    from hhsar.cli import main as ref_main
    cube_path, vol_path = HERE / "io_cube.bin", HERE / "io_vol.bin"
    bpa_path = HERE / "io_bpa.bin"
    assert ref_main(["reconstruct", "--algo", "bpa", "--in", str(cube_path), "--out",
                     str(bpa_path), "--dims", "17,17,9"]) == 0
    for axis, depth in (("z", 8), ("x", 16)):
        assert ref_main(["project", "--in", str(vol_path), "--axis", axis, "--depth",
                         str(depth), "--out", str(HERE / f"io_proj_{axis}{depth}.pgm")]) == 0
    assert ref_main(["metrics", "--ref", str(bpa_path), "--test", str(vol_path),
                     "--out", str(HERE / "io_metrics.json")]) == 0


def case_metrics():
    """metrics.py outputs (psnr, max_intensity_projection, psf_metrics,
    profile_cut) on seeded volumes and profiles; error messages of the
    rejected inputs."""
    from hhsar.bpa import ImageVolume
    from hhsar import metrics as rm
    rng = np.random.default_rng(2026)
    dims = (12, 10, 9)
    origin, step = np.array([-0.05, -0.04, 0.2]), np.array([0.01, 0.009, 0.012])
    ref = rng.standard_normal(dims) + 1j * rng.standard_normal(dims)
    ref[5, 4, 3] = 12.0 - 3.0j  # a dominant peak
    noisy = ref * (0.7 - 0.4j) + 0.05 * (rng.standard_normal(dims) + 1j * rng.standard_normal(dims))
    ref64 = ref.astype(np.complex64)
    noisy64 = noisy.astype(np.complex64)
    out = {"dims": np.array(dims), "origin": origin, "step": step, "ref": ref, "noisy": noisy,
           "ref64": ref64, "noisy64": noisy64}
    V = lambda v: ImageVolume(v, origin, step)  # noqa: E731
    out["psnr_noisy"] = rm.psnr(V(ref), V(noisy))
    out["psnr_noisy64"] = rm.psnr(V(ref64.astype(np.complex128)), V(noisy64.astype(np.complex128)))
    out["psnr_same"] = rm.psnr(V(ref), V(ref.copy()))
    out["psnr_scaled"] = rm.psnr(V(ref), V(ref * (0.3 + 2.1j)))
    out["psnr_zero_test"] = rm.psnr(V(ref), V(np.zeros(dims, complex)))
    for ax in ("x", "y", "z"):
        for fl in (-40.0, -25.0):
            out[f"mip_{ax}_{int(-fl)}"] = rm.max_intensity_projection(V(ref), ax, fl)
    out["mip_zero"] = rm.max_intensity_projection(V(np.zeros(dims, complex)), 1)
    # PSF of a sampled sinc-like response (with a sidelobe floor) and a shifted copy
    x = np.arange(96) - 40.3
    prof = np.sinc(x / 3.7) * np.exp(0.3j * x) + 1e-3
    out["psf_profile"] = prof
    rep = rm.psf_metrics(prof, 0.002)
    out["psf"] = np.array([rep.mainlobe_width_mm, rep.pslr_db, rep.islr_db, rep.peak_position_m])
    cut, sp = rm.profile_cut(V(ref), "y", (0.0, 0.0, 0.23))
    out["cut_y"] = cut
    out["cut_spacing"] = sp
    errs = []
    for fn in (lambda: rm.psf_metrics(np.ones(64, complex), 0.002),
               lambda: rm.psf_metrics(np.zeros(64, complex), 0.002),
               lambda: rm.psf_metrics(prof[:3], 0.002),
               lambda: rm.psf_metrics(prof, 0.0),
               lambda: rm.psf_metrics(np.exp(-np.linspace(-2, 2, 65) ** 2).astype(complex), 0.01),
               lambda: rm.psf_metrics(np.array([8.2, 8.0, 8.5, 8.6, 9.0, 8.7, 8.1, 8.3, 1.0], complex), 0.01),
               lambda: rm.max_intensity_projection(V(ref), "w"),
               lambda: rm.max_intensity_projection(V(ref), 3),
               lambda: rm.max_intensity_projection(V(ref), "z", 0.0),
               lambda: rm.psnr(V(ref), ImageVolume(ref, origin + 1.0, step))):
        try:
            fn()
            errs.append("")
        except Exception as e:  # noqa: BLE001
            errs.append(f"{type(e).__name__}: {e}")
    out["errors"] = np.array(errs)
    np.savez_compressed(HERE / "metrics.npz", **out)


def main():
    if sys.argv[1:] == ["metrics"]:
        case_metrics()
        return
    if sys.argv[1:] == ["cli_tools"]:
        case_cli_tools()
        return
    case_io()
    case_cli_tools()
    case_metrics()
    for name, fn in (("small", case_small), ("medium", case_medium), ("config0", case_config0)):
        out = {}
        fn(out)
        path = HERE / f"{name}.npz"
        np.savez_compressed(path, **out)
        print(f"{path}: {path.stat().st_size / 1e6:.2f} MB, {len(out)} arrays")


if __name__ == "__main__":
    main()
