"""File formats and the CLI drop-in against artefacts written by the
reference's own io.py / CLI (tests/golden/make_golden.py case_io).

CPU tests: config schema, byte formats, exit codes that fire before any GPU
work.  `gpu` tests: `reconstruct` / `simulate` through the CLI vs the
reference's files."""

import json
import shutil
from pathlib import Path

import numpy as np
import pytest

from paper_2506_23568_b200 import cli, io
from paper_2506_23568_b200.errors import ConfigError, IoFormatError

GOLD = Path(__file__).resolve().parent / "golden"


@pytest.fixture(scope="module")
def ref():
    return dict(np.load(GOLD / "io_reference.npz"))


def test_run_config_matches_reference_parse(ref):
    cfg = cli.load_run_config(GOLD / "run_config.json")
    assert np.array_equal(cfg.build_aperture().elements, ref["elements"])
    assert np.array_equal(cfg.scene.positions, ref["scene_positions"])
    assert cfg.dims == (17, 17, 9)
    assert cfg.algorithm == {"name": "hhffbpa", "levels": 3, "oversample": 1.4,
                             "kernel": "linear"}


def _write(tmp_path, doc):
    p = tmp_path / "cfg.json"
    p.write_text(json.dumps(doc))
    return p


@pytest.mark.parametrize("mutate,needle", [
    (lambda d: d.update(bogus=1), "unknown field(s) bogus"),
    (lambda d: d.pop("region"), "config.region: is required"),
    (lambda d: d["frequencies"].update(step_hz=1e6), "give exactly one of stop_hz or step_hz"),
    (lambda d: d["aperture"].update(nx=1), "aperture.nx: must be at least 2"),
    (lambda d: d.update(dims=[1, 2]), "config.dims: must be a list of 3 numbers"),
    (lambda d: d["algorithm"].update(kernel="nearest"), "must be 'linear' or 'cubic'"),
    (lambda d: d["scene"].update(center=[0, 0, 5.0]), "lies outside the imaging region"),
])
def test_config_validation_messages(tmp_path, mutate, needle):
    doc = json.loads((GOLD / "run_config.json").read_text())
    mutate(doc)
    with pytest.raises(ConfigError, match=None) as exc:
        cli.load_run_config(_write(tmp_path, doc))
    assert needle in str(exc.value)


def test_exit_codes_before_gpu_work(tmp_path, capsys):
    assert cli.main(["simulate", "--config", str(tmp_path / "absent.json"),
                     "--out", str(tmp_path / "c.bin")]) == 3
    bad = tmp_path / "bad.json"
    bad.write_text("{not json")
    assert cli.main(["simulate", "--config", str(bad), "--out", str(tmp_path / "c.bin")]) == 3
    doc = json.loads((GOLD / "run_config.json").read_text())
    doc["seed"] = -1
    assert cli.main(["simulate", "--config", str(_write(tmp_path, doc)),
                     "--out", str(tmp_path / "c.bin")]) == 2
    assert cli.main(["reconstruct", "--algo", "bpa", "--in", str(tmp_path / "none.bin"),
                     "--out", str(tmp_path / "v.bin")]) == 3
    assert cli.main(["reconstruct", "--algo", "bpa", "--in", str(GOLD / "io_cube.bin"),
                     "--out", str(tmp_path / "v.bin"), "--dims", "1,2"]) == 2
    assert cli.main(["--threads", "0", "reconstruct", "--algo", "bpa", "--in", "x",
                     "--out", "y"]) == 2


def test_cube_roundtrip_is_byte_identical(tmp_path):
    cube, region = io.read_cube(GOLD / "io_cube.bin")
    assert cube.values.dtype == np.complex64 and cube.values.shape == (81, 16)
    out = tmp_path / "c.bin"
    io.write_cube(out, cube, region=region,
                  provenance=json.loads((GOLD / "io_cube.bin.json").read_text())["provenance"])
    assert out.read_bytes() == (GOLD / "io_cube.bin").read_bytes()
    assert json.loads(io.sidecar_path(out).read_text()) == \
        json.loads((GOLD / "io_cube.bin.json").read_text())


def test_volume_roundtrip_is_byte_identical(tmp_path, ref):
    vol = io.read_volume(GOLD / "io_vol.bin")
    assert np.array_equal(vol.values, ref["volume"].astype(np.complex64))
    out = tmp_path / "v.bin"
    io.write_volume(out, vol)
    assert out.read_bytes() == (GOLD / "io_vol.bin").read_bytes()


def test_format_guards(tmp_path):
    shutil.copy(GOLD / "io_cube.bin", tmp_path / "c.bin")
    shutil.copy(GOLD / "io_cube.bin.json", tmp_path / "c.bin.json")
    with open(tmp_path / "c.bin", "ab") as fh:
        fh.write(b"\0" * 8)
    with pytest.raises(IoFormatError, match="dimension mismatch"):
        io.read_cube(tmp_path / "c.bin")
    (tmp_path / "c.bin").write_bytes((GOLD / "io_cube.bin").read_bytes()[:-8])
    with pytest.raises(IoFormatError, match="truncated"):
        io.read_cube(tmp_path / "c.bin")
    side = json.loads((GOLD / "io_cube.bin.json").read_text())
    side["schema"] = "other"
    (tmp_path / "c.bin.json").write_text(json.dumps(side))
    with pytest.raises(IoFormatError, match="schema mismatch"):
        io.read_cube(tmp_path / "c.bin")


@pytest.mark.gpu
def test_cli_reconstruct_matches_reference_file(tmp_path, ref):
    out = tmp_path / "v.bin"
    assert cli.main(["reconstruct", "--algo", "hhffbpa", "--levels", "3", "--in",
                     str(GOLD / "io_cube.bin"), "--out", str(out), "--dims", "17,17,9"]) == 0
    got = io.read_volume(out)
    want = ref["volume"]
    err = np.linalg.norm(got.values - want) / np.linalg.norm(want)
    assert err <= 1e-3, err
    assert got.provenance["level_points"] == json.loads(
        (GOLD / "io_vol.bin.json").read_text())["provenance"]["level_points"]


@pytest.mark.gpu
def test_cli_single_level_equals_direct(tmp_path):
    a, b = tmp_path / "bpa.bin", tmp_path / "one.bin"
    args = ["--in", str(GOLD / "io_cube.bin"), "--dims", "17,17,9"]
    assert cli.main(["reconstruct", "--algo", "bpa", "--out", str(a)] + args) == 0
    assert cli.main(["reconstruct", "--algo", "hhffbpa", "--levels", "1", "--out", str(b)]
                    + args) == 0
    assert io.read_volume(a).values.tobytes() == io.read_volume(b).values.tobytes()


@pytest.mark.gpu
def test_cli_simulate_matches_reference_cube(tmp_path):
    out = tmp_path / "c.bin"
    assert cli.main(["simulate", "--config", str(GOLD / "run_config.json"),
                     "--out", str(out)]) == 0
    got, region = io.read_cube(out)
    want, wregion = io.read_cube(GOLD / "io_cube.bin")
    err = np.linalg.norm(got.values - want.values) / np.linalg.norm(want.values)
    assert err < 1e-6, err
    assert region == wregion


# ---- project / metrics / bench subcommands and the PGM / report formats --------

@pytest.mark.parametrize("name,depth", [("io_proj_z8.pgm", 8), ("io_proj_x16.pgm", 16)])
def test_pgm_round_trip_of_reference_files(tmp_path, name, depth):
    img = io.read_projection(GOLD / name)
    assert img.min() >= 0.0 and img.max() == 1.0
    out = tmp_path / name
    io.export_projection(img, out, depth=depth)
    assert out.read_bytes() == (GOLD / name).read_bytes()


def test_pgm_and_report_validation(tmp_path):
    with pytest.raises(ConfigError, match="must be 2-D"):
        io.export_projection(np.zeros(4), tmp_path / "a.pgm")
    with pytest.raises(ConfigError, match=r"lie in \[0, 1\]"):
        io.export_projection(np.full((2, 2), 1.5), tmp_path / "a.pgm")
    with pytest.raises(ConfigError, match="depth must be 8 or 16"):
        io.export_projection(np.zeros((2, 2)), tmp_path / "a.pgm", depth=12)
    (tmp_path / "bad.pgm").write_bytes(b"P2\n1 1\n255\n\x00")
    with pytest.raises(IoFormatError, match="not a binary PGM"):
        io.read_projection(tmp_path / "bad.pgm")
    io.write_report(tmp_path / "r.json", {"b": 1, "a": [1.5]})
    assert json.loads((tmp_path / "r.json").read_text()) == {"a": [1.5], "b": 1}


def test_unexpected_errors_exit_1(tmp_path, capsys, monkeypatch):
    def boom(args):
        raise RuntimeError("boom")
    monkeypatch.setattr(cli, "cmd_project", boom)
    assert cli.main(["project", "--in", "x", "--out", str(tmp_path / "p.pgm")]) == 1
    assert "unexpected error: RuntimeError: boom" in capsys.readouterr().err


@pytest.mark.gpu
@pytest.mark.parametrize("axis,depth", [("z", 8), ("x", 16)])
def test_cli_project_matches_reference_pgm(tmp_path, axis, depth):
    out = tmp_path / "p.pgm"
    assert cli.main(["project", "--in", str(GOLD / "io_vol.bin"), "--axis", axis, "--depth",
                     str(depth), "--out", str(out)]) == 0
    assert out.read_bytes() == (GOLD / f"io_proj_{axis}{depth}.pgm").read_bytes()


@pytest.mark.gpu
def test_cli_metrics_matches_reference_report(tmp_path):
    out = tmp_path / "m.json"
    assert cli.main(["metrics", "--ref", str(GOLD / "io_bpa.bin"), "--test",
                     str(GOLD / "io_vol.bin"), "--out", str(out)]) == 0
    got = json.loads(out.read_text())
    want = json.loads((GOLD / "io_metrics.json").read_text())
    assert set(got) == set(want)
    assert abs(got["psnr_db"] - want["psnr_db"]) < 1e-6


@pytest.mark.gpu
def test_cli_bench_sweep_csv(tmp_path):
    out = tmp_path / "b.csv"
    assert cli.main(["bench", "--config", str(GOLD / "run_config.json"), "--sizes", "9,13",
                     "--out", str(out)]) == 0
    rows = out.read_text().splitlines()
    assert rows[0] == "size,algo,seconds,predicted_ops"
    body = [r.split(",") for r in rows[1:]]
    assert [(r[0], r[1]) for r in body] == [("9", "bpa"), ("9", "hhffbpa"), ("13", "bpa"),
                                            ("13", "hhffbpa")]
    assert all(float(r[2]) > 0 and float(r[3]) > 0 for r in body)
