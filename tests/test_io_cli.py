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
