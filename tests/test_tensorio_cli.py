"""TNS1 files and report JSON, CPU only; the GPU CLI run
is in test_gpu_parity.py."""
import json
import os
import struct

import numpy as np
import pytest

from conftest import GOLDEN

from paper_2511_11571_b200.core import FormatError, LengthError, ShapeError
from paper_2511_11571_b200.tensorio import RunReport, Tensor, tensor_read, tensor_write

NAMES = ["tns1_f32_rank2", "tns1_f64_rank3", "tns1_f64_rank1"]


@pytest.mark.parametrize("name", NAMES)
def test_tns1_byte_identical_to_reference(name, tmp_path):
    """Files written by the reference's tensor_write (tests/golden/make_tns1.py)
    read back exactly and are rewritten byte for byte."""
    src = os.path.join(GOLDEN, name + ".bin")
    t = tensor_read(src)
    out = tmp_path / "x.bin"
    tensor_write(t, out)
    assert open(src, "rb").read() == open(out, "rb").read()
    assert tensor_read(out).array.dtype == t.array.dtype
    np.testing.assert_array_equal(tensor_read(out).array, t.array)


def _blob(magic=b"TNS1", version=1, code=0, rank=2, reserved=0, dims=(2, 3), payload=None):
    head = struct.pack("<4sIBBH", magic, version, code, rank, reserved) + np.asarray(dims, "<u8").tobytes()
    if payload is None:
        payload = np.zeros(int(np.prod(dims)), "<f4" if code == 0 else "<f8").tobytes()
    return head + payload


@pytest.mark.parametrize("blob,err", [
    (_blob(magic=b"TNS2"), FormatError),
    (_blob(version=2), FormatError),
    (_blob(code=7), FormatError),
    (_blob(rank=4, dims=(1, 1, 1, 1)), FormatError),
    (_blob(reserved=1), FormatError),
    (_blob(dims=(0, 3)), FormatError),
    (_blob()[:10], LengthError),
    (_blob()[:-4], LengthError),
    (_blob() + b"\0\0\0\0", LengthError),
    (_blob(payload=np.array([np.nan] * 6, "<f4").tobytes()), FormatError),
])
def test_tns1_rejects_malformed(blob, err, tmp_path):
    p = tmp_path / "bad.bin"
    p.write_bytes(blob)
    with pytest.raises(err):
        tensor_read(p)


def test_tensor_validation():
    for bad in (np.zeros((2, 2), np.int32), np.zeros((1, 1, 1, 1)), np.array([np.inf])):
        with pytest.raises(ShapeError):
            Tensor(bad)


def test_report_matches_reference_schema():
    """src/report_schema.json: exactly command/config/metrics/pass/version,
    metrics are numbers or number lists, strict JSON."""
    r = RunReport("bench", {"n": [1, 2]}, {"a": 1.0, "b": [1.0, 2.0]}, True)
    d = json.loads(r.to_json())
    assert set(d) == {"command", "config", "metrics", "pass", "version"}
    assert isinstance(d["pass"], bool) and isinstance(d["version"], str)
    for v in d["metrics"].values():
        assert isinstance(v, (int, float)) or all(isinstance(x, (int, float)) for x in v)
    with pytest.raises(ValueError):
        RunReport("x", {}, {"bad": float("nan")}).to_json()


def test_cli_settings_layers(tmp_path):
    """defaults < --config JSON object < explicit flags; unknown config keys
    and missing required options are ConfigErrors (src/cli.py:54-68)."""
    from paper_2511_11571_b200 import cli
    from paper_2511_11571_b200.core import ConfigError
    cfg = tmp_path / "c.json"
    cfg.write_text(json.dumps({"topk": 3, "block": 32, "k": "kk", "v": "vv", "out": "o"}))
    args = cli.build_parser().parse_args(["attend", "--q", "a", "--block", "64", "--config", str(cfg)])
    s = cli.settings(cli.ATTEND, args)
    assert (s["q"], s["block"], s["topk"], s["conv"], s["mode"]) == ("a", 64, 3, 0, "fp32")   # flag > file > default
    cfg.write_text(json.dumps({"nope": 1}))
    with pytest.raises(ConfigError):
        cli.settings(cli.ATTEND, args)
    args = cli.build_parser().parse_args(["attend", "--q", "a"])
    with pytest.raises(ConfigError):
        cli.settings(cli.ATTEND, args)            # --k / --v / --out missing
    b = cli.settings(cli.BENCH, cli.build_parser().parse_args(["bench", "--n", "256,512"]))
    assert b["n"] == "256,512" and b["block"] == 128 and b["dim"] == 64


def test_cli_errors_exit_2(tmp_path, capsys):
    from paper_2511_11571_b200 import cli
    rc = cli.main(["attend", "--q", "a"])
    assert rc == 2
    err = json.loads(capsys.readouterr().err)
    assert err["error"] == "ConfigError"
    rc = cli.main(["bench", "--n", "64", "--block", "128"])     # N shorter than the block
    assert rc == 2
