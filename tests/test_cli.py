"""CLI: host-only commands and exit codes on CPU; the
GPU commands are exercised in test_gpu_parity.py."""

import json
from pathlib import Path

import pytest

from paper_2410_16144_b200 import cli

GOLD = json.loads((Path(__file__).parent / "golden" / "tpk_golden.json").read_text())


def test_info_reference_file(tmp_path, capsys):
    path = tmp_path / "m.tpk"
    path.write_bytes(bytes.fromhex(GOLD["files"]["tl2"]))
    assert cli.main(["info", str(path)]) == 0
    out = capsys.readouterr().out
    assert "format: TL2" in out and "matrices: 3" in out and "layer0.wq: 5x37" in out
    assert "bits/weight: 1.67" in out


def test_exit_codes(tmp_path, capsys):
    bad = tmp_path / "bad.tpk"
    bad.write_bytes(bytes.fromhex(GOLD["errors"][0]["blob"]))
    assert cli.main(["info", str(bad)]) == 3
    assert "bad magic (at offset 0)" in capsys.readouterr().err
    assert cli.main(["info", str(tmp_path / "missing.tpk")]) == 3
    assert cli.main(["verify"]) == 2
    assert cli.main(["bench", "--config", "nope"]) == 2
    raw = tmp_path / "w.bin"
    raw.write_bytes(b"\0" * 12)
    assert cli.main(["pack", str(raw), str(tmp_path / "o.tpk"), "--rows", "2", "--cols", "2",
                     "--format", "i2s"]) == 3
    with pytest.raises(SystemExit):
        cli.main(["pack"])  # argparse usage error
