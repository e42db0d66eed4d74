"""CLI drop-in (next row f-1): analyze / predict / explore reports are byte-identical to the
reference CLI's (golden outputs in tests/golden/ref_cli.json), including exit codes and the
one-line JSON error records."""
from __future__ import annotations

import json
from pathlib import Path

from paper_2601_13345_b200 import cli

G = Path(__file__).parent / "golden"
CASES = json.loads((G / "ref_cli.json").read_text())
FIXT = json.loads((G / "ref_fixtures.json").read_text())["sources"]


def test_cli_reports_match_reference(backend, tmp_path, capsys):
    for case in CASES if backend == "gpu" else CASES[:6]:
        ptx = tmp_path / f"{case['fixture']}.ptx"
        ptx.write_text(FIXT[case["fixture"]])
        argv = [str(ptx) if a == "@PTX@" else a for a in case["argv"]]
        rc = cli.main(argv)
        got = capsys.readouterr()
        assert rc == case["rc"], case["argv"]
        assert got.out == case["stdout"], case["argv"]
        want_err = case["stderr"]
        if rc == 0:
            assert got.err.replace(str(ptx), "@PTX@") == want_err
        else:       # same error class in the JSON record; messages are free text
            assert json.loads(got.err.strip().splitlines()[-1])["error"] == json.loads(want_err.strip().splitlines()[-1])["error"]


def test_cli_usage_error_exit_code(backend):
    import pytest
    with pytest.raises(SystemExit) as ex:
        cli.main(["explore"])
    assert ex.value.code == 1
