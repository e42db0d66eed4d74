"""f-3: authored spec files and the directory -> packed SoA loader (calibration.py:358-510 schema)."""
from __future__ import annotations

import json

import numpy as np
import pytest

from paper_2601_13345_b200 import errors as E
from paper_2601_13345_b200 import specs


def test_shipped_spec_files_load_and_pack():
    names, pairs, rows = specs.load_profiles()
    assert names == ["rtx3070", "rtx5000ada", "synthetic-48sm"]          # PAPER.md:254 + the built-in part
    assert rows.shape == (3, specs.SPEC_WIDTH) and rows.dtype == np.float64
    for (a, p), row in zip(pairs, rows):
        assert row.tolist() == specs.pack_spec(a, p)
    a, p = pairs[names.index("synthetic-48sm")]
    assert a == specs.default_architecture() and p == specs.default_calibration()
    assert rows[:, specs.SPEC_COLUMNS.index("regs_per_sm")].tolist() == [0.0, 0.0, 0.0]
    _, _, rows_r = specs.load_profiles(with_register_limit=True)
    assert rows_r[:, specs.SPEC_COLUMNS.index("regs_per_sm")].tolist() == [65536.0] * 3


def test_round_trip_is_the_identity(tmp_path):
    """Like pkg/tests/test_calibration.py:220: save -> load gives equal objects, and a directory of saved
    profiles packs to the same rows."""
    names, pairs, rows = specs.load_profiles()
    for n, (a, p) in zip(names, pairs):
        specs.save_profile(tmp_path / f"{n}.json", a, p)
        assert specs.load_profile(tmp_path / f"{n}.json") == (a, p)
    names2, pairs2, rows2 = specs.load_profiles(tmp_path)
    assert names2 == names and pairs2 == pairs and np.array_equal(rows2, rows)


def test_directory_errors(tmp_path):
    with pytest.raises(E.SchemaViolation):
        specs.load_profiles(tmp_path)                                   # empty directory
    obj = json.loads((specs.SPEC_DIR / "rtx3070.json").read_text())
    (tmp_path / "a.json").write_text(json.dumps(obj))
    (tmp_path / "b.json").write_text(json.dumps(obj))
    with pytest.raises(E.SchemaViolation, match="duplicate"):
        specs.load_profiles(tmp_path)
    (tmp_path / "b.json").unlink()
    obj["extensions"] = {"regs_per_sm": -1}
    (tmp_path / "a.json").write_text(json.dumps(obj))
    with pytest.raises(E.SchemaViolation, match="regs_per_sm"):
        specs.load_profiles(tmp_path, with_register_limit=True)
    del obj["architecture"]["bw_max"]
    (tmp_path / "a.json").write_text(json.dumps(obj))
    with pytest.raises(E.SchemaViolation, match="bw_max"):
        specs.load_profiles(tmp_path)
