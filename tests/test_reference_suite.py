"""The reference's OWN unit tests (pkg/tests/test_{ptx_parser,cfg,alignment,features,time_model,
power_model,explorer}.py) run against the drop-in through the `ptxwatt` import path of
paper_2601_13345_b200.compat.  Only possible where /root/reference exists (the build container);
skipped elsewhere - the GPU box runs the committed goldens instead.  The CPU run uses the
SIMT-emulated kernels."""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
REF_TESTS = Path("/root/reference/pkg/tests")
FILES = ("test_ptx_parser.py", "test_cfg.py", "test_alignment.py", "test_features.py", "test_time_model.py",
         "test_power_model.py", "test_explorer.py")

RUNNER = r'''
import sys
sys.path.insert(0, {root!r}); sys.path.insert(0, {root!r} + "/tests"); sys.path.insert(0, {root!r} + "/tests/simt"); sys.path.insert(0, {root!r} + "/oracle")
from paper_2601_13345_b200 import compat, native
sys.path.insert(0, compat.PATH)
import torch
if {emul!r}:
    from build_emul import build_emul
    native.install_runtime_for_tests(native.Runtime(native.bind(build_emul()), torch.device("cpu")))
import ptxwatt
assert "compat" in ptxwatt.__file__, ptxwatt.__file__
import pytest
sys.exit(pytest.main(["-q", "-x", "-p", "no:cacheprovider", "--rootdir", {tests!r},
                      *[{tests!r} + "/" + f for f in {files!r}]]))
'''


def _run(emul: bool):
    code = RUNNER.format(root=str(ROOT), emul=emul, tests=str(REF_TESTS), files=FILES)
    env = dict(os.environ)
    env.pop("PYTHONPATH", None)
    res = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd="/tmp", env=env, timeout=1500)
    tail = (res.stdout + res.stderr)[-3000:]
    assert res.returncode == 0, tail
    assert " passed" in res.stdout and "failed" not in res.stdout.splitlines()[-1], tail


@pytest.mark.skipif(not REF_TESTS.exists(), reason="the reference tree is only present in the build container")
def test_reference_unit_tests_pass_against_the_dropin_emulated():
    _run(emul=True)


@pytest.mark.gpu
@pytest.mark.skipif(not REF_TESTS.exists(), reason="the reference tree is only present in the build container")
def test_reference_unit_tests_pass_against_the_dropin_gpu():
    _run(emul=False)
