"""bench.py's CPU legs: the unmodified reference (oracle/_ref, when present) and the oracle port give the
same fronts for the same kernels - the cross-check bench.py repeats on the GPU box against the GPU step."""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import bench_extra  # noqa: E402
from paper_2601_13345_b200 import synth  # noqa: E402


def test_sample_is_bounded_and_rotates():
    _, offs = synth.ptx_corpus(4, 64, lo=20, hi=2000)
    a = bench_extra.cpu_sample_kernels(offs, 4, 0)
    b = bench_extra.cpu_sample_kernels(offs, 4, 1)
    sizes = np.diff(offs)
    assert len(a) == 4 and all(sizes[k] <= bench_extra.SAMPLE_MAX_BYTES for k in a + b) and a != b


@pytest.mark.skipif(bench_extra.cpu_kind() != "reference", reason="oracle/_ref (copy of the reference) not present")
def test_reference_and_port_agree_on_the_full_path():
    text, offs = synth.ptx_corpus(11, 3, lo=20, hi=60)
    srcs = [text[offs[i]:offs[i + 1]].decode("ascii") for i in range(3)]
    blocks = [7, 300, 65536]
    pr, br, fr = bench_extra._analysis_worker(("reference", srcs, blocks))
    pp, bp, fp = bench_extra._analysis_worker(("port", srcs, blocks))
    assert pr == pp == 3 * 3248 and br == bp
    assert fr == fp and all(len(f) > 0 for f in fr)
