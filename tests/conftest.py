from __future__ import annotations

import sys
from pathlib import Path

import pytest
import torch

ROOT = Path(__file__).resolve().parent.parent
for p in (ROOT, ROOT / "tests" / "simt", ROOT / "oracle"):
    if str(p) not in sys.path:
        sys.path.insert(0, str(p))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device and the nvcc-built libffb.so")


_EMUL = {}


def _emul_runtime():
    """SIMT-emulated build of csrc/*.cu on host memory (test-only, see tests/simt)."""
    if "rt" not in _EMUL:
        from build_emul import build_emul
        from paper_2601_13345_b200 import native
        lib = native.bind(build_emul())
        _EMUL["rt"] = native.Runtime(lib, torch.device("cpu"))
    return _EMUL["rt"]


@pytest.fixture(params=["emul", pytest.param("gpu", marks=pytest.mark.gpu)])
def backend(request):
    """Installs the runtime the shim uses: emulated kernels (CPU suite) or the real library."""
    from paper_2601_13345_b200 import native
    if request.param == "emul":
        native.install_runtime_for_tests(_emul_runtime())
        yield "emul"
        native.install_runtime_for_tests(None)
    else:
        native.install_runtime_for_tests(None)
        if not torch.cuda.is_available():
            pytest.fail("gpu-marked test selected but no CUDA device is visible")
        native.get_runtime()       # raises NativeLibraryMissing when libffb.so is absent
        yield "gpu"


@pytest.fixture
def gpu_only():
    from paper_2601_13345_b200 import native
    native.install_runtime_for_tests(None)
    if not torch.cuda.is_available():
        pytest.fail("gpu-marked test selected but no CUDA device is visible")
    return native.get_runtime()
