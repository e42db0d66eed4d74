"""TEST-ONLY: compile csrc/*.cu as host C++ against the SIMT emulation shim."""
from __future__ import annotations

import hashlib
import subprocess
from pathlib import Path

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
CSRC = ROOT / "paper_2601_13345_b200" / "csrc"
OUT = HERE / "_build"
LIB = OUT / "libffb_emul.so"


def build_emul(force: bool = False) -> Path:
    OUT.mkdir(exist_ok=True)
    srcs = sorted(CSRC.glob("*.cu"))
    h = hashlib.sha256()
    for p in [*srcs, *sorted(CSRC.glob("*.cuh")), ROOT / "include" / "ffb.h", HERE / "simt_emul.h",
              HERE / "simt_emul.cpp", Path(__file__)]:
        h.update(p.read_bytes())
    stamp = OUT / "stamp"
    if not force and LIB.exists() and stamp.exists() and stamp.read_text() == h.hexdigest():
        return LIB
    objs = []
    procs = []
    for src in [*srcs, HERE / "simt_emul.cpp"]:
        obj = OUT / (src.stem + ".o")
        cmd = ["g++", "-x", "c++", "-std=c++17", "-O1", "-g", "-fPIC", "-pthread", "-ffp-contract=off",
               "-DFFB_SIMT_EMUL", f"-I{HERE}", "-Wno-unused-value", "-c", str(src), "-o", str(obj)]
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
        objs.append(str(obj))
    for src, pr in procs:
        out, _ = pr.communicate()
        if pr.returncode != 0:
            raise RuntimeError(f"emul build failed on {src.name}:\n{out}")
    res = subprocess.run(["g++", "-shared", "-pthread", "-o", str(LIB), *objs], capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(res.stdout + res.stderr)
    stamp.write_text(h.hexdigest())
    return LIB


if __name__ == "__main__":
    print(build_emul(force=True))
