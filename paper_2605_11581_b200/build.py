"""In-tree build of libadamk.so (nvcc, sm_100a only).

The built library lives next to the sources (paper_2605_11581_b200/csrc/) so it
travels with a repo snapshot to the GPU box; it is git-ignored.
"""

from __future__ import annotations

import os
import shutil
import subprocess
from pathlib import Path

CSRC = Path(__file__).resolve().parent / "csrc"
LIB = CSRC / "libadamk.so"
SOURCES = [CSRC / "adamk.cu", CSRC / "prefill_gemm.cu", CSRC / "prefill_ops.cu", CSRC / "prefill_attn.cu", CSRC / "prefill_pass.cu"]
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
    "-shared", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
]


def find_nvcc() -> str:
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not Path(nvcc).exists():
        raise RuntimeError("nvcc not found; cannot build libadamk.so")
    return nvcc


def is_stale() -> bool:
    if not LIB.exists():
        return True
    deps = SOURCES + [CSRC.parents[1] / "include" / "adamk.h", CSRC.parents[1] / "include" / "adamk_prefill.h"]
    return any(d.stat().st_mtime > LIB.stat().st_mtime for d in deps)


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not is_stale():
        return LIB
    cmd = [find_nvcc(), *NVCC_FLAGS, "-o", str(LIB), *map(str, SOURCES)]
    res = subprocess.run(cmd, capture_output=True, text=True, env=dict(os.environ))
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed:\n{res.stdout}\n{res.stderr}")
    if verbose:
        print(res.stderr)
    (CSRC / "ptxas_info.txt").write_text(res.stderr)
    return LIB


if __name__ == "__main__":
    print(build(force=True, verbose=True))
