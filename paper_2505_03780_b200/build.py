"""Build libb200attn.so for sm_100a with nvcc (in-tree, so the .so travels with the repo)."""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
REPO = PKG_DIR.parent
CSRC = PKG_DIR / "csrc"
OUT = PKG_DIR / "_lib" / "libb200attn.so"

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17", "--use_fast_math",
    "-Xcompiler", "-fPIC", "-shared", f"-I{REPO / 'include'}",
]


def sources():
    return sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cuh")) + [REPO / "include" / "b200attn.h"]


def needs_build() -> bool:
    if not OUT.exists():
        return True
    t = OUT.stat().st_mtime
    return any(s.stat().st_mtime > t for s in sources())


def build(force: bool = False, verbose: bool = False, trace: bool = False) -> Path:
    """trace: a separate debug library (-DB200_TRACE: clock/globaltimer timelines) at
    _lib/libb200attn_trace.so, loaded with B200ATTN_LIB=... by scripts/perf.py."""
    out = OUT.with_name("libb200attn_trace.so") if trace else OUT
    if not force and not trace and not needs_build():
        return OUT
    OUT.parent.mkdir(parents=True, exist_ok=True)
    cmd = [NVCC, *FLAGS, *(["-DB200_TRACE"] if trace else []), "-o", str(out) + ".tmp", str(CSRC / "capi.cu")]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"nvcc failed ({r.returncode})")
    if verbose:
        sys.stderr.write(r.stderr)
    os.replace(str(out) + ".tmp", out)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, trace="--trace" in sys.argv))
