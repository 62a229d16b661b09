"""Build the sm_100a C-ABI library ``libaskv.so`` in-tree with nvcc.

    python -m paper_2403_19708_b200.build        # or __graft_entry__.build()

The .so is git-ignored but travels to the GPU box with the gpurun snapshot.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libaskv.so"
SOURCES = ["rope.cu", "attention.cu", "copy_engine.cu", "elementwise.cu", "runtime.cu",
           "collective.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    cand = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(cand):
        raise RuntimeError("nvcc not found")
    return cand


def _deps() -> list[Path]:
    return sorted([CSRC / s for s in SOURCES] + list(CSRC.glob("*.h")) +
                  list(CSRC.glob("*.cuh")) + [ROOT / "include" / "askv.h"])


def _src_hash() -> str:
    """Content hash of the sources and the build command: file copies (the
    gpurun snapshot) reorder mtimes, contents do not."""
    import hashlib
    h = hashlib.sha256(" ".join(ARCH).encode())
    for p in _deps():
        h.update(p.name.encode())
        h.update(p.read_bytes())
    return h.hexdigest()


STAMP = PKG / "libaskv.so.srchash"


def _stale() -> bool:
    if not LIB.exists():
        return True
    if STAMP.exists():
        return STAMP.read_text().strip() != _src_hash()
    t = LIB.stat().st_mtime
    return any(p.stat().st_mtime > t for p in _deps())


def build(force: bool = False, verbose: bool = False) -> Path:
    """Compile libaskv.so if its sources changed.  Safe to call from every
    rank of a multi-process run at once: one process compiles under an
    exclusive file lock, the others wait and then find it fresh."""
    if not force and not _stale():
        return LIB
    import fcntl
    with open(PKG / ".build.lock", "w") as lock:
        fcntl.flock(lock, fcntl.LOCK_EX)
        if not force and not _stale():
            return LIB
        tmp = LIB.with_suffix(f".so.tmp{os.getpid()}")
        cmd = [nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler",
               "-fPIC", "-Xptxas", "-v" if verbose else "-O3", "--expt-relaxed-constexpr",
               "-I", str(ROOT / "include"), "-o", str(tmp)]
        cmd += [str(CSRC / s) for s in SOURCES]
        cmd += ["-lcublasLt", "-ldl"]
        digest = _src_hash()
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            sys.stderr.write(res.stdout + res.stderr)
            tmp.unlink(missing_ok=True)
            raise RuntimeError("nvcc build of libaskv.so failed")
        if verbose:
            sys.stderr.write(res.stderr)
        os.replace(tmp, LIB)
        STAMP.write_text(digest + "\n")
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
