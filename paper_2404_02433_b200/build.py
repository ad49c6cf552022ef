"""In-tree build of the CUDA extension: csrc/*.cu -> libetc_b200.so (sm_100a).

Each translation unit is compiled to an object in parallel, then the objects
are linked into one shared library.

    python -m paper_2404_02433_b200.build        # or __graft_entry__.build()
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
SOURCES = sorted(CSRC.glob("*.cu"))
HEADERS = [*sorted(CSRC.glob("*.cuh")), ROOT / "include" / "etc_b200.h"]
LIB = PKG / "libetc_b200.so"
OBJ = PKG / "build"

NVCC_FLAGS = [
    "-O3", "-std=c++17", "-lineinfo",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-Xcompiler", "-fPIC",
    "-Xptxas", "-v",
    "--expt-relaxed-constexpr",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def _obj(src: Path) -> Path:
    return OBJ / (src.stem + ".o")


def _stale_obj(src: Path) -> bool:
    o = _obj(src)
    if not o.exists():
        return True
    t = o.stat().st_mtime
    return src.stat().st_mtime > t or any(h.stat().st_mtime > t for h in HEADERS)


def stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    return any(d.stat().st_mtime > t for d in [*SOURCES, *HEADERS])


def _compile(src: Path) -> tuple[Path, subprocess.CompletedProcess]:
    cmd = [nvcc(), *NVCC_FLAGS, "-c", "-o", str(_obj(src)), str(src)]
    return src, subprocess.run(cmd, capture_output=True, text=True)


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not stale():
        return LIB
    OBJ.mkdir(exist_ok=True)
    todo = [s for s in SOURCES if force or _stale_obj(s)]
    log = []
    with ThreadPoolExecutor(max_workers=max(1, len(todo))) as ex:
        results = list(ex.map(_compile, todo))
    failed = False
    for src, proc in results:
        log.append(f"== {src.name}\n{proc.stdout}{proc.stderr}")
        if proc.returncode != 0:
            failed = True
            sys.stderr.write(proc.stderr[-8000:])
    tmp = LIB.with_suffix(".so.tmp")
    if not failed:
        cmd = [nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", str(tmp),
               *[str(_obj(s)) for s in SOURCES]]
        proc = subprocess.run(cmd, capture_output=True, text=True)
        log.append(" ".join(cmd) + "\n" + proc.stdout + proc.stderr)
        if proc.returncode != 0:
            failed = True
            sys.stderr.write(proc.stderr[-8000:])
    (PKG / "build.log").write_text("\n".join(log))
    if failed:
        raise RuntimeError(f"nvcc failed (see {PKG / 'build.log'})")
    if verbose:
        sys.stderr.write("\n".join(log))
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
