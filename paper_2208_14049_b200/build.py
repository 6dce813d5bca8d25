"""Build recipe for libenserve_b200.so (in-tree, sm_100a only).

Every translation unit under csrc/ is compiled by nvcc with
``-gencode arch=compute_100a,code=sm_100a -lineinfo`` and linked into one
shared library next to this file.  The CUDA runtime is linked statically so the
library loads on any box with the driver, independent of torch's copy.

    python -m paper_2208_14049_b200.build          # incremental
    python -m paper_2208_14049_b200.build --force  # rebuild everything
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
REPO = PKG.parent
CSRC = PKG / "csrc"
OBJ = REPO / "build" / "obj"
LIB = PKG / "libenserve_b200.so"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = [
    "-O3", "-lineinfo", "-std=c++20", "-Xcompiler", "-fPIC",
    "-Xcompiler", "-Wall", "--expt-relaxed-constexpr",
    f"-I{CSRC}", f"-I{REPO / 'include'}",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found: the enserve-b200 library cannot be built")


def sources() -> list[Path]:
    return sorted(p for p in CSRC.rglob("*") if p.suffix in (".cu", ".cpp"))


def headers() -> list[Path]:
    return sorted(p for p in list(CSRC.rglob("*")) + list((REPO / "include").rglob("*"))
                  if p.suffix in (".h", ".hpp", ".cuh"))


def _compile(src: Path, force: bool, newest_header: float) -> Path:
    obj = OBJ / (src.relative_to(CSRC).as_posix().replace("/", "__") + ".o")
    if not force and obj.exists() and obj.stat().st_mtime >= max(src.stat().st_mtime, newest_header):
        return obj
    obj.parent.mkdir(parents=True, exist_ok=True)
    lang = ["-x", "cu"] if src.suffix == ".cu" else ["-x", "c++"]
    cmd = [nvcc(), *ARCH, *COMMON, *lang, "-c", str(src), "-o", str(obj)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed on {src.name}:\n{res.stderr}")
    return obj


def build(force: bool = False, verbose: bool = False) -> Path:
    srcs = sources()
    newest_header = max((h.stat().st_mtime for h in headers()), default=0.0)
    with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as pool:
        objs = list(pool.map(lambda s: _compile(s, force, newest_header), srcs))
    if force or not LIB.exists() or LIB.stat().st_mtime < max(o.stat().st_mtime for o in objs):
        cmd = [nvcc(), *ARCH, "-shared", "-cudart", "static", "-o", str(LIB), *map(str, objs),
               "-lpthread", "-ldl", "-lrt"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"link failed:\n{res.stderr}")
    if verbose:
        print(f"built {LIB}")
    return LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    args = ap.parse_args()
    try:
        build(force=args.force, verbose=True)
    except RuntimeError as e:
        print(e, file=sys.stderr)
        sys.exit(1)
