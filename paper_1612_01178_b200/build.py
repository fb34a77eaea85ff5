"""Build libhookcc_cuda.so in-tree for sm_100a.

`python -m paper_1612_01178_b200.build` (or __graft_entry__.build()) compiles
every CUDA translation unit under csrc/ with
`nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3` and links the
C-ABI shared library into paper_1612_01178_b200/lib/.  Objects are rebuilt
only when a source or header is newer than the object.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OBJ = PKG / "build"
LIB = PKG / "lib"
SONAME = "libhookcc_cuda.so"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def _flags() -> list[str]:
    return ARCH + [
        "-lineinfo", "-O3", "-std=c++17", "--expt-relaxed-constexpr",
        "-Xcompiler", "-fPIC",
        "-I", str(ROOT / "include"), "-I", str(CSRC),
        "-DHCC_BUILDING_LIBRARY",
    ]


def _newest_header() -> float:
    hdrs = list(CSRC.glob("*.h")) + list(CSRC.glob("*.cuh")) + list((ROOT / "include").glob("*.h"))
    return max((h.stat().st_mtime for h in hdrs), default=0.0)


def _compile(src: Path, verbose: bool) -> Path:
    obj = OBJ / (src.stem + ".o")
    if obj.exists() and obj.stat().st_mtime >= max(src.stat().st_mtime, _newest_header()):
        return obj
    cmd = [nvcc(), *_flags(), "-Xptxas", "-v", "-c", str(src), "-o", str(obj)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    (OBJ / (src.stem + ".ptxas.log")).write_text(res.stdout + res.stderr)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"nvcc failed on {src.name}")
    if verbose:
        print(f"  compiled {src.name}")
    return obj


def build(verbose: bool = True) -> Path:
    OBJ.mkdir(exist_ok=True)
    LIB.mkdir(exist_ok=True)
    srcs = sorted(CSRC.glob("*.cu"))
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), srcs))
    out = LIB / SONAME
    if out.exists() and out.stat().st_mtime >= max(o.stat().st_mtime for o in objs):
        return out
    # The visibility script exports only the hcc_* C-ABI.
    vs = OBJ / "exports.map"
    vs.write_text("{ global: hcc_*; local: *; };\n")
    cmd = [nvcc(), *ARCH, "-shared", "-Xcompiler", "-fPIC", *[str(o) for o in objs],
           "-Xlinker", f"--version-script={vs}", "-Xlinker", f"-soname={SONAME}",
           "-o", str(out)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("link failed")
    if verbose:
        print(f"  linked {out.relative_to(ROOT)}")
    return out


if __name__ == "__main__":
    build()
