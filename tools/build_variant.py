"""Build an experimental variant of libhookcc_cuda.so for A/B timing.

python tools/build_variant.py NAME [--rev GITREV] [-DMACRO=VAL ...]

Compiles csrc/*.cu (from the working tree, or from git revision GITREV) with
the extra -D flags into paper_1612_01178_b200/lib/variants/NAME.so
(git-ignored; it travels to the GPU box with the snapshot).  Load it with
HCC_LIB=paper_1612_01178_b200/lib/variants/NAME.so.
"""
from __future__ import annotations

import argparse
import subprocess
import sys
import tempfile
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_1612_01178_b200 import build as B  # noqa: E402


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("name")
    ap.add_argument("--rev")
    args, defines = ap.parse_known_args()
    args.defines = defines
    tmp = Path(tempfile.mkdtemp(prefix=f"hcc_var_{args.name}_"))
    if args.rev:
        arch = subprocess.run(["git", "-C", str(ROOT), "archive", args.rev,
                               "paper_1612_01178_b200/csrc", "include"],
                              check=True, capture_output=True).stdout
        subprocess.run(["tar", "-x", "-C", str(tmp)], input=arch, check=True)
        csrc, inc = tmp / "paper_1612_01178_b200" / "csrc", tmp / "include"
    else:
        csrc, inc = B.CSRC, ROOT / "include"
    flags = [f for f in B._flags() if f not in (str(B.CSRC), str(ROOT / "include"))]
    flags += ["-I", str(inc), "-I", str(csrc), *args.defines]
    objs = []
    for src in sorted(csrc.glob("*.cu")):
        obj = tmp / (src.stem + ".o")
        subprocess.run([B.nvcc(), *flags, "-c", str(src), "-o", str(obj)], check=True)
        objs.append(str(obj))
    out = B.LIB / "variants" / f"{args.name}.so"
    out.parent.mkdir(parents=True, exist_ok=True)
    vs = tmp / "exports.map"
    vs.write_text("{ global: hcc_*; local: *; };\n")
    subprocess.run([B.nvcc(), *B.ARCH, "-shared", "-Xcompiler", "-fPIC", *objs,
                    "-Xlinker", f"--version-script={vs}", "-o", str(out)], check=True)
    print(out.relative_to(ROOT))


if __name__ == "__main__":
    main()
