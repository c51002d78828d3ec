"""Build libfastfca_b200.so in-tree (sm_100a) with nvcc.

    python -m paper_1805_06572_b200.build [--verbose-ptxas] [--jobs N]

Each ``csrc/*.cu`` is compiled to an object in ``build/`` (parallel), then
linked into ``paper_1805_06572_b200/lib/libfastfca_b200.so``. Objects are
rebuilt only when a source or header is newer.
"""

from __future__ import annotations

import argparse
import os
import re
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
REPO = PKG.parent
CSRC = PKG / "csrc"
INCLUDE = REPO / "include"
BUILD = REPO / "build" / "csrc"
LIB = PKG / "lib" / "libfastfca_b200.so"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [
    "-O3",
    "-lineinfo",
    "-std=c++17",
    "-Xcompiler",
    "-fPIC",
    "-Xcompiler",
    "-O2",
    "--expt-relaxed-constexpr",
    "-Wno-deprecated-gpu-targets",
]


def nvcc():
    cand = os.environ.get("NVCC") or "/usr/local/cuda/bin/nvcc"
    return cand if Path(cand).exists() else "nvcc"


_INC = re.compile(r'^\s*#\s*include\s+"([^"]+)"', re.M)


def _deps(src: Path, seen=None):
    """Transitive quoted includes of ``src`` (for incremental rebuilds)."""
    seen = set() if seen is None else seen
    for name in _INC.findall(src.read_text()):
        dep = (src.parent / name).resolve()
        if dep.exists() and dep not in seen:
            seen.add(dep)
            _deps(dep, seen)
    return seen


def _needs(obj: Path, src: Path) -> bool:
    if not obj.exists():
        return True
    t = obj.stat().st_mtime
    return any(p.stat().st_mtime > t for p in [src, *_deps(src)])


def compile_one(src: Path, verbose_ptxas=False, build_dir=None, defines=()) -> Path:
    obj = (build_dir or BUILD) / (src.stem + ".o")
    if not _needs(obj, src):
        return obj
    cmd = [nvcc(), *ARCH, *NVCC_FLAGS, *[f"-D{d}" for d in defines], f"-I{INCLUDE}", "-c",
           str(src), "-o", str(obj)]
    if verbose_ptxas:
        cmd.insert(1, "-Xptxas=-v")
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src.name}:\n{res.stderr}")
    if verbose_ptxas and res.stderr:
        ((build_dir or BUILD) / (src.stem + ".ptxas.txt")).write_text(res.stderr)
    return obj


def build(verbose_ptxas=False, jobs=None, defines=(), out=None) -> Path:
    """Build the library; ``defines`` (experiment variants) go to a separate
    object directory and, with ``out``, to a separate .so (load it with
    FFCA_LIBRARY=<path>)."""
    lib_path = Path(out) if out else LIB
    bdir = BUILD if not defines else BUILD.parent / ("var-" + "-".join(
        d.replace("=", "_") for d in defines))
    bdir.mkdir(parents=True, exist_ok=True)
    lib_path.parent.mkdir(parents=True, exist_ok=True)
    sources = sorted(CSRC.glob("*.cu"))
    jobs = jobs or min(len(sources), os.cpu_count() or 4)
    with ThreadPoolExecutor(jobs) as ex:
        objs = list(ex.map(lambda s: compile_one(s, verbose_ptxas, bdir, defines), sources))
    if lib_path.exists() and all(lib_path.stat().st_mtime >= o.stat().st_mtime for o in objs):
        return lib_path
    tmp = lib_path.with_suffix(".so.tmp")
    cmd = [nvcc(), *ARCH, "-shared", "-o", str(tmp), *map(str, objs), "-lcudart"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{res.stderr}")
    os.replace(tmp, lib_path)
    return lib_path


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__)
    ap.add_argument("--verbose-ptxas", action="store_true")
    ap.add_argument("--jobs", type=int, default=None)
    ap.add_argument("--define", action="append", default=[],
                    help="extra -D for an experiment variant (needs --out)")
    ap.add_argument("--out", default=None, help="library path for a variant build")
    args = ap.parse_args(argv)
    if args.define and not args.out:
        ap.error("--define needs --out (variants never overwrite the shipped library)")
    lib = build(args.verbose_ptxas, args.jobs, tuple(args.define), args.out)
    print(lib)


if __name__ == "__main__":
    sys.exit(main())
