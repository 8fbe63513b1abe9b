"""Build libpolykv.so (sm_100a) in-tree with nvcc.

The shared library is the product: hand-written CUDA kernels plus a C ABI
(include/polykv.h). It is built with plain nvcc — no --use_fast_math, since
IEEE division and square root are part of the bit-exactness contract — and
with -lineinfo so ncu source pages map back to the kernels.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
CSRC = PKG_DIR / "csrc"
LIB_DIR = PKG_DIR / "lib"
LIB_PATH = LIB_DIR / "libpolykv.so"
INCLUDE = PKG_DIR.parent / "include"

ARCH_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [
    "-O3",
    "-std=c++17",
    "-lineinfo",
    "-Xcompiler",
    "-fPIC",
    "-Xcompiler",
    "-O3",
    "--expt-relaxed-constexpr",
]


def _nvcc() -> str:
    cand = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(cand):
        raise RuntimeError("nvcc not found; CUDA 12.9 toolkit required to build libpolykv.so")
    return cand


def sources() -> list[Path]:
    return sorted(list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cpp")))


def _stale() -> bool:
    if not LIB_PATH.exists():
        return True
    t = LIB_PATH.stat().st_mtime
    deps = sources() + list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h")) + list(INCLUDE.glob("*.h"))
    return any(p.stat().st_mtime > t for p in deps)


def build(force: bool = False, verbose: bool = False) -> Path:
    """Compile every csrc/*.cu and *.cpp into lib/libpolykv.so."""
    if not force and not _stale():
        return LIB_PATH
    return _compile(LIB_PATH, LIB_DIR / "obj", [], verbose)


def build_variant(name: str, defines: list[str], verbose: bool = False) -> Path:
    """A tuning build with extra -D flags: lib/variants/libpolykv_<name>.so,
    loaded instead of the default library when PKV_LIB_VARIANT=<name>."""
    out = LIB_DIR / "variants" / f"libpolykv_{name}.so"
    return _compile(out, LIB_DIR / "variants" / f"obj_{name}", [f"-D{d}" for d in defines], verbose)


def _compile(lib_path: Path, build_dir: Path, extra: list[str], verbose: bool) -> Path:
    lib_path.parent.mkdir(parents=True, exist_ok=True)
    nvcc = _nvcc()
    objs = []
    build_dir.mkdir(parents=True, exist_ok=True)
    procs = []
    for src in sources():
        obj = build_dir / (src.stem + ".o")
        cmd = [nvcc, *ARCH_FLAGS, *NVCC_FLAGS, *extra, "-I", str(INCLUDE), "-c", str(src), "-o", str(obj)]
        if src.suffix == ".cu":
            cmd.insert(1, "-Xptxas=-v" if verbose else "-Xptxas=-O3")
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        procs.append((cmd, subprocess.Popen(cmd)))  # translation units compile in parallel
        objs.append(obj)
    for cmd, pr in procs:
        if pr.wait() != 0:
            raise subprocess.CalledProcessError(pr.returncode, cmd)
    tmp = lib_path.with_suffix(".so.tmp")
    link = [nvcc, *ARCH_FLAGS, "-shared", "-cudart", "static", "-o", str(tmp), *map(str, objs)]
    subprocess.run(link, check=True)
    os.replace(tmp, lib_path)
    return lib_path


if __name__ == "__main__":
    if "--variant" in sys.argv:  # --variant NAME DEF=VAL ...
        i = sys.argv.index("--variant")
        print(build_variant(sys.argv[i + 1], sys.argv[i + 2:], verbose="-v" in sys.argv))
    else:
        build(force="--force" in sys.argv, verbose="-v" in sys.argv)
        print(LIB_PATH)
