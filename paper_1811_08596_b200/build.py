"""Build the in-tree C-ABI library ``libfgc_b200.so`` for sm_100a.

    python -m paper_1811_08596_b200.build [--force] [--verbose]

nvcc cross-compiles without a GPU; the .so is git-ignored but travels to the
GPU box with the gpurun snapshot.  NCCL comes from the torch-bundled
``nvidia/nccl`` wheel (headers + libnccl.so.2, linked with an rpath).
"""

from __future__ import annotations

import argparse
import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OUT = PKG / "libfgc_b200.so"
OBJ = ROOT / "build" / "obj"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dirs():
    import nvidia.nccl  # the torch-bundled NCCL (2.28.x)
    base = Path(list(nvidia.nccl.__path__)[0])
    return base / "include", base / "lib"


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def sources():
    return sorted(list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cpp")))


def headers():
    return list(CSRC.glob("*.h")) + list(CSRC.glob("*.cuh")) + [ROOT / "include" / "fgc_b200.h"]


def stale(force: bool) -> bool:
    if force or not OUT.exists():
        return True
    t = OUT.stat().st_mtime
    flags_file = PKG / "libfgc_b200.flags"
    if not flags_file.exists() or flags_file.read_text() != os.environ.get("FGC_NVCC_FLAGS", ""):
        return True
    return any(p.stat().st_mtime > t for p in sources() + headers() + [Path(__file__)])


def build(force: bool = False, verbose: bool = False) -> Path:
    if not stale(force):
        return OUT
    inc, lib = nccl_dirs()
    OBJ.mkdir(parents=True, exist_ok=True)
    cc = nvcc()
    common = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-O3", "-I", str(inc),
              "-I", str(ROOT / "include"), "--expt-relaxed-constexpr"]
    common += os.environ.get("FGC_NVCC_FLAGS", "").split()

    def compile_one(src: Path):
        obj = OBJ / (src.name + ".o")
        cmd = [cc, *ARCH, *common, "-c", str(src), "-o", str(obj)]
        if src.suffix == ".cu":
            cmd[1:1] = ["-Xptxas", "-v"] if verbose else []
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src.name}:\n{r.stderr}")
        if verbose and r.stderr:
            print(r.stderr, file=sys.stderr)
        return obj

    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(compile_one, sources()))
    tmp = OUT.with_suffix(".so.tmp")
    cmd = [cc, *ARCH, "-shared", "-o", str(tmp), *map(str, objs), "-L", str(lib), "-l:libnccl.so.2",
           "-Xlinker", f"-rpath={lib}", "-lpthread", "-ldl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    tmp.replace(OUT)
    (PKG / "libfgc_b200.flags").write_text(os.environ.get("FGC_NVCC_FLAGS", ""))
    return OUT


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    a = ap.parse_args()
    print(build(a.force, a.verbose))
