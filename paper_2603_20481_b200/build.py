"""In-tree build of the native library (sm_100a CUDA + C++ host code).

Produces ``paper_2603_20481_b200/_lib/libspecsense_b200.so``: the kernels,
the C ABI (include/specsense_b200.h) and the C++ drop-in API
(include/specsense/*.hpp).  Incremental on source mtimes; objects go to
``paper_2603_20481_b200/_lib/obj``.  Invoked by ``__graft_entry__.build()``.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = Path(os.environ.get("SSB_CSRC", PKG / "csrc"))  # override: A/B builds of patched sources
LIB = Path(os.environ.get("SSB_BUILD_DIR", PKG / "_lib"))
OBJ = LIB / "obj"
SO = LIB / "libspecsense_b200.so"

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
EXTRA = os.environ.get("SSB_NVCC_EXTRA", "").split()
NVCC_FLAGS = EXTRA + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-ffp-contract=off",
              "-Xptxas", "-v", f"-I{ROOT / 'include'}", f"-I{CSRC}"] + ARCH
CXX_FLAGS = ["-O2", "-std=c++20", "-fPIC", "-ffp-contract=off", "-Wall", "-Wextra",
             f"-I{ROOT / 'include'}", f"-I{CSRC}", "-I/usr/local/cuda/include"]

CU = ["fft_mag.cu", "floor.cu", "binarize.cu", "morph.cu", "ccl.cu", "baseline.cu", "capi.cu"]
CPP = ["host_consts.cpp", "dropin.cpp", "engine.cpp", "runtime_dropin.cpp", "baseline_host.cpp", "baseline_dropin.cpp"]
HEADERS = ["common.cuh", "internal.h", "glibc_libm.cuh", "baseline_host.h"]


def _deps_mtime() -> float:
    hs = [CSRC / h for h in HEADERS] + list((ROOT / "include").rglob("*.h*"))
    return max(p.stat().st_mtime for p in hs if p.exists())


def _compile(src: Path, verbose: bool) -> tuple[Path, str]:
    obj = OBJ / (src.name + ".o")
    if obj.exists() and obj.stat().st_mtime > max(src.stat().st_mtime, _deps_mtime()):
        return obj, ""
    if src.suffix == ".cu":
        cmd = [NVCC, *NVCC_FLAGS, "-c", str(src), "-o", str(obj)]
    else:
        cmd = ["g++", *CXX_FLAGS, "-c", str(src), "-o", str(obj)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    (OBJ / (src.name + ".ptxas.txt")).write_text(r.stderr)
    return obj, r.stderr if verbose else ""


def build(verbose: bool = False) -> Path:
    OBJ.mkdir(parents=True, exist_ok=True)
    srcs = [CSRC / f for f in CU + CPP if (CSRC / f).exists()]
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        results = list(ex.map(lambda s: _compile(s, verbose), srcs))
    objs = [o for o, _ in results]
    for _, log in results:
        if log:
            print(log, file=sys.stderr)
    if not SO.exists() or SO.stat().st_mtime < max(o.stat().st_mtime for o in objs):
        cmd = [NVCC, "-shared", *ARCH, "-o", str(SO), *map(str, objs), "-lcudart_static", "-lpthread", "-ldl", "-lrt"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return SO


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
