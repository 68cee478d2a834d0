"""Build the in-tree CUDA library `_lib/libfgbd_b200.so` for sm_100a.

Plain nvcc, no torch extension machinery: the product is a C-ABI shared
library (include/fgbd_b200.h) with the CUDA runtime linked statically, so
it loads next to any torch build.  Objects are rebuilt only when a source
or header is newer than them.
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
INCLUDE = ROOT / "include"
OUT_DIR = PKG / "_lib"
LIB = OUT_DIR / "libfgbd_b200.so"
SOURCES = ["graph.cu", "noise.cu", "filter.cu", "stage.cu", "slab.cu", "ply.cu", "knn.cu", "measure.cu", "noisegen.cu", "hoststage.cu", "slg.cu", "api.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3",
              "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills"]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found; the B200 library cannot be built")


def _headers():
    return list(CSRC.glob("*.cuh")) + list(INCLUDE.glob("*.h"))


def build(verbose: bool = False, force: bool = False, ptxas_v: bool = False,
          defines: tuple = (), lib: Path | None = None) -> Path:
    """Build the library; `defines`/`lib` make an experiment variant (e.g.
    ("FGBD_LF_TLOG=1",) -> tools/_lib_tlog.so) in its own object directory."""
    nvcc = _nvcc()
    OUT_DIR.mkdir(exist_ok=True)
    LIB_OUT = Path(lib) if lib else LIB
    tag = "_".join(d.replace("=", "") for d in defines)
    obj_dir = ROOT / "build" / ("obj_" + tag if tag else "obj")
    obj_dir.mkdir(parents=True, exist_ok=True)
    hdr_mtime = max((h.stat().st_mtime for h in _headers()), default=0)
    objs = []
    cmds = []
    for src in SOURCES:
        s = CSRC / src
        o = obj_dir / (s.stem + ".o")
        objs.append(o)
        if not force and o.exists() and o.stat().st_mtime >= max(s.stat().st_mtime, hdr_mtime):
            continue
        cmd = [nvcc, *ARCH, *NVCC_FLAGS, *[f"-D{d}" for d in defines], f"-I{INCLUDE}", f"-I{CSRC}",
               "-c", str(s), "-o", str(o)]
        if ptxas_v:
            cmd[1:1] = ["-Xptxas", "-v"]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        cmds.append(cmd)
    rebuilt = bool(cmds)
    # one nvcc per source, in parallel (a clean build was ~2.5 min serially)
    from concurrent.futures import ThreadPoolExecutor

    with ThreadPoolExecutor(max_workers=max(1, min(len(cmds), os.cpu_count() or 1))) as ex:
        for r in list(ex.map(lambda c: subprocess.run(c), cmds)):
            if r.returncode != 0:
                raise subprocess.CalledProcessError(r.returncode, r.args)
    if rebuilt or force or not LIB_OUT.exists():
        tmp = LIB_OUT.with_suffix(".so.tmp")
        cmd = [nvcc, *ARCH, "-shared", "-o", str(tmp), *map(str, objs), "-cudart", "static"]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True)
        os.replace(tmp, LIB_OUT)
    return LIB_OUT


if __name__ == "__main__":
    build(verbose=True, force="--force" in sys.argv, ptxas_v="-v" in sys.argv)
    print(LIB)
