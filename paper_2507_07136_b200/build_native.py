"""Build libsplatfield_b200.so (sm_100a) in-tree with nvcc.

Usage: python -m paper_2507_07136_b200.build_native [--force]
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "csrc", "obj")
LIB = os.path.join(HERE, "libsplatfield_b200.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
          "-Xptxas", "-v"] + ARCH
# Files whose fp64 arithmetic must follow the reference op order bit for bit:
# no FMA contraction except the explicit fma() calls that mirror BLAS.
NO_FMAD = {"sf_preprocess.cu", "sf_binning.cu"}
SOURCES = ["sf_preprocess.cu", "sf_binning.cu", "sf_sort.cu", "sf_blend.cu", "sf_splat_tc.cu", "sf_runtime.cu", "sf_post.cu", "sf_decode.cu",
           "sf_decode_tc.cu", "sf_io.cu", "sf_train.cu", "sf_capi.cu"]


def nvcc() -> str:
    p = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    return p


def _compile(src: str, log_dir: str) -> tuple[str, str]:
    out = os.path.join(OBJ, src.replace(".cu", ".o"))
    flags = list(COMMON)
    if src in NO_FMAD:
        flags.append("-fmad=false")
    flags += os.environ.get("SF_NVCC_DEFINES", "").split()  # development experiments only
    cmd = [nvcc(), "-c", os.path.join(CSRC, src), "-o", out] + flags
    r = subprocess.run(cmd, capture_output=True, text=True)
    with open(os.path.join(log_dir, src + ".log"), "w") as f:
        f.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr[-4000:]}")
    return out, r.stderr


def _stale(force: bool) -> bool:
    if force or not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in os.listdir(CSRC) if s.endswith((".cu", ".cuh"))]
    deps.append(os.path.join(HERE, "..", "include", "splatfield_b200.h"))
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False) -> str:
    if not _stale(force):
        return LIB
    os.makedirs(OBJ, exist_ok=True)
    srcs = [s for s in SOURCES if os.path.exists(os.path.join(CSRC, s))]
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        results = list(ex.map(lambda s: _compile(s, OBJ), srcs))
    objs = [o for o, _ in results]
    if verbose:
        for _, log in results:
            sys.stderr.write(log)
    tmp = LIB + ".tmp"
    cmd = [nvcc(), "-shared", "-o", tmp] + objs + ARCH + ["-Xcompiler", "-fPIC"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr[-4000:]}")
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
