"""Build libcurvekit_b200.so in-tree for sm_100a (nvcc cross-compiles without a GPU).

    python -m paper_1201_1548_b200.build        # incremental
    python -m paper_1201_1548_b200.build --force
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(REPO, "build", "obj")
OUT = os.path.join(HERE, "libcurvekit_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
         "--expt-relaxed-constexpr"]
SOURCES = ["ckb_capi.cu", "ckb_plan.cu", "ckb_images.cu", "ckb_interp.cu", "ckb_crt.cu", "ckb_gcd.cu", "ckb_general.cu",
           "ckb_peak.cu", "ckb_psc.cu", "ckb_crt_mma.cu",
           "ckb_descartes.cu", "ckb_bivgcd.cu"]
HEADERS = [os.path.join(CSRC, h) for h in os.listdir(CSRC) if h.endswith(".cuh")] + \
    [os.path.join(REPO, "include", "curvekit_b200.h")]


def _newest(paths):
    return max(os.path.getmtime(p) for p in paths)


def _compile(src: str, force: bool, obj: str = OBJ, extra=()) -> str:
    s = os.path.join(CSRC, src)
    o = os.path.join(obj, src.replace(".cu", ".o"))
    if not force and os.path.exists(o) and os.path.getmtime(o) >= _newest([s] + HEADERS):
        return o
    cmd = [NVCC, *ARCH, *FLAGS, *extra, "-c", s, "-o", o]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
    return o


def build(force: bool = False, verbose: bool = True, out: str = OUT, defines=()) -> str:
    """Build the library; `defines` (tuning experiments only) go to a separate object dir."""
    extra = [f"-D{d}" for d in defines]
    obj = OBJ if not extra else os.path.join(REPO, "build", "obj_" + "_".join(d.replace("=", "") for d in defines))
    os.makedirs(obj, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(lambda s: _compile(s, force, obj, extra), SOURCES))
    if force or not os.path.exists(out) or os.path.getmtime(out) < _newest(objs):
        cmd = [NVCC, *ARCH, "-shared", "-Xlinker", "--no-undefined", "-o", out, *objs, "-lcudart", "-ldl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
    if out == OUT:
        build_host(force)
    if verbose:
        print("built", out)
    return out


def build_host(force: bool = False) -> str:
    """The CPython helper that turns output limbs into Python ints (host glue)."""
    import sysconfig
    src = os.path.join(HERE, "host", "ckb_limbs.c")
    dst = os.path.join(HERE, "ckb_limbs" + sysconfig.get_config_var("EXT_SUFFIX"))
    if force or not os.path.exists(dst) or os.path.getmtime(dst) < os.path.getmtime(src):
        cmd = ["gcc", "-O3", "-shared", "-fPIC", "-I" + sysconfig.get_paths()["include"], src, "-o", dst, "-lm"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"host helper build failed:\n{r.stderr}")
    return dst


if __name__ == "__main__":
    build(force="--force" in sys.argv)
