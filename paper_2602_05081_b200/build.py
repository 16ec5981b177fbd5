"""Build libgf.so (all CUDA kernels + the C ABI) for sm_100a with nvcc, in-tree.

    python -m paper_2602_05081_b200.build          # or __graft_entry__.build()

Static cudart, so the library only needs the driver (580+ supports CUDA 12.9).
"""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "_obj")
LIB = os.path.join(HERE, "libgf.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
SOURCES = ["gf_api.cu", "gf_build.cu", "gf_trace.cu", "gf_render.cu", "gf_ffa_pkt.cu", "gf_ffa_w.cu", "gf_ffb.cu", "gf_ff.cu", "gf_nee.cu"]
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xptxas", "-v", "--expt-relaxed-constexpr",
         "-I" + os.path.join(ROOT, "include"), "-I" + CSRC]


def _deps():
    files = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "gf.h")]
    return max(os.path.getmtime(f) for f in files)


def build(force=False, verbose=False, defines=(), lib=None, flags=()):
    """Build libgf.so; `defines` (e.g. ["GF_BATCH=16"]) / extra nvcc `flags` + `lib` build a tuning
    variant elsewhere."""
    lib = lib or LIB
    if not force and not defines and not flags and os.path.exists(lib) and os.path.getmtime(lib) >= _deps():
        return lib
    obj_dir = OBJ if not (defines or flags) else OBJ + "_" + os.path.basename(lib).replace(".so", "")
    os.makedirs(obj_dir, exist_ok=True)

    def comp(src):
        obj = os.path.join(obj_dir, src.replace(".cu", ".o"))
        cmd = [NVCC] + FLAGS + list(flags) + ["-D" + d for d in defines] + ["-c", os.path.join(CSRC, src), "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
        with open(os.path.join(obj_dir, src + ".ptxas.txt"), "w") as f:
            f.write(r.stderr)
        return obj

    with ThreadPoolExecutor(len(SOURCES)) as ex:
        objs = list(ex.map(comp, SOURCES))
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "static", "-o", lib] + objs
    subprocess.check_call(cmd)
    if verbose:
        for s in SOURCES:
            print(open(os.path.join(obj_dir, s + ".ptxas.txt")).read())
    return lib


def build_checked():
    """Debug variant with the device bounds checks (GF_DEBUG_CHECKS): variants/libgf_checked.so."""
    return build(defines=["GF_DEBUG_CHECKS"], lib=os.path.join(HERE, "variants", "libgf_checked.so"))


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
