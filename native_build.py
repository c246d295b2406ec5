"""Build libsc_b200.so (the C-ABI library) in-tree with nvcc for sm_100a.

    python native_build.py [--verbose-ptxas]

Sources: paper_1509_08863_b200/csrc/*.cu, *.cpp; public header include/sc_b200.h.
The .so lands next to the Python binding (paper_1509_08863_b200/libsc_b200.so)
so it travels with the repo snapshot to the GPU box.
"""

from __future__ import annotations

import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.abspath(__file__))
PKG = os.path.join(ROOT, "paper_1509_08863_b200")
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(ROOT, "build", "native")
LIB = os.path.join(PKG, "libsc_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_dirs():
    """NCCL headers/library: the copy bundled with torch (the one torch.distributed loads,
    so both share one libnccl.so.2 in the process), else the system one."""
    import sysconfig
    base = os.path.join(sysconfig.get_paths()["purelib"], "nvidia", "nccl")
    inc, lib = os.path.join(base, "include"), os.path.join(base, "lib")
    if os.path.exists(os.path.join(inc, "nccl.h")) and os.path.exists(os.path.join(lib, "libnccl.so.2")):
        return inc, lib
    return "/usr/include", "/usr/lib/x86_64-linux-gnu"


NCCL_INC, NCCL_LIB = _nccl_dirs()
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-O3", "-I", os.path.join(ROOT, "include"),
          "-I", CSRC, "-I", NCCL_INC]


def _compile(src: str, verbose_ptxas: bool, defs=(), tag="") -> str:
    obj = os.path.join(BUILD, os.path.basename(src) + tag + ".o")
    deps = [src] + glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "sc_b200.h")]
    if os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(d) for d in deps):
        return obj
    cmd = [NVCC, *ARCH, *COMMON, *defs, "-c", src, "-o", obj]
    if src.endswith(".cpp"):
        cmd = [NVCC, *COMMON, "-x", "c++", "-c", src, "-o", obj]
    elif verbose_ptxas:
        cmd.insert(1, "-Xptxas=-v")
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    if verbose_ptxas and r.stderr:
        print(r.stderr)
    return obj


def build(verbose_ptxas: bool = False, defs=(), out: str = LIB) -> str:
    """Compile every source and link ``out``.  ``defs`` (e.g. ["-DSC_EB_F32=12"]) build a
    tuning variant; its objects get their own names so variants do not clobber each other."""
    os.makedirs(BUILD, exist_ok=True)
    import re
    tag = "" if not defs else "." + re.sub(r"[^A-Za-z0-9]+", "_", "_".join(d.lstrip("-D") for d in defs))
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))
    with ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose_ptxas, defs, tag), srcs))
    if os.path.exists(out) and os.path.getmtime(out) >= max(os.path.getmtime(o) for o in objs):
        return out
    nccl = os.path.join(NCCL_LIB, "libnccl.so.2")
    cmd = [NVCC, *ARCH, "-shared", "-o", out, *objs, "-Xlinker", nccl, "-Xlinker", f"-rpath={NCCL_LIB}",
           "-lcudart_static", "-lrt", "-ldl", "-lpthread"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    check_sass(out)
    return out


def check_sass(lib: str) -> None:
    """Reject SASS whose 64-bit memory descriptor sits in an odd uniform register pair
    (desc[UR1], desc[UR3], ...): a misaligned wide operand that faults at run time with
    cudaErrorIllegalInstruction.  ptxas 12.9 emitted it once for cp.async with an L2 cache
    hint (round 2, SELL kernel)."""
    import re
    cuobjdump = os.path.join(os.path.dirname(NVCC), "cuobjdump")
    r = subprocess.run([cuobjdump, "-sass", lib], capture_output=True, text=True)
    if r.returncode != 0:
        return
    bad, fn = [], ""
    for ln in r.stdout.splitlines():
        if "Function :" in ln:
            fn = ln.split("Function :")[1].strip()
        elif re.search(r"(?<![a-z])desc\[UR\d*[13579]\]", ln):   # memory descriptors only (not idesc/gdesc)
            bad.append(fn)
    if bad:
        os.remove(lib)
        raise RuntimeError("SASS with a misaligned (odd) uniform descriptor register in: " + ", ".join(sorted(set(bad))))


if __name__ == "__main__":
    defs = sys.argv[sys.argv.index("--defs") + 1].split() if "--defs" in sys.argv else []
    out = sys.argv[sys.argv.index("--out") + 1] if "--out" in sys.argv else LIB
    print(build(verbose_ptxas="--verbose-ptxas" in sys.argv, defs=defs, out=out))
