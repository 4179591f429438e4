"""Build libdip.so in-tree: sm_100a kernels + C-ABI host code (nvcc, no JIT cache)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SO = os.path.join(HERE, "libdip.so")
SRCS = [os.path.join(HERE, "csrc", f) for f in ("dip_kernels.cu", "dip_order.cu", "dip_host.cpp", "dip_search.cpp",
                                                  "dip_plan.cpp", "dip_memopt.cu", "dip_memopt_host.cpp", "dip_ubench.cu", "dip_encode.cu")]
DEPS = SRCS + [os.path.join(HERE, "csrc", h) for h in ("dip_internal.h", "dip_host_internal.h")] + \
    [os.path.join(ROOT, "include", "dip.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def _nccl_dirs():
    """Link the NCCL that PyTorch itself loads (nvidia-nccl wheel), so that importing libdip before
    torch cannot pin an older system libnccl.so.2 into the process."""
    try:
        import nvidia.nccl as nn
        base = list(nn.__path__)[0]
        inc, lib = os.path.join(base, "include"), os.path.join(base, "lib")
        if os.path.exists(os.path.join(lib, "libnccl.so.2")):
            return inc, lib
    except ImportError:
        pass
    return None, None


def build(force: bool = False, verbose: bool = False, defines=(), out: str = SO) -> str:
    """Build libdip.so (or, with `defines` / `out`, a variant library for kernel A/B runs)."""
    if not force and os.path.exists(out) and all(os.path.getmtime(out) >= os.path.getmtime(d) for d in DEPS):
        return out
    cmd = [NVCC, "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
           "-Xcompiler", "-fPIC", "-shared", "-I", os.path.join(ROOT, "include"), "-I", os.path.join(HERE, "csrc"),
           *[f"-D{d}" for d in defines], *SRCS, "-o", out]
    inc, lib = _nccl_dirs()
    if inc:
        cmd[1:1] = ["-I", inc]
        cmd += ["-L", lib, "-l:libnccl.so.2", "-Xlinker", f"-rpath={lib}"]
    else:
        cmd += ["-lnccl"]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    subprocess.check_call(cmd)
    return out


if __name__ == "__main__":
    print(build(force=True, verbose="-v" in sys.argv))
