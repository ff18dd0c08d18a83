"""Build libdualip.so in-tree for sm_100a (explicit nvcc, no JIT cache).

    python -m paper_2603_04621_b200.build          # or __graft_entry__.build()
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
import tempfile
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "lib")
LIB = os.path.join(LIBDIR, "libdualip.so")
SOURCES = [f"grad_m{m}_k{k}.cu" for m in (1, 2, 3, 4) for k in (0, 1, 2)] + ["plan.cpp", "grad.cu", "step.cu", "api.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def build(verbose: bool = False, extra: list[str] | None = None, out: str = LIB) -> str:
    """Compile every source (in parallel: the per-m kernel TUs dominate) and link ``out``."""
    os.makedirs(os.path.dirname(out), exist_ok=True)
    common = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-I", os.path.join(ROOT, "include"), *ARCH]
    if verbose:
        common += ["-Xptxas", "-v"]
    common += extra or []
    with tempfile.TemporaryDirectory(prefix="dualip_build_") as tmpdir:
        def compile_one(src):
            obj = os.path.join(tmpdir, src.rsplit(".", 1)[0] + ".o")
            lang = ["-x", "cu"] if src.endswith(".cpp") else []
            r = subprocess.run([nvcc(), *lang, *common, "-c", os.path.join(CSRC, src), "-o", obj],
                               capture_output=True, text=True)
            if r.returncode != 0:
                raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
            if verbose and r.stderr:
                sys.stderr.write(f"---- {src}\n{r.stderr}")
            return obj
        with ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 4)) as ex:
            objs = list(ex.map(compile_one, SOURCES))
        tmp = out + ".tmp"
        cmd = [nvcc(), *ARCH, "-shared", "-o", tmp, *objs, "-ldl", "-Xlinker", "--no-undefined"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
        os.replace(tmp, out)
    return out

if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
