"""Builds librapp_b200.so in-tree with nvcc for sm_100a (no JIT cache, no torch types).

    python -m paper_2505_01968_b200._build        # incremental
    python -m paper_2505_01968_b200._build --force
"""

from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "librapp_b200.so")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
# --fmad=false: no multiply-add contraction anywhere (bit parity with the reference's
# IEEE binary64 evaluation order); the kernels also use explicit _rn intrinsics.
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "--fmad=false", "-std=c++17",
    "-Xcompiler", "-fPIC,-O2", "-Xptxas", "-v",
    "-I" + os.path.join(ROOT, "include"),
]


def sources() -> list[str]:
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.h")) + \
        glob.glob(os.path.join(CSRC, "*.cuh")) + \
        glob.glob(os.path.join(ROOT, "include", "*.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str | None = None,
          defines: tuple[str, ...] = ()) -> str:
    """Builds the library; `out`/`defines` make tuning variants (e.g. RAPP_STREAM_ILP=1).
    Translation units compile in parallel (no device code crosses files), then link."""
    import concurrent.futures
    import tempfile
    target = out or LIB
    if out is None and not force and not _stale():
        return LIB
    tmp = target + ".tmp"
    flags = [*NVCC_FLAGS, *[f"-D{d}" for d in defines]]
    with tempfile.TemporaryDirectory() as objdir:
        def compile_one(src):
            obj = os.path.join(objdir, os.path.basename(src) + ".o")
            res = subprocess.run([NVCC, *flags, "-c", "-o", obj, src], capture_output=True,
                                 text=True)
            return src, obj, res
        srcs = sources()
        with concurrent.futures.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
            results = list(ex.map(compile_one, srcs))
        log = ""
        for src, _, res in results:
            log += res.stdout + res.stderr
            if res.returncode != 0:
                sys.stderr.write(res.stdout + res.stderr)
                raise RuntimeError(f"nvcc failed on {os.path.basename(src)}")
        res = subprocess.run([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared",
                              "-o", tmp, *[obj for _, obj, _ in results], "-lcudart"],
                             capture_output=True, text=True)
        if res.returncode != 0:
            sys.stderr.write(res.stdout + res.stderr)
            raise RuntimeError("nvcc failed linking librapp_b200.so")
    if verbose:
        sys.stderr.write(log)
    os.replace(tmp, target)
    return target


if __name__ == "__main__":
    defs = tuple(a[2:] for a in sys.argv[1:] if a.startswith("-D"))
    outs = [a[len("--out="):] for a in sys.argv[1:] if a.startswith("--out=")]
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv,
                out=outs[0] if outs else None, defines=defs))
