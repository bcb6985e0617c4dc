"""Build libfhv_b200.so in-tree for sm_100a (nvcc cross-compiles without a GPU).

    python -m paper_2211_15460_b200.build [--force]
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SOURCES = ["fhv_abi.cu", "fhv_scan.cu", "fhv_capture.cu", "fhv_splat.cu", "fhv_raycast.cu", "fhv_ops.cu"]
HEADERS = ["fhv_common.cuh", "fhv_internal.h", "fhv_lookback.cuh"]
OUT = os.path.join(HERE, "libfhv_b200.so")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    # exactness: never contract mul+add; explicit __fma_rn where numpy/BLAS fuse
    "-fmad=false", "-prec-div=true", "-prec-sqrt=true", "-ftz=false",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-ffp-contract=off",
    "-shared", "--expt-relaxed-constexpr", "-diag-suppress", "177,549",
]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    return "nvcc"


def up_to_date() -> bool:
    if not os.path.exists(OUT):
        return False
    t = os.path.getmtime(OUT)
    deps = [os.path.join(HERE, "csrc", f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "fhv_b200.h")]
    return all(os.path.getmtime(d) <= t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str | None = None, defines=()) -> str:
    """Compile the library (default: in-tree libfhv_b200.so).  ``out`` +
    ``defines`` build an experiment variant (e.g. a launch-bounds sweep) that
    ``FHV_LIB=<path>`` selects at load time."""
    if out is None and not force and up_to_date():
        return OUT
    out = out or OUT
    # one nvcc per translation unit, in parallel, then one link
    import concurrent.futures
    import tempfile
    tmp = tempfile.mkdtemp(prefix="fhv_build_")
    flags = [f for f in NVCC_FLAGS if f != "-shared"]
    objs = [os.path.join(tmp, f.replace(".cu", ".o")) for f in SOURCES]

    def compile_one(src_obj):
        src, obj = src_obj
        cmd = [_nvcc(), *flags, *[f"-D{d}" for d in defines], "-c", "-o", obj,
               os.path.join(HERE, "csrc", src)]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        subprocess.run(cmd, check=True, cwd=HERE)
    with concurrent.futures.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        list(ex.map(compile_one, zip(SOURCES, objs)))
    subprocess.run([_nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", out, *objs],
                   check=True, cwd=HERE)
    for o in objs:
        os.remove(o)
    os.rmdir(tmp)
    return out


if __name__ == "__main__":
    args = sys.argv[1:]
    o = args[args.index("--out") + 1] if "--out" in args else None
    defs = [args[i + 1] for i, a in enumerate(args) if a == "-D"]
    print(build(force="--force" in args, verbose="-v" in args, out=o, defines=defs))
