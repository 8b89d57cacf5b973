"""Build libcm.so (sm_100a) in-tree with nvcc. No JIT cache: the .so lives next
to this file so it travels to the GPU box with the repo snapshot."""

from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libcm.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo", "-O3", "-std=c++17",
    "-Xcompiler", "-fPIC",
    "-shared", "--expt-relaxed-constexpr",
]


# csrc/inst.cu is compiled once per (element type, reduce op): the kernel
# tables are the long pole of the build, so they are split ten ways
INST = [(t, tl, o, ol) for t, tl in (("BF16", "bf16"), ("F32", "f32"), ("F64", "f64"), ("I64", "i64"), ("I32", "i32"))
        for o, ol in (("CM_SUM", "sum"), ("CM_MAX", "max"))]


PYFAST_SRC = os.path.join(HERE, "csrc", "pyfast.cpp")


def sources():
    return sorted(f for f in glob.glob(os.path.join(HERE, "csrc", "*.cu")) if not f.endswith("inst.cu")) + \
        sorted(f for f in glob.glob(os.path.join(HERE, "csrc", "*.cpp")) if f != PYFAST_SRC)


def pyfast_path() -> str:
    import sysconfig
    return os.path.join(HERE, "_cmfast" + sysconfig.get_config_var("EXT_SUFFIX"))


def build_pyfast(verbose: bool = False) -> str:
    """The CPython fast-call module (csrc/pyfast.cpp). It does not link
    libcm.so: the ctypes binding hands it the entry points at import."""
    import sysconfig
    out = pyfast_path()
    cmd = [os.environ.get("CXX", "g++"), "-O2", "-std=c++17", "-fPIC", "-shared", "-Wall",
           "-I", sysconfig.get_paths()["include"], "-I", os.path.join(ROOT, "include"),
           PYFAST_SRC, "-o", out + ".tmp"]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    os.replace(out + ".tmp", out)
    return out


def pyfast_stale() -> bool:
    out = pyfast_path()
    return not os.path.exists(out) or any(
        os.path.getmtime(d) > os.path.getmtime(out) for d in (PYFAST_SRC, os.path.join(ROOT, "include", "cm.h")))


def units():
    """(source, object name, extra defines) for every translation unit."""
    inst = os.path.join(HERE, "csrc", "inst.cu")
    out = [(inst, f"inst_{tl}_{ol}.o", [f"-DCM_INST_T={t}", f"-DCM_INST_OP={o}",
                                        f"-DCM_INST_FN=cm_kernels_{tl}_{ol}"])
           for t, tl, o, ol in INST]
    return out + [(s, os.path.basename(s) + ".o", []) for s in sources()]


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + [os.path.join(HERE, "csrc", "inst.cu")] + glob.glob(os.path.join(HERE, "csrc", "*.h*")) + \
        glob.glob(os.path.join(HERE, "csrc", "*.cuh")) + [os.path.join(ROOT, "include", "cm.h")]
    return any(os.path.getmtime(d) > t for d in deps)


LIB_CHECKED = os.path.join(HERE, "libcm_checked.so")


def build(verbose: bool = False, extra=(), ptxas_log: str | None = None, checked: bool = False) -> str:
    """Compile every translation unit in parallel (the per-dtype kernel
    tables dominate), then link libcm.so. ``ptxas_log``: also write the
    `-Xptxas -v` register/spill report of every kernel to this file.
    ``checked``: the device-side bounds-checked variant (-DCM_CHECKED) as
    libcm_checked.so (load it with CM_LIB=...), for test runs only."""
    from concurrent.futures import ThreadPoolExecutor
    objdir = os.path.join(HERE, "build_checked" if checked else "build")
    lib = LIB_CHECKED if checked else LIB
    if checked:
        extra = (*extra, "-DCM_CHECKED")
    os.makedirs(objdir, exist_ok=True)
    inc = ["-I", os.path.join(ROOT, "include"), "-I", os.path.join(HERE, "csrc")]
    cflags = [f for f in FLAGS if f != "-shared"]

    def compile_one(unit):
        src, name, defs = unit
        obj = os.path.join(objdir, name)
        cmd = [NVCC, *cflags, *extra, *defs, *inc, "-c", src, "-o", obj]
        if ptxas_log:
            cmd += ["-Xptxas", "-v"]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        r = subprocess.run(cmd, capture_output=bool(ptxas_log), text=True)
        if r.returncode:
            sys.stderr.write((r.stderr or "") if ptxas_log else "")
            raise subprocess.CalledProcessError(r.returncode, cmd)
        return obj, (r.stderr or "") if ptxas_log else ""

    todo = units()
    with ThreadPoolExecutor(max_workers=min(len(todo), os.cpu_count() or 4)) as ex:
        res = list(ex.map(compile_one, todo))
    objs = [o for o, _ in res]
    if ptxas_log:
        with open(ptxas_log, "w") as fh:
            for (_, name, _), (_, log) in zip(todo, res):
                fh.write(f"==== {name}\n{log}")
    cmd = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", *objs, "-o", lib + ".tmp"]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    os.replace(lib + ".tmp", lib)
    return lib


if __name__ == "__main__":
    args = sys.argv[1:]
    log = None
    checked = "--checked" in args
    args = [a for a in args if a != "--checked"]
    if args and args[0].startswith("--ptxas-log="):
        log = args.pop(0).split("=", 1)[1]
    print(build(verbose=True, extra=args, ptxas_log=log, checked=checked))
    if not checked:
        print(build_pyfast(verbose=True))
