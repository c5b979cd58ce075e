"""Build libpaste.so in-tree for sm_100a (python -m paper_2603_18897_b200.build)."""

from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libpaste.so")

COMPILE_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "--fmad=false",            # fp64 utilities / EWMA must round like the reference
    "-Xcompiler", "-fPIC", "-Xcompiler", "-fopenmp",
    "-Xptxas", "-v",
]
LINK_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-lgomp",
              "-cudart=static", "-Xcompiler", "-fopenmp"]
NVCC_FLAGS = COMPILE_FLAGS + LINK_FLAGS  # kept for scripts that print the recipe
OBJ = os.path.join(ROOT, "build", "obj")


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    return "nvcc"


PYEXT_SRC = os.path.join(CSRC, "tapes_py.cpp")  # CPython extension, built apart


def sources() -> list[str]:
    return sorted(f for f in glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp"))
                  if f != PYEXT_SRC)


def pyext_path() -> str:
    import sysconfig

    return os.path.join(HERE, "_tapes" + sysconfig.get_config_var("EXT_SUFFIX"))


def build_pyext(force: bool = False) -> str:
    """The native payload-tape encoder (csrc/tapes_py.cpp) as an in-tree
    CPython extension module (host code: g++)."""
    import sysconfig

    out = pyext_path()
    if not force and os.path.exists(out) and os.path.getmtime(out) > os.path.getmtime(PYEXT_SRC):
        return out
    cmd = [os.environ.get("CXX", "g++"), "-O3", "-std=c++17", "-shared", "-fPIC",
           "-I", sysconfig.get_paths()["include"], PYEXT_SRC, "-o", out + ".tmp"]
    proc = subprocess.run(cmd, capture_output=True, text=True)
    if proc.returncode != 0:
        sys.stderr.write(proc.stdout + proc.stderr)
        raise RuntimeError("g++ failed building the tape encoder extension")
    os.replace(out + ".tmp", out)
    return out


def needs_build() -> bool:
    if not os.path.exists(OUT):
        return True
    mtime = os.path.getmtime(OUT)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "paste.h")]
    return any(os.path.getmtime(d) > mtime for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    build_pyext(force)
    if not force and not needs_build():
        return OUT
    # one nvcc per translation unit, in parallel, then one link
    from concurrent.futures import ThreadPoolExecutor

    os.makedirs(OBJ, exist_ok=True)
    inc = ["-I", os.path.join(ROOT, "include"), "-I", CSRC]

    headers = glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "paste.h")]
    newest_header = max(os.path.getmtime(h) for h in headers)

    def compile_one(src: str):
        obj = os.path.join(OBJ, os.path.basename(src) + ".o")
        if (not force and os.path.exists(obj)
                and os.path.getmtime(obj) > max(os.path.getmtime(src), newest_header)):
            return obj, subprocess.CompletedProcess([], 0, "", "")
        cmd = [nvcc(), *COMPILE_FLAGS, *inc, "-c", src, "-o", obj]
        return obj, subprocess.run(cmd, capture_output=True, text=True)

    srcs = sorted(sources(), key=lambda f: -os.path.getsize(f))  # longest first
    with ThreadPoolExecutor(max_workers=max(1, min(len(srcs), os.cpu_count() or 1))) as ex:
        results = list(ex.map(compile_one, srcs))
    for obj, proc in results:
        if proc.returncode != 0:
            sys.stderr.write(proc.stdout + proc.stderr)
            raise RuntimeError(f"nvcc failed building {os.path.basename(obj)}")
        if verbose:
            sys.stderr.write(proc.stderr)
    proc = subprocess.run([nvcc(), *LINK_FLAGS, *[o for o, _ in results], "-o", OUT + ".tmp"],
                          capture_output=True, text=True)
    if proc.returncode != 0:
        sys.stderr.write(proc.stdout + proc.stderr)
        raise RuntimeError("nvcc failed linking libpaste.so")
    os.replace(OUT + ".tmp", OUT)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
