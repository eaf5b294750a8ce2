"""In-tree build of libstk.so for sm_100a (nvcc cross-compiles without a GPU)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libstk.so")

SOURCES = ["stk_kernels.cu", "stk_capi.cu"]
CXX_SOURCES = ["stripley_api.cpp"]
HEADERS = ["stk_device.cuh", "stk_kernels.h", "stk_types.h"]

# -fmad=false: no FP64 mul+add contraction (the reference's Release build has
# none; bit-exact distances and bins depend on it).  -prec-sqrt/-prec-div only
# affect FP32 (the approximate bucket guess), never the FP64 path.
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-fmad=false", "-prec-sqrt=false", "-prec-div=false",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
]


def source_hash() -> str:
    """Hash of everything libstk.so is built from (sources, headers, flags): the
    stamp that ties a committed ncu capture to the build it profiled."""
    import hashlib

    h = hashlib.sha256()
    for f in SOURCES + HEADERS + CXX_SOURCES:
        with open(os.path.join(CSRC, f), "rb") as fh:
            h.update(f.encode() + b"\0" + fh.read())
    for f in ("stk.h", "stripley_gpu.hpp"):
        with open(os.path.join(ROOT, "include", f), "rb") as fh:
            h.update(f.encode() + b"\0" + fh.read())
    h.update(" ".join(NVCC_FLAGS).encode())
    return h.hexdigest()[:16]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    return "nvcc"


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS + CXX_SOURCES]
    deps.append(os.path.join(ROOT, "include", "stripley_gpu.hpp"))
    deps.append(os.path.join(ROOT, "include", "stk.h"))
    deps.append(os.path.abspath(__file__))
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build_library(force: bool = False, verbose: bool = False, extra=(), out=None) -> str:
    lib = out or LIB
    if not force and not extra and out is None and not _stale():
        return LIB
    nvcc = _nvcc()
    objs = []
    procs = []
    for src in SOURCES:
        obj = os.path.join(CSRC, src.replace(".cu", ".o"))
        obj = obj.replace(".o", ".%d.o" % os.getpid()) if out else obj
        cmd = [nvcc, *NVCC_FLAGS, *extra, "-c", os.path.join(CSRC, src), "-o", obj]
        if verbose:
            cmd += ["-Xptxas", "-v"]
            print(" ".join(cmd), file=sys.stderr)
        procs.append(subprocess.Popen(cmd))
        objs.append(obj)
    for src in CXX_SOURCES:
        obj = os.path.join(CSRC, src.replace(".cpp", ".o"))
        obj = obj.replace(".o", ".%d.o" % os.getpid()) if out else obj
        procs.append(subprocess.Popen(["g++", "-std=c++20", "-O2", "-fPIC", "-c",
                                       os.path.join(CSRC, src), "-o", obj]))
        objs.append(obj)
    for p in procs:
        if p.wait() != 0:
            raise RuntimeError("compiler failed building libstk.so")
    tmp = lib + ".tmp"
    link = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp, *objs]
    subprocess.run(link, check=True)
    os.replace(tmp, lib)
    for o in objs:
        try:
            os.remove(o)
        except OSError:
            pass
    return lib


TEST_BIN = os.path.join(ROOT, "tests", "cpp", "test_api")


def build_cpp_tests(force: bool = False) -> str:
    """The C++ API test program (tests/cpp/test_api.cpp), linked to libstk.so."""
    src = os.path.join(ROOT, "tests", "cpp", "test_api.cpp")
    if not force and os.path.exists(TEST_BIN) and os.path.getmtime(TEST_BIN) > max(
            os.path.getmtime(src), os.path.getmtime(LIB)):
        return TEST_BIN
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"), src, "-o",
                    TEST_BIN, "-L", HERE, "-lstk", "-Wl,-rpath," + HERE], check=True)
    return TEST_BIN


REFPROG_BIN = os.path.join(ROOT, "tests", "cpp", "reference_program")


def build_reference_program(force: bool = False) -> str:
    """tests/cpp/reference_program.cpp: a program written against the reference's
    runtime.hpp, compiled unchanged against include/stripley/ (the drop-in path)."""
    src = os.path.join(ROOT, "tests", "cpp", "reference_program.cpp")
    hdr = os.path.join(ROOT, "include", "stripley_gpu.hpp")
    if not force and os.path.exists(REFPROG_BIN) and os.path.getmtime(REFPROG_BIN) > max(
            os.path.getmtime(src), os.path.getmtime(LIB), os.path.getmtime(hdr)):
        return REFPROG_BIN
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"), src, "-o",
                    REFPROG_BIN, "-L", HERE, "-lstk", "-Wl,-rpath," + HERE], check=True)
    return REFPROG_BIN


CLI_BIN = os.path.join(HERE, "stripley_gpu")
CLI_SOURCES = ["stripley_cli.cpp", "stripley_io.cpp"]


def nlohmann_include():
    """Directory holding nlohmann/json.hpp (the JSON header the reference's
    io.cpp uses; this image ships it in cudnn_frontend's third-party tree)."""
    import site
    import sysconfig

    roots = {sysconfig.get_paths()["purelib"], *site.getsitepackages()}
    for root in sorted(roots):
        for sub in ("include/cudnn_frontend/thirdparty", "include"):
            d = os.path.join(root, sub)
            if os.path.exists(os.path.join(d, "nlohmann", "json.hpp")):
                return d
    for d in ("/usr/include", "/usr/local/include"):
        if os.path.exists(os.path.join(d, "nlohmann", "json.hpp")):
            return d
    return None


def build_cli(force: bool = False) -> str | None:
    """The `stripley_gpu run` CLI (csrc/stripley_cli.cpp + stripley_io.cpp), linked
    to libstk.so; None when no nlohmann/json.hpp is available."""
    srcs = [os.path.join(CSRC, f) for f in CLI_SOURCES]
    hdrs = [os.path.join(ROOT, "include", h) for h in ("stripley_gpu.hpp", "stripley_gpu_io.hpp")]
    if not force and os.path.exists(CLI_BIN) and os.path.getmtime(CLI_BIN) > max(
            os.path.getmtime(f) for f in srcs + hdrs + [LIB]):
        return CLI_BIN
    inc = nlohmann_include()
    if inc is None:
        print("warning: nlohmann/json.hpp not found; stripley_gpu CLI not built", file=sys.stderr)
        return None
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"), "-isystem",
                    inc, *srcs, "-o", CLI_BIN, "-L", HERE, "-lstk", "-Wl,-rpath," + HERE],
                   check=True)
    return CLI_BIN


if __name__ == "__main__":
    print(build_library(force="--force" in sys.argv, verbose="-v" in sys.argv))
