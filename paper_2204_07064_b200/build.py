"""Build the sm_100a engine library in-tree: paper_2204_07064_b200/lib/libstreamconv_b200.so.

nvcc cross-compiles for sm_100a without a GPU.  Every CUDA/C++ source under csrc/ is
compiled with -gencode arch=compute_100a,code=sm_100a -lineinfo and linked into one shared
library exposing the C-ABI of include/streamconv_b200.h.  Incremental: a source is rebuilt
only when it or a header is newer than its object.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OBJ = PKG / "build"
LIB = PKG / "lib" / "libstreamconv_b200.so"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-fvisibility=hidden",
          "-I", str(ROOT / "include"), "-ccbin", "/usr/bin/g++"]
CUFLAGS = ARCH + ["--expt-relaxed-constexpr"] + (["-Xptxas", "-v"] if os.environ.get("SC_PTXAS_V") else [])


def _sources():
    return sorted(list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cpp")))


def _headers_mtime():
    hs = list(CSRC.glob("*.hpp")) + list(CSRC.glob("*.cuh")) + list((ROOT / "include").glob("*.h"))
    return max((h.stat().st_mtime for h in hs), default=0)


def _compile(src: Path, hdr_mtime: float, verbose: bool) -> Path:
    obj = OBJ / (src.name + ".o")
    if obj.exists() and obj.stat().st_mtime >= max(src.stat().st_mtime, hdr_mtime):
        return obj
    cmd = [NVCC] + COMMON + (CUFLAGS if src.suffix == ".cu" else ARCH) + ["-c", str(src), "-o", str(obj)]
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src.name}:\n{r.stdout}\n{r.stderr}")
    if r.stderr.strip() and verbose:
        print(r.stderr, file=sys.stderr)
    return obj


def build(verbose: bool = False) -> Path:
    OBJ.mkdir(exist_ok=True)
    LIB.parent.mkdir(exist_ok=True)
    hm = _headers_mtime()
    srcs = _sources()
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(lambda s: _compile(s, hm, verbose), srcs))
    if not LIB.exists() or LIB.stat().st_mtime < max(o.stat().st_mtime for o in objs):
        cmd = [NVCC] + ARCH + ["-shared", "-o", str(LIB)] + [str(o) for o in objs] + ["-lcuda", "-lcufft"]
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return LIB


CPP_TEST = ROOT / "tests" / "cpp" / "test_modules.cpp"
CPP_BIN = OBJ / "test_modules"


def build_cpp_tests(verbose: bool = False) -> Path:
    """The C++ cached-module API test (include/streamconv_b200.hpp), linked to the library."""
    if CPP_BIN.exists() and CPP_BIN.stat().st_mtime >= max(CPP_TEST.stat().st_mtime, LIB.stat().st_mtime,
                                                            _headers_mtime()):
        return CPP_BIN
    cmd = ["/usr/bin/g++", "-std=c++17", "-O2", "-I", str(ROOT / "include"), "-I", "/usr/local/cuda/include",
           str(CPP_TEST), "-o", str(CPP_BIN), "-L", str(LIB.parent), "-lstreamconv_b200",
           "-L", "/usr/local/cuda/lib64", "-lcudart", "-Wl,-rpath,$ORIGIN/../lib", "-Wl,-rpath,/usr/local/cuda/lib64"]
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"C++ test build failed:\n{r.stdout}\n{r.stderr}")
    return CPP_BIN


def build_oracle(verbose: bool = False) -> None:
    """Test infrastructure: oracle/build/liboracle.so and (when /root/reference exists)
    oracle/_ref/libref_streamconv.so.  Never linked into the library above."""
    r = subprocess.run(["make", "-C", str(ROOT / "oracle")], capture_output=True, text=True)
    if verbose:
        print(r.stdout, r.stderr)
    if r.returncode != 0:
        raise RuntimeError(f"oracle build failed:\n{r.stdout}\n{r.stderr}")


if __name__ == "__main__":
    print(build(verbose=True))
    build_cpp_tests(verbose=True)
    build_oracle(verbose=True)
