"""Build recipe for the native libraries (in-tree, sm_100a only).

    liboptb_cuda.so  csrc/{codec,sbs,capi}.cu -> the C ABI of include/optb_cuda.h
    liboptb_shim.so  csrc/shim/src/*.cpp       -> the reference's C++ API
                     (optb::codec / optb::sampler / optb::Rng / decode_input)
                     re-implemented over liboptb_cuda.so

Called by __graft_entry__.build(); also runnable as
``python paper_2105_00619_b200/build.py``.  Objects go to build/, the shared
libraries next to this file so they travel with the repo snapshot.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
BUILD = os.path.join(ROOT, "build")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
CUDA_LIB = "/usr/local/cuda/lib64"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
              "--expt-relaxed-constexpr", "-diag-suppress", "177", "-I" + INCLUDE]
CUDA_SOURCES = ["codec.cu"] + [f"codec_v{v}.cu" for v in range(6)] + ["sbs.cu", "capi.cu", "pipeline.cu", "io.cu",
                                                                      "peer.cu"]
CUDA_LIB_NAME = os.path.join(PKG, "liboptb_cuda.so")
SHIM_LIB_NAME = os.path.join(PKG, "liboptb_shim.so")
SHIM_SOURCES = ["codec.cpp", "sampler.cpp", "nn.cpp", "pipeline.cpp", "metering.cpp"]


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("build failed: " + " ".join(cmd) + "\n" + r.stdout + r.stderr)
    return r.stdout + r.stderr


def _stale(target, sources):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def build_cuda(force: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    headers = [os.path.join(CSRC, "internal.h"), os.path.join(CSRC, "codec_impl.cuh"),
               os.path.join(INCLUDE, "optb_cuda.h")]
    objs = []
    jobs = []
    for src in CUDA_SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src.replace(".cu", ".o"))
        objs.append(o)
        if force or _stale(o, [s] + headers):
            jobs.append([NVCC] + ARCH + NVCC_FLAGS + ["-c", s, "-o", o])
    with cf.ThreadPoolExecutor(max_workers=min(len(CUDA_SOURCES), os.cpu_count() or 4)) as ex:
        list(ex.map(_run, jobs))
    if force or _stale(CUDA_LIB_NAME, objs):
        _run([NVCC] + ARCH + ["-shared", "-o", CUDA_LIB_NAME] + objs + ["-cudart", "static"])
    return CUDA_LIB_NAME


def build_shim(force: bool = False) -> str:
    inc = os.path.join(CSRC, "shim", "include")
    srcs = [os.path.join(CSRC, "shim", "src", f) for f in SHIM_SOURCES]
    hdrs = [os.path.join(inc, "optb", h) for h in os.listdir(os.path.join(inc, "optb"))]
    if force or _stale(SHIM_LIB_NAME, srcs + hdrs + [CUDA_LIB_NAME]):
        _run(["g++", "-std=c++20", "-O2", "-fPIC", "-shared", "-Wall", "-Wextra", "-pthread", "-I" + inc,
              "-I" + INCLUDE] + srcs + ["-o", SHIM_LIB_NAME, "-L" + PKG, "-loptb_cuda",
                                        "-Wl,-rpath,$ORIGIN"])
    return SHIM_LIB_NAME


REF_TESTS = "/root/reference/proj/tests"
REF_SUITES = ["test_codec.cpp", "test_sampler.cpp", "test_pipeline.cpp"]
REF_SUITES_BIN = os.path.join(ROOT, "tests", "cpp", "_bin", "ref_suites_on_b200")


def build_ref_suites(force: bool = False):
    """Compile the REFERENCE's own unit suites (test_codec.cpp,
    test_sampler.cpp and its doctest_main.cpp), in place from
    /root/reference, against the drop-in shim headers + libraries -- the
    drop-in proof.  Uses tests/cpp/doctest.h (written for this repo) since
    the reference's vendor/doctest.h is not shipped.  Only where the
    reference exists; the binary travels to the GPU box like the .so files."""
    if not os.path.isdir(REF_TESTS):
        return None
    srcs = [os.path.join(REF_TESTS, f) for f in REF_SUITES + ["doctest_main.cpp"]]
    if not force and not _stale(REF_SUITES_BIN, srcs + [SHIM_LIB_NAME, CUDA_LIB_NAME]):
        return REF_SUITES_BIN
    os.makedirs(os.path.dirname(REF_SUITES_BIN), exist_ok=True)
    _run(["g++", "-std=c++20", "-O2", "-w", "-pthread", "-I" + os.path.join(ROOT, "tests", "cpp"),
          "-I" + os.path.join(CSRC, "shim", "include"), "-I" + INCLUDE, "-I" + REF_TESTS] + srcs +
         ["-o", REF_SUITES_BIN, "-L" + PKG, "-loptb_shim", "-loptb_cuda", "-Wl,-rpath," + PKG,
          "-Wl,-rpath,$ORIGIN/../../../paper_2105_00619_b200"])
    return REF_SUITES_BIN


CLI_SRC = os.path.join(ROOT, "tools", "optb_cli.cpp")
CLI_BIN = os.path.join(PKG, "optb_b200")


def build_cli(force: bool = False) -> str:
    """The reference CLI's encode/decode subcommands over the shim."""
    if force or _stale(CLI_BIN, [CLI_SRC, SHIM_LIB_NAME]):
        _run(["g++", "-std=c++20", "-O2", "-Wall", "-I" + os.path.join(CSRC, "shim", "include"), CLI_SRC,
              "-o", CLI_BIN, "-L" + PKG, "-loptb_shim", "-loptb_cuda", "-Wl,-rpath,$ORIGIN"])
    return CLI_BIN


API_BENCH_SRC = os.path.join(ROOT, "tools", "shim_api_bench.cpp")
API_BENCH_BIN = os.path.join(PKG, "optb_shim_api_bench")


def build_api_bench(force: bool = False) -> str:
    """The reference runner's call pattern over the drop-in shim (bench.py shim_api)."""
    if force or _stale(API_BENCH_BIN, [API_BENCH_SRC, SHIM_LIB_NAME]):
        _run(["g++", "-std=c++20", "-O3", "-Wall", "-I" + os.path.join(CSRC, "shim", "include"), API_BENCH_SRC,
              "-o", API_BENCH_BIN, "-L" + PKG, "-loptb_shim", "-loptb_cuda", "-Wl,-rpath,$ORIGIN"])
    return API_BENCH_BIN


SHIM_TESTS_SRC = os.path.join(ROOT, "tests", "cpp", "shim_extra.cpp")
SHIM_TESTS_BIN = os.path.join(ROOT, "tests", "cpp", "_bin", "shim_extra")


def build_shim_tests(force: bool = False) -> str:
    """tests/cpp/shim_extra.cpp (cursor copies, acceptance criteria 1/6/8,
    the GPU pipeline) against the shim; needs no reference sources."""
    if force or _stale(SHIM_TESTS_BIN, [SHIM_TESTS_SRC, SHIM_LIB_NAME, CUDA_LIB_NAME]):
        os.makedirs(os.path.dirname(SHIM_TESTS_BIN), exist_ok=True)
        _run(["g++", "-std=c++20", "-O2", "-w", "-pthread", "-I" + os.path.join(ROOT, "tests", "cpp"),
              "-I" + os.path.join(CSRC, "shim", "include"), SHIM_TESTS_SRC, "-o", SHIM_TESTS_BIN, "-L" + PKG,
              "-loptb_shim", "-loptb_cuda", "-Wl,-rpath,$ORIGIN/../../../paper_2105_00619_b200"])
    return SHIM_TESTS_BIN


def build(force: bool = False) -> None:
    build_cuda(force)
    if os.path.isdir(os.path.join(CSRC, "shim", "src")) and all(
            os.path.exists(os.path.join(CSRC, "shim", "src", f)) for f in SHIM_SOURCES):
        build_shim(force)
        build_cli(force)
        build_api_bench(force)
        build_shim_tests(force)
        build_ref_suites(force)


if __name__ == "__main__":
    build(force="--force" in sys.argv)
    print("built", CUDA_LIB_NAME)
