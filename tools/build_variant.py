"""Build an A/B variant of liboptb_cuda.so with extra nvcc flags.

    python tools/build_variant.py NAME -DOPTB_X=1 [...]
    OPTB_CUDA_LIB=_ab/NAME.so python tools/cfg_ab.py C3_n18

Objects go to /tmp/optb_ab_NAME, the library to _ab/NAME.so (git-ignored,
shipped to the GPU box with the snapshot).
"""
import concurrent.futures as cf
import importlib.util
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    name, defs = sys.argv[1], sys.argv[2:]
    spec = importlib.util.spec_from_file_location("optb_build", os.path.join(ROOT, "paper_2105_00619_b200",
                                                                            "build.py"))
    b = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(b)
    objdir = f"/tmp/optb_ab_{name}"
    os.makedirs(objdir, exist_ok=True)
    os.makedirs(os.path.join(ROOT, "_ab"), exist_ok=True)
    jobs, objs = [], []
    for src in b.CUDA_SOURCES:
        o = os.path.join(objdir, src.replace(".cu", ".o"))
        objs.append(o)
        jobs.append([b.NVCC] + b.ARCH + b.NVCC_FLAGS + defs + ["-c", os.path.join(b.CSRC, src), "-o", o])
    with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        list(ex.map(b._run, jobs))
    out = os.path.join(ROOT, "_ab", name + ".so")
    b._run([b.NVCC] + b.ARCH + ["-shared", "-o", out] + objs + ["-cudart", "static"])
    print(out)


if __name__ == "__main__":
    main()
