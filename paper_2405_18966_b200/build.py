"""Build libsvdsc.so in-tree with nvcc for sm_100a (no JIT, no torch extension).

    python -m paper_2405_18966_b200.build
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libsvdsc.so")
SOURCES = ["svdsc.cu", "comm.cu", "matvec.cu", "cgs.cu", "cgs_fused.cu", "svd.cu", "pro.cu", "paper_api.cpp"]
CLI = os.path.join(HERE, "svdsc-cli")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden", "-cudart", "static",
         "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills"]


def stale() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps += [os.path.join(HERE, "..", "include", f) for f in ("svdsc.h", "svdsc_paper.h")]
    if not os.path.exists(CLI):
        return True
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not stale():
        return OUT
    objs = []
    os.makedirs(os.path.join(HERE, "build"), exist_ok=True)
    procs = []
    for src in SOURCES:
        obj = os.path.join(HERE, "build", os.path.splitext(src)[0] + ".o")
        cmd = [NVCC, *FLAGS, "-dc" if False else "-c", os.path.join(CSRC, src), "-o", obj]
        if verbose:
            cmd += ["-Xptxas", "-v"]
        procs.append((subprocess.Popen(cmd), cmd))
        objs.append(obj)
    for p, cmd in procs:
        if p.wait() != 0:
            raise RuntimeError("nvcc failed: " + " ".join(cmd))
    link = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-cudart", "static",
            "-o", OUT, *objs, "-ldl", "-lpthread", "-Xlinker", "--no-undefined"]
    subprocess.check_call(link)
    # batch CLI (host C++ over the C ABI), rpath to the in-tree library
    subprocess.check_call(["g++", "-O2", "-std=c++17", os.path.join(CSRC, "cli.cpp"), "-o", CLI,
                           "-L" + HERE, "-lsvdsc", "-Wl,-rpath,$ORIGIN"])
    return OUT


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(OUT)
