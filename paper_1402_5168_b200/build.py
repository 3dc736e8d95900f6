"""Build librexp.so in-tree (sm_100a).  Used by __graft_entry__.build().

nvcc compiles the CUDA hot path for sm_100a only; the host C++ (rational
approximation, mesh/tree, factorization, C ABI) is compiled by g++.
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "librexp.so")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA, "bin", "nvcc")

CU = ["device.cu", "cgemm_sym.cu", "fused_tree.cu"]
CPP = ["rational.cpp", "mesh.cpp", "setup_host.cpp", "eig.cpp", "api.cpp"]
GENCODE = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _run(cmd):
    print(" ".join(cmd[:2] + ["..."] + cmd[-3:]), flush=True)
    subprocess.check_call(cmd)


def build(force=False, verbose_ptxas=False, variant=None):
    """Compile every translation unit (in parallel) and link librexp.so.
    variant="cmul4": an experiment build (librexp_cmul4.so, four real DMMAs per
    complex k-step instead of the three-multiply form) loaded with REXP_LIB."""
    import concurrent.futures as cf
    BUILD, LIB = globals()["BUILD"], globals()["LIB"]
    extra = []
    if variant == "cmul4":
        BUILD, LIB, extra = BUILD + "_cmul4", os.path.join(HERE, "librexp_cmul4.so"), ["-DREXP_CMUL3=0"]
    os.makedirs(BUILD, exist_ok=True)
    srcs = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    srcs.append(os.path.join(os.path.dirname(HERE), "include", "rexp.h"))
    srcs.append(os.path.abspath(__file__))     # compile flags live here
    if not force and os.path.exists(LIB):
        t = os.path.getmtime(LIB)
        if all(os.path.getmtime(s) <= t for s in srcs):
            return LIB
    jobs = []
    for f in CU:
        o = os.path.join(BUILD, f + ".o")
        cmd = [NVCC, *GENCODE, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", *extra, "-c",
               os.path.join(CSRC, f), "-o", o]
        if verbose_ptxas:
            cmd.insert(1, "-Xptxas=-v")
        jobs.append((cmd, o))
    for mode in range(6):   # k_cgemm tile instantiations, one object per mode
        o = os.path.join(BUILD, f"cgemm_mode{mode}.o")
        jobs.append(([NVCC, *GENCODE, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", *extra, f"-DCG_MODE={mode}",
                      "-c", os.path.join(CSRC, "cgemm_mode.cu"), "-o", o], o))
    for f in CPP:
        o = os.path.join(BUILD, f + ".o")
        jobs.append((["g++", "-O3", "-mavx2", "-mfma", "-std=c++17", "-fPIC", "-Wall", "-I",
                      os.path.join(CUDA, "include"), "-c", os.path.join(CSRC, f), "-o", o], o))
    with cf.ThreadPoolExecutor(max_workers=max(1, os.cpu_count() or 1)) as ex:
        futs = [ex.submit(_run, cmd) for cmd, _ in jobs]
        for fu in futs:
            fu.result()
    objs = [o for _, o in jobs]
    _run([NVCC, *GENCODE, "-shared", "-cudart", "static", "-o", LIB, *objs, "-lpthread"])
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose_ptxas="-v" in sys.argv,
          variant="cmul4" if "--cmul4" in sys.argv else None)
