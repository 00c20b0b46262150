"""Builds libsk_b200.so (sm_100a) in-tree with nvcc.

Flags: -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 --fmad=false.
--fmad=false is part of the arithmetic contract: no implicit FMA contraction,
so the device results are bitwise identical to oracle/ (SKO_REPRODUCIBLE).
The kernels are instantiated per block size s in separate translation units
(compiled in parallel).
"""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
# SK_VARIANT=name SK_DEFS="-DX=1 ..." builds an experiment variant libsk_b200_<name>.so
VARIANT = os.environ.get("SK_VARIANT", "")
EXTRA_DEFS = os.environ.get("SK_DEFS", "").split()
LIB = os.path.join(HERE, f"libsk_b200_{VARIANT}.so" if VARIANT else "libsk_b200.so")
OBJ_SUFFIX = f"_{VARIANT}" if VARIANT else ""
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ARCH + ["-lineinfo", "-O3", "--fmad=false", "-std=c++17", "-Xcompiler", "-fPIC",
                "-Xcompiler", "-Wall", "--expt-relaxed-constexpr",
                "-I" + os.path.join(HERE, "..", "include")]
S_VALUES = range(1, 9)


def units():
    u = [("sk_kernels.cu", f"sk_kernels_s{s}.o", [f"-DSK_INST_S={s}"]) for s in S_VALUES]
    u.append(("sk_kernels.cu", "sk_kernels_common.o", ["-DSK_INST_COMMON"]))
    u.append(("sk_driver.cu", "sk_driver.o", []))
    u.append(("sk_residual.cu", "sk_residual.o", []))
    u.append(("sk_peak.cu", "sk_peak.o", []))
    u.append(("sk_problems.cpp", "sk_problems.o", []))
    u.append(("sk_comm.cpp", "sk_comm.o", []))
    u.append(("sk_export.cpp", "sk_export.o", []))
    return [(src, obj.replace(".o", OBJ_SUFFIX + ".o"), defs + EXTRA_DEFS) for src, obj, defs in u]


if EXTRA_DEFS and not VARIANT:
    raise RuntimeError("SK_DEFS builds an experiment variant: set SK_VARIANT=<name> too "
                       "(the default libsk_b200.so is only built from the default flags)")


def _flags_stamp() -> str:
    import hashlib
    return hashlib.sha256(" ".join(FLAGS + EXTRA_DEFS + [NVCC]).encode()).hexdigest()[:16]


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    try:  # the flags a library was built with are stamped next to it
        if open(LIB + ".flags").read().strip() != _flags_stamp():
            return True
    except OSError:
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if not f.endswith(".o")]
    deps.append(os.path.join(HERE, "..", "include", "sylkrylov_b200.h"))
    deps.append(os.path.abspath(__file__))
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(unit, verbose):
    src, obj, defs = unit
    if src.endswith(".cpp"):
        cmd = ["g++", "-O3", "-std=c++17", "-fPIC", "-Wall", "-ffp-contract=off", "-pthread",
               "-I/usr/local/cuda/include", "-I" + os.path.join(HERE, "..", "include"), *defs,
               "-c", os.path.join(CSRC, src), "-o", os.path.join(CSRC, obj)]
    else:
        cmd = [NVCC, *FLAGS, *defs, "-c", os.path.join(CSRC, src), "-o", os.path.join(CSRC, obj)]
    if verbose and not src.endswith(".cpp"):
        cmd.insert(1, "-Xptxas=-v")
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {obj}:\n{r.stderr}")
    return r.stderr


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return LIB
    us = units()
    with ThreadPoolExecutor(max_workers=min(len(us), os.cpu_count() or 4)) as ex:
        logs = list(ex.map(lambda u: _compile(u, verbose), us))
    if verbose:
        for lg in logs:
            sys.stderr.write(lg)
    objs = [os.path.join(CSRC, u[1]) for u in us]
    subprocess.check_call([NVCC, "-shared", *ARCH, *objs, "-o", LIB + ".tmp", "-lcudart", "-lcublas", "-lcusolver",
                           "-Xcompiler", "-pthread", "-ldl"])
    os.replace(LIB + ".tmp", LIB)
    with open(LIB + ".flags", "w") as f:
        f.write(_flags_stamp() + "\n")
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
