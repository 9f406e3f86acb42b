"""Build libnmq.so in-tree with nvcc for sm_100a (no torch JIT cache).

Each translation unit compiles in parallel to an object file under build/,
then one nvcc call links the shared library.
"""

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libnmq.so")
OBJ = os.path.join(os.path.dirname(HERE), "build", "nmq")
SOURCES = ["nmq_kernels.cu", "nmq_fast.cu", "nmq_lod.cu", "nmq_train.cu", "nmq_kl.cu", "nmq_abi.cu",
           "nmq_multi.cu"]
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-lineinfo",
         "-Xcompiler", "-fPIC", "-Xptxas", "-v"]


def _compile(src, extra):
    obj = os.path.join(OBJ, os.path.basename(src) + ".o")
    cmd = [os.environ.get("NVCC", "nvcc"), *FLAGS, *extra, "-c", src, "-o", obj]
    res = subprocess.run(cmd, capture_output=True, text=True)
    return src, obj, res


def build(verbose=False, extra=()):
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    deps = srcs + [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [
        os.path.join(os.path.dirname(HERE), "include", "nmq.h")]
    newest = max(os.path.getmtime(p) for p in deps if os.path.exists(p))
    if (os.path.exists(OUT) and os.path.getmtime(OUT) >= newest and not extra
            and not os.environ.get("NMQ_REBUILD")):
        return OUT
    os.makedirs(OBJ, exist_ok=True)
    extra = list(extra) + os.environ.get("NMQ_NVCC_EXTRA", "").split()
    with ThreadPoolExecutor(max_workers=len(srcs)) as ex:
        results = list(ex.map(lambda s: _compile(s, extra), srcs))
    failed = [r for r in results if r[2].returncode != 0]
    for src, _, res in results:
        if verbose or res.returncode != 0:
            sys.stderr.write(res.stdout + res.stderr)
    if failed:
        raise RuntimeError("nvcc failed: " + ", ".join(os.path.basename(f[0]) for f in failed))
    cmd = [os.environ.get("NVCC", "nvcc"), "-gencode", "arch=compute_100a,code=sm_100a", "-shared",
           "-Xcompiler", "-fPIC", "-o", OUT + ".tmp", *[r[1] for r in results]]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed linking libnmq.so")
    os.replace(OUT + ".tmp", OUT)
    return OUT


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
