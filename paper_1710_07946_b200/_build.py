"""Build liblra.so in-tree with nvcc for sm_100a (no JIT cache: the .so travels with the repo)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
SO = os.environ.get("LRA_BUILD_OUT") or os.path.join(HERE, "liblra.so")   # LRA_BUILD_OUT: diagnostic builds
SOURCES = ["lra_api.cu", "sketch.cu", "sketch_tc.cu", "ca.cu", "ca_cluster.cu", "ca_global.cu", "ca_small.cu", "nucleus.cu", "residual.cu", "residual_tc.cu", "shard.cu", "expand.cu", "qrp.cu", "leverage.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xptxas", "-v", "--expt-relaxed-constexpr"] + os.environ.get("LRA_EXTRA_FLAGS", "").split()


def _stale() -> bool:
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cu", ".cuh", ".h"))]
    deps.append(os.path.join(HERE, "..", "include", "lra.h"))
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return SO
    from concurrent.futures import ThreadPoolExecutor

    # LRA_KEEP_OBJ=1 (development): objects are kept under build/ and a translation unit is
    # recompiled only when it, or any header, is newer than its object
    keep = os.environ.get("LRA_KEEP_OBJ") == "1"
    odir = os.path.join(HERE, "..", "build", "obj" + os.environ.get("LRA_OBJ_TAG", "")) if keep else CSRC
    os.makedirs(odir, exist_ok=True)
    hdr = max([os.path.getmtime(os.path.join(CSRC, f)) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))] +
              [os.path.getmtime(os.path.join(HERE, "..", "include", "lra.h"))])

    def compile_one(src):
        obj = os.path.join(odir, src.replace(".cu", (os.environ.get("LRA_OBJ_TAG", "") + ".o")))
        if keep and os.path.exists(obj) and os.path.getmtime(obj) > max(hdr, os.path.getmtime(os.path.join(CSRC, src))):
            return src, obj, subprocess.CompletedProcess([], 0, "", "")
        cmd = [NVCC, *FLAGS, "-c", os.path.join(CSRC, src), "-o", obj]
        return src, obj, subprocess.run(cmd, capture_output=True, text=True)

    # translation units compile in parallel (the heavy templated ones dominate)
    with ThreadPoolExecutor(max_workers=max(1, min(len(SOURCES), os.cpu_count() or 1))) as ex:
        results = list(ex.map(compile_one, SOURCES))
    objs, logs = [], []
    for src, obj, p in results:
        logs.append(p.stderr)
        if p.returncode != 0:
            sys.stderr.write(p.stdout + p.stderr)
            raise RuntimeError(f"nvcc failed on {src}")
        objs.append(obj)
    tmp = SO + ".tmp"
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp, *objs]
    p = subprocess.run(cmd, capture_output=True, text=True)
    if p.returncode != 0:
        sys.stderr.write(p.stdout + p.stderr)
        raise RuntimeError("nvcc link failed")
    os.replace(tmp, SO)
    with open(os.path.join(CSRC, "ptxas.log"), "w") as f:
        f.write("\n".join(logs))
    if verbose:
        print("\n".join(logs))
    if not keep:
        for o in objs:
            os.remove(o)
    return SO


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
