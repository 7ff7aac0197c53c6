"""In-tree build of the native libraries (nvcc, sm_100a only).

``libvbdr.so``  -- the product: C ABI (include/vbdr.h) + the hot-path kernels.
``synth/libsynth.so`` -- the CUDA twin of the shared input generator.

Built artefacts live in the source tree (git-ignored) so they travel to the GPU
box with the gpurun snapshot.
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "_lib")
LIBVBDR = os.path.join(LIBDIR, "libvbdr.so")
SYNTH_SRC = os.path.join(ROOT, "synth", "synth_gen.cu")
LIBSYNTH = os.path.join(ROOT, "synth", "libsynth.so")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
                 "-I", os.path.join(ROOT, "include")]

# (source, extra flags).  The estimate kernel is compiled without FMA
# contraction so its fp64 finish has the oracle's operation order (R#17).
SOURCES = [
    ("k_scan_slide.cu", []),
    ("k_estimate.cu", ["-fmad=false"]),
    ("k_plan.cu", ["-fmad=false"]),
    ("k_splan.cu", ["-fmad=false"]),
    ("vbdr_host.cu", []),
    ("vbdr_mc.cu", []),
]


def _newer(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd, log):
    r = subprocess.run(cmd, capture_output=True, text=True)
    with open(log, "a") as f:
        f.write(" ".join(cmd) + "\n" + r.stdout + r.stderr + "\n")
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"nvcc failed: {' '.join(cmd)}")


def build_vbdr(force: bool = False) -> str:
    os.makedirs(LIBDIR, exist_ok=True)
    deps = [os.path.join(CSRC, s) for s, _ in SOURCES] + [
        os.path.join(CSRC, "vbdr_dev.cuh"), os.path.join(ROOT, "include", "vbdr.h"), __file__]
    if not force and not _newer(LIBVBDR, deps):
        return LIBVBDR
    log = os.path.join(LIBDIR, "build.log")
    open(log, "w").close()
    objs = []
    for src, extra in SOURCES:
        obj = os.path.join(LIBDIR, src.replace(".cu", ".o"))
        _run([NVCC, *COMMON, *extra, "-c", os.path.join(CSRC, src), "-o", obj], log)
        objs.append(obj)
    tmp = LIBVBDR + f".tmp{os.getpid()}"
    _run([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs], log)
    os.replace(tmp, LIBVBDR)
    return LIBVBDR


def build_synth(force: bool = False) -> str:
    if not force and not _newer(LIBSYNTH, [SYNTH_SRC, __file__]):
        return LIBSYNTH
    log = os.path.join(os.path.dirname(LIBSYNTH), "build.log")
    open(log, "w").close()
    tmp = LIBSYNTH + f".tmp{os.getpid()}"
    _run([NVCC, *ARCH, "-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-shared", "-cudart", "static",
          "-o", tmp, SYNTH_SRC], log)
    os.replace(tmp, LIBSYNTH)
    return LIBSYNTH


def build_all(force: bool = False):
    return build_vbdr(force), build_synth(force)


if __name__ == "__main__":
    print(build_all(force="--force" in sys.argv))
