"""Build libvbdr.so variants with extra nvcc defines into tools/var_build/<name>/
(for kernel A/B experiments: VBDR_LIB=tools/var_build/<name>/libvbdr.so)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1810_13132_b200 import _build  # noqa: E402


def build(name, defines):
    out = os.path.join(ROOT, "tools", "var_build", name)
    os.makedirs(out, exist_ok=True)
    objs = []
    for src, extra in _build.SOURCES:
        obj = os.path.join(out, src.replace(".cu", ".o"))
        subprocess.check_call([_build.NVCC, *_build.COMMON, *extra, *[f"-D{d}" for d in defines],
                               "-c", os.path.join(_build.CSRC, src), "-o", obj],
                              stdout=subprocess.DEVNULL)
        objs.append(obj)
    lib = os.path.join(out, "libvbdr.so")
    subprocess.check_call([_build.NVCC, *_build.ARCH, "-shared", "-cudart", "static", "-o", lib, *objs])
    return lib


if __name__ == "__main__":
    # usage: build_variant.py name DEF=1 DEF2=0 ...
    print(build(sys.argv[1], sys.argv[2:]))
