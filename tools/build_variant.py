"""Build an A/B variant of libesp_b200.so with extra nvcc defines.

    python tools/build_variant.py <tag> -DNAME=VALUE ...

Writes tools/bin/libesp_<tag>.so (travels to the GPU box with gpurun; load
it with ESP_LIB=tools/bin/libesp_<tag>.so)."""
import concurrent.futures as cf
import glob
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
from paper_2601_00161_b200 import _build  # noqa: E402

tag, defines = sys.argv[1], sys.argv[2:]
out = os.path.join(REPO, "tools", "bin", f"libesp_{tag}.so")
bdir = os.path.join(REPO, "tools", "bin", f"build_{tag}")
os.makedirs(bdir, exist_ok=True)
srcs = sorted(glob.glob(os.path.join(_build.CSRC, "*.cu")))


def comp(src):
    obj = os.path.join(bdir, os.path.basename(src).replace(".cu", ".o"))
    r = subprocess.run([_build.nvcc(), "-c", src, "-o", obj] + _build._flags() + defines,
                       capture_output=True, text=True)
    if r.returncode:
        raise RuntimeError(r.stderr)
    return obj


with cf.ThreadPoolExecutor(8) as ex:
    objs = list(ex.map(comp, srcs))
libdir = _build.cufft_libdir()
r = subprocess.run([_build.nvcc(), "-shared", "-o", out] + objs + _build.ARCH + [
    "-L", libdir, "-l:libcufft.so.11", "-Xlinker", f"-rpath,{libdir}",
    "-Xlinker", "-rpath,/usr/local/cuda/lib64"], capture_output=True, text=True)
if r.returncode:
    raise RuntimeError(r.stderr)
print(out)
