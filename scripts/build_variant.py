"""Tuning A/B helper: build librgb.so from a csrc snapshot into another directory.

  python scripts/build_variant.py OUT_DIR [GIT_REV] [-D...]
GIT_REV (default: the working tree) selects the csrc/ and include/ to compile;
extra -D flags are passed to nvcc.  Point RGB_LIB_PATH at OUT_DIR/librgb.so.
"""
import os
import subprocess
import sys
import tempfile
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2106_11594_b200 import _build  # noqa: E402

out = os.path.abspath(sys.argv[1])
rest = sys.argv[2:]
rev = rest.pop(0) if rest and not rest[0].startswith("-") else None
defs = rest
os.makedirs(out, exist_ok=True)
src_root = _build.ROOT
if rev:
    tmp = tempfile.mkdtemp()
    subprocess.run(f"git archive {rev} paper_2106_11594_b200/csrc include | tar -x -C {tmp}", shell=True,
                   check=True, cwd=_build.ROOT)
    src_root = tmp
csrc = os.path.join(src_root, "paper_2106_11594_b200", "csrc")
srcs = sorted(os.path.join(csrc, f) for f in os.listdir(csrc) if f.endswith(".cu"))
nvcc = "/usr/local/cuda/bin/nvcc"
flags = [f for f in _build.COMPILE_FLAGS if f not in ("-Xptxas", "-v")]


def cc(src):
    obj = os.path.join(out, os.path.basename(src)[:-3] + ".o")
    subprocess.run([nvcc, *flags, *defs, "-I" + os.path.join(src_root, "include"), "-c", "-o", obj, src],
                   check=True)
    return obj


with ThreadPoolExecutor(len(srcs)) as pool:
    objs = list(pool.map(cc, srcs))
subprocess.run([nvcc, *_build.ARCH_FLAGS, "-shared", "-o", os.path.join(out, "librgb.so"), *objs], check=True)
print(os.path.join(out, "librgb.so"))
