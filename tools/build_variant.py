"""Build an experimental variant of libhrpb.so into .variants/NAME.so with extra nvcc -D flags.

usage: python tools/build_variant.py NAME [-DFOO=1 ...]      (tools/spmm_probe.py --lib .variants/NAME.so)
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2504_06443_b200 import _build  # noqa: E402

name, extra = sys.argv[1], sys.argv[2:]
os.makedirs(os.path.join(ROOT, ".variants"), exist_ok=True)
out = os.path.join(ROOT, ".variants", name + ".so")
flags = [f for f in _build.FLAGS if f not in ("-Xptxas", "-v")]
r = subprocess.run([_build.NVCC, *flags, *extra, "-o", out, *_build.SOURCES], cwd=_build.HERE,
                   capture_output=True, text=True)
if r.returncode:
    sys.exit(r.stderr)
print(out)
