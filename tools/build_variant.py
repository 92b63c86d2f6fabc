"""Build an experimental variant of libhrpb.so into .variants/NAME.so with extra nvcc -D flags.

usage: python tools/build_variant.py NAME [-DFOO=1 ...]      (tools/spmm_probe.py --lib .variants/NAME.so)
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2504_06443_b200 import _build  # noqa: E402

name, extra = sys.argv[1], sys.argv[2:]
os.makedirs(os.path.join(ROOT, ".variants"), exist_ok=True)
print(_build.compile_so(os.path.join(ROOT, ".variants", name + ".so"), extra))
