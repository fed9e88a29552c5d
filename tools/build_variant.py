"""Build libgspn.so with extra nvcc flags into build_ab/ (A/B tooling; loaded with GSPN_EXPERIMENTS=1
GSPN_LIB=<path>). Usage: python tools/build_variant.py NAME -DFLAG ..."""
import glob
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_07884_b200 import build as b  # noqa: E402

name, flags = sys.argv[1], sys.argv[2:]
srcs = sorted(glob.glob(os.path.join(b.CSRC, "*.cu")))
out = os.path.join(b.ROOT, "build_ab", f"libgspn_{name}.so")
b._nvcc(srcs, out, ["-I" + os.path.join(b.ROOT, "include"), *flags], False, srcs)
print(out)
