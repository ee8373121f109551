"""Build an A/B variant of both libraries into variants/<tag>/ with extra
nvcc defines: python tools/build_variant.py <tag> -DSPH_X=0 [...]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2603_11868_b200 import build as b  # noqa: E402

tag, flags = sys.argv[1], sys.argv[2:]
out = os.path.join(ROOT, "variants", tag)
b.build_library(force=True, extra_flags=flags, out=os.path.join(out, "libsphb200.so"))
b.build_library(force=True, extra_flags=list(flags) + list(b.PERIODIC_FLAGS),
                out=os.path.join(out, "libsphb200_periodic.so"))
print(out)
