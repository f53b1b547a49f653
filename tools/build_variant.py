"""Build tuning variants of the library with different staged-kernel geometry.

    python tools/build_variant.py NAME DEFINE=VALUE ...
    GRKAN_LIB=tools/variants/NAME/libgrkan_b200.so python bench.py ...
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_13813_b200 import build  # noqa: E402

name, defines = sys.argv[1], tuple(sys.argv[2:])
out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "variants", name, "libgrkan_b200.so")
print(build.build(force=True, out=out, defines=defines, ptxas_v=True))
