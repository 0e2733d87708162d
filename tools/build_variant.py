"""Build a variant of liblora_server.so with extra nvcc defines for A/B runs.

    python tools/build_variant.py NAME [-DFOO=1 ...]   -> tools/ab/lib_NAME.so
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2604_07173_b200 import build as b  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
b.OBJ = os.path.join(ROOT, "tools", "ab", "_obj_" + name)
b.OUT = os.path.join(ROOT, "tools", "ab", "lib_" + name + ".so")
b.FLAGS = b.FLAGS + defs
print(b.build(force=True))
