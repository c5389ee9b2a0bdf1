"""Build an experimental variant of libsrl.so with extra -D flags into variants/<name>/.

    python tools/build_variant.py <name> [DEFINE=VAL ...]
    SRL_LIB=variants/<name>/libsrl.so python bench.py ...
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_16688_b200 import build  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
name, defs = sys.argv[1], sys.argv[2:]
out = os.path.join(ROOT, "variants", name, "libsrl.so")
os.makedirs(os.path.dirname(out), exist_ok=True)
print(build.build(force=True, defines=defs, out=out))
