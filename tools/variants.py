"""Build tuning variants of the native library side by side.

    python tools/variants.py NAME DEF=VAL [DEF=VAL ...]

writes variants/NAME/libppmlr_b200.so (git-ignored, travels with gpurun);
select one at run time with PPMLR_LIB=variants/NAME/libppmlr_b200.so.
"""
import importlib.util
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
spec = importlib.util.spec_from_file_location(
    "ppmlr_build", os.path.join(ROOT, "paper_1607_02214_b200", "build.py"))
build = importlib.util.module_from_spec(spec)
spec.loader.exec_module(build)

name, defs = sys.argv[1], sys.argv[2:]
d = os.path.join(ROOT, "variants", name)
os.makedirs(d, exist_ok=True)
print(build.build_native(defines=defs, out=os.path.join(d, "libppmlr_b200.so"),
                         objdir=os.path.join(d, "obj")))
