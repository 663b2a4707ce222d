"""Build a compile-time variant of libfdsdf.so for A/B timing on the GPU box.
usage: python scripts/build_variant.py NAME -DMACRO=V ...
-> paper_2511_08980_b200/variants/libfdsdf_NAME.so (load it with FDSDF_LIB=<path>)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
name, flags = sys.argv[1], sys.argv[2:]
from paper_2511_08980_b200 import _build  # noqa: E402

_build.EXTRA = _build.EXTRA + flags
out = os.path.join(_build.PKG, "variants", f"libfdsdf_{name}.so")
os.makedirs(os.path.dirname(out), exist_ok=True)
print(_build.build(force=True, lib=out, build_dir=os.path.join(_build.ROOT, "build", "var_" + name)))
