#!/usr/bin/env python
"""Build A/B variants of libgk.so: python tools/ab_build.py NAME DEFINE [DEFINE ...]
-> paper_2103_14978_b200/libgk_NAME.so (use with GK_LIB=...)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2103_14978_b200 import _build  # noqa: E402

name, defines = sys.argv[1], sys.argv[2:]
print(_build.build(defines=defines, out=os.path.join(_build.HERE, f"libgk_{name}.so")))
