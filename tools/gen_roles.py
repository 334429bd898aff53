#!/usr/bin/env python3
"""Experiment: write ablib/roles_gen.cuh, the branch-parallel ABA warp roles
of tree29 (codegen.gen_aba_role), for tools/roles_sweep.cu."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2604_04310_b200 import _lib  # noqa: E402
from paper_2604_04310_b200 import codegen as cg  # noqa: E402

lib = _lib.load()
h = ctypes.c_void_p()
lib.vd_model_builtin(b"tree29", ctypes.byref(h))
rb = cg.Robot(cg.packed_model(lib, h), cg.frame_joints(lib, h))
text = "\n".join(["#pragma once", '#include "vd_gen_prelude.cuh"', "namespace vdk {"] + cg.emit_roles("Tree29", rb)
                 + ["}  // namespace vdk", ""])
os.makedirs(os.path.join(ROOT, "ablib"), exist_ok=True)
with open(os.path.join(ROOT, "ablib", "roles_gen.cuh"), "w") as f:
    f.write(text)
print("wrote ablib/roles_gen.cuh", len(text))
