"""The C-ABI library loads and exports every symbol include/mgrit_b200.h declares
(no compute: this runs without a GPU); the package refuses to fall back to the CPU."""

import ctypes
import os
import re

import pytest

from paper_2209_06916_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "mgrit_b200.h")).read()
    return sorted(set(re.findall(r"\b(mgb_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_exported_list():
    assert sorted(_native.EXPORTED) == header_symbols()


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_native.lib_path())
    for name in header_symbols():
        assert hasattr(lib, name), name
    assert _native.load().mgb_version() >= 1


def test_struct_layouts_match_header():
    # field order/names of the ctypes mirrors follow the C structs
    text = open(os.path.join(ROOT, "include", "mgrit_b200.h")).read()
    for cls, cname in ((_native.StepDesc, "mgb_step_desc"), (_native.RelaxArgs, "mgb_relax_args")):
        body = text[:text.index("} " + cname + ";")]
        body = body[body.rindex("typedef struct {"):]
        fields = re.findall(r"\b(?:int32_t|int64_t|double)\s*\*?\s*(\w+)\s*;", body)
        assert [f[0] for f in cls._fields_] == fields, cname


def test_no_cpu_fallback_without_cuda():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import numpy as np
    import paper_2209_06916_b200 as P
    st = P.mol_stepper(P.DiscretizationSpec("erk", 1, 0.5, 64, 8))
    with pytest.raises(RuntimeError, match="CUDA"):
        st.apply(np.zeros(64))
