"""Host-side checks of the C-ABI boundary (no GPU needed): librs.so builds,
loads, and exports every entry point include/rs.h declares; the Python binding
declares exactly those; the product never links the oracle."""
import os
import re
import subprocess

import pytest

import paper_2508_01485_b200 as rsb
from paper_2508_01485_b200 import build as rsbuild

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(REPO, "include", "rs.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(rs_[a-z_0-9]+)\s*\(", src)))


def test_library_builds_and_exports_header_symbols():
    lib = rsbuild.build()
    out = subprocess.check_output(["nm", "-D", "--defined-only", lib]).decode()
    exported = set(re.findall(r" T (rs_[a-z_0-9]+)", out))
    want = header_symbols()
    assert want, "no declarations parsed"
    missing = [s for s in want if s not in exported]
    assert not missing, f"declared but not exported: {missing}"
    assert sorted(n for n, _, _ in rsb.SIGNATURES) == want


def test_library_loads_and_binds():
    lib = rsb.load_library()
    for name, _, _ in rsb.SIGNATURES:
        assert hasattr(lib, name)


def test_sm100a_code_only():
    lib = rsbuild.build()
    out = subprocess.check_output(["cuobjdump", "--list-elf", lib]).decode()
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_product_does_not_link_oracle():
    lib = rsbuild.build()
    out = subprocess.check_output(["nm", "-D", lib]).decode() + subprocess.check_output(["ldd", lib]).decode()
    assert "oracle" not in out
    # the package never imports the oracle module
    for root, _, files in os.walk(os.path.join(REPO, "paper_2508_01485_b200")):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(root, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "rsi_oracle" not in txt, f


def test_create_without_device_fails_cleanly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(rsb.RsError) as ei:
        rsb.rs_create(0)
    assert ei.value.status == rsb.RS_EINVAL
