"""The C-ABI library loads and exports every symbol include/fftpim.h declares
(no compute calls: this runs without a GPU)."""
import ctypes
import os
import re

import numpy as np
import pytest

from conftest import REPO
from paper_2312_02376_b200 import _native as nat

HEADER = os.path.join(REPO, "include", "fftpim.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"FFTPIM_API\s+[\w\s\*]+?\b(fftpim_\w+)\s*\(", text)))


def test_header_declares_expected_entry_points():
    assert set(declared_symbols()) == set(nat.EXPORTED)


def test_library_exports_every_declared_symbol():
    lib = nat.load()
    for name in declared_symbols():
        assert hasattr(lib, name), name


def test_struct_layout_matches_header(tmp_path):
    """ctypes mirrors == the C layout gcc computes from the header (a mismatch
    would silently corrupt every plan)."""
    import shutil
    import subprocess
    if not shutil.which("gcc"):
        pytest.skip("gcc not available")
    fields = [("FftpimProblem", nat.Problem), ("FftpimInfo", nat.Info), ("FftpimDirectReport", nat.DirectReport)]
    lines = ['#include <stdio.h>', '#include <stddef.h>', f'#include "{HEADER}"', "int main(void){"]
    for cname, cls in fields:
        lines.append(f'printf("%zu\\n", sizeof({cname}));')
        for f, _ in cls._fields_:
            lines.append(f'printf("%zu\\n", offsetof({cname}, {f}));')
    lines.append("return 0;}")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    subprocess.run(["gcc", str(src), "-o", str(tmp_path / "layout")], check=True)
    got = [int(v) for v in subprocess.run([str(tmp_path / "layout")], capture_output=True,
                                          text=True, check=True).stdout.split()]
    want = []
    for _, cls in fields:
        want.append(ctypes.sizeof(cls))
        want += [getattr(cls, f).offset for f, _ in cls._fields_]
    assert got == want


def test_missing_library_fails_loudly(tmp_path):
    saved = nat._lib
    try:
        nat._lib = None
        with pytest.raises(nat.NativeLibraryError):
            nat.load(str(tmp_path / "nope.so"))
    finally:
        nat._lib = saved


def test_sm100a_code_in_library():
    """The shipped .so carries sm_100a SASS (cuobjdump), not PTX-only or another arch."""
    import shutil
    import subprocess
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([exe, "--list-elf", nat.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
