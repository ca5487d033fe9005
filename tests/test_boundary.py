"""The C-ABI boundary: libdffm.so loads, exports every symbol include/dffm.h
declares, and the ctypes structs match the C layout (CPU only, no compute)."""

import ctypes
import os
import re
import subprocess

import pytest

from paper_2407_10115_b200 import _lib

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(REPO, "include", "dffm.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w\s\*]+?\b(\w+)\s*\(", text, flags=re.M))
                  - {"defined"})


def test_library_exports_every_declared_symbol():
    lib = _lib.lib()
    names = declared_functions()
    assert "dffm_forward" in names and "fwq_quantize" in names
    for n in names:
        assert hasattr(lib, n), f"libdffm.so does not export {n}"
    assert set(names) == set(_lib.SIGNATURES), "ctypes bindings drifted from include/dffm.h"
    assert lib.dffm_abi_version() == 1


def test_struct_layout_matches_c(tmp_path):
    src = tmp_path / "lay.c"
    src.write_text(
        '#include <stdio.h>\n#include <stddef.h>\n#include "dffm.h"\n'
        "int main(){printf(\"%zu %zu %zu %zu %zu %zu\\n\", sizeof(dffm_model),"
        " offsetof(dffm_model, lr), offsetof(dffm_model, q_ffm_bucket), sizeof(dffm_train_state),"
        " offsetof(dffm_train_state, lr_ffm), offsetof(dffm_train_state, sparse));return 0;}\n")
    exe = tmp_path / "lay"
    subprocess.run(["gcc", "-I", os.path.dirname(HEADER), str(src), "-o", str(exe)], check=True)
    got = [int(x) for x in subprocess.check_output([str(exe)]).split()]
    M, T = _lib.DffmModel, _lib.DffmTrainState
    want = [ctypes.sizeof(M), M.lr.offset, M.q_ffm_bucket.offset, ctypes.sizeof(T),
            T.lr_ffm.offset, T.sparse.offset]
    assert got == want


def test_status_word_decoding():
    from paper_2407_10115_b200.errors import ContractError, NumericError
    _lib.raise_status(_lib.STATUS_CLEAR)
    with pytest.raises(NumericError) as ei:
        _lib.raise_status((17 << 8) | (3 << 4) | 3)
    assert ei.value.block == "merge" and ei.value.example == 17
    with pytest.raises(ContractError):
        _lib.raise_status((2 << 8) | 1)


def test_fwq_header_host_entry_matches_oracle():
    """fwq_header is the one host-side (no device) entry point: check it here."""
    import numpy as np

    from oracle import fieldwise_oracle as fo
    from paper_2407_10115_b200 import quant
    rng = np.random.default_rng(0)
    for _ in range(2000):
        a, b = sorted((rng.standard_normal(2) * rng.choice([1e-3, 0.05, 3.0])).astype(np.float32))
        assert quant.header(a, b) == fo.quant_header(float(a), float(b))
        al, be = int(rng.integers(0, 7)), int(rng.integers(0, 7))
        assert quant.header(a, b, al, be) == fo.quant_header(float(a), float(b), al, be)
    assert quant.header(np.float32(0.25), np.float32(0.25))[1] == 0.0
