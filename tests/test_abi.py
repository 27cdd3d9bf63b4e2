"""Host-side checks of the C ABI that need no GPU (-m "not gpu"): the library loads, exports every
symbol include/ntbc.h declares, and rejects bad arguments with the documented status codes before
touching the device."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2407_09543_b200", "libntbc.so")


def _declared():
    src = open(os.path.join(ROOT, "include", "ntbc.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ntbc_[a-z_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        import subprocess
        subprocess.check_call(["make", "-s", "-C", os.path.join(ROOT, "paper_2407_09543_b200", "csrc")])
    return C.CDLL(LIB)


def test_exports_every_declared_symbol(lib):
    names = _declared()
    assert len(names) >= 10
    for n in names:
        assert hasattr(lib, n), n


def test_binding_exposes_same_names():
    from paper_2407_09543_b200 import ntbc
    assert sorted(ntbc.EXPORTED) == _declared()


def test_load_model_rejects_bad_blobs_without_gpu(lib):
    lib.ntbc_load_model.restype = C.c_int
    lib.ntbc_last_error.restype = C.c_char_p
    h = C.c_void_p()
    assert lib.ntbc_load_model(None, 0, 0, C.byref(h)) == -1                     # NTBC_EINVAL
    bad = C.create_string_buffer(b"XTBC" + b"\0" * 200)
    assert lib.ntbc_load_model(bad, 204, 0, C.byref(h)) == -2                    # NTBC_EFORMAT
    assert b"magic" in lib.ntbc_last_error()
    import synth
    blob = synth.model_blob(1)
    trunc = C.create_string_buffer(blob[:1000])
    assert lib.ntbc_load_model(trunc, 1000, 0, C.byref(h)) == -2
    assert b"truncated" in lib.ntbc_last_error()


def test_decode_rejects_bad_dims_without_gpu(lib):
    lib.ntbc_decode_bc.restype = C.c_int
    buf = C.create_string_buffer(64)
    assert lib.ntbc_decode_bc(buf, 1, 6, 8, buf, None) == -1                      # width % 4
    assert lib.ntbc_decode_bc(buf, 2, 8, 8, buf, None) == -1                      # bad format
    lib.ntbc_pack.restype = C.c_int
    f = (C.c_int * 1)(3)
    ptrs = (C.c_void_p * 1)(C.addressof(buf))
    assert lib.ntbc_pack(1, f, buf, buf, 8, 8, 0, 2, ptrs, None) == -1           # bad format code
    f = (C.c_int * 1)(1)
    assert lib.ntbc_pack(1, f, buf, buf, 8, 8, 1, 1, ptrs, None) == -1           # empty row range


def test_load_model_fuzzed_blobs_never_crash(lib):
    """Truncations and random byte corruptions of valid containers (both variants) are rejected with
    a status code (EFORMAT / EMISMATCH / EINVAL, or ECUDA once parsing passes on a GPU-less host) --
    the parser never reads out of bounds or crashes."""
    import numpy as np
    import synth
    lib.ntbc_load_model.restype = C.c_int
    lib.ntbc_free_model.restype = None
    rng = np.random.default_rng(0)
    for cfg in (1, 8):
        blob = bytearray(synth.model_blob(cfg))
        cases = [bytes(blob[:n]) for n in (0, 4, 95, 96, 97, 150, len(blob) // 2, len(blob) - 1)]
        for _ in range(150):
            b = bytearray(blob)
            for _ in range(int(rng.integers(1, 4))):
                pos = int(rng.integers(0, 160)) if rng.random() < 0.7 else int(rng.integers(0, len(b)))
                b[pos] = int(rng.integers(0, 256))
            cases.append(bytes(b))
        for data in cases:
            h = C.c_void_p()
            buf = C.create_string_buffer(data, max(1, len(data)))
            st = lib.ntbc_load_model(buf, len(data), 0, C.byref(h))
            assert st in (0, -1, -2, -3, -4, -5)
            if st == 0:
                lib.ntbc_free_model(h)
