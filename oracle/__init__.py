"""ctypes wrapper of the CPU oracle (oracle/ntbc_oracle.c).

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / `--impl reference` arm may import this module.  The
product package (paper_2407_09543_b200) never imports it and shares no code
with it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
BC1, BC4 = 1, 4


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "ntbc_oracle.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(["make", "-s", "-C", _HERE, "liboracle.so"])
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB_PATH)
        f32, i32, u16, u8, u64, vp, sz = C.c_float, C.c_int, C.c_uint16, C.c_uint8, C.c_uint64, C.c_void_p, C.c_size_t
        sig = {
            "o_model_parse": (i32, [vp, sz, C.POINTER(vp)]),
            "o_model_free": (None, [vp]),
            "o_model_info": (None, [vp, vp]),
            "o_f16_to_f32": (f32, [u16]),
            "o_f32_to_f16": (u16, [f32]),
            "o_f32_to_f16_n": (None, [vp, vp, sz]),
            "o_dequant": (f32, [u8, f32, C.c_int32]),
            "o_exp": (f32, [f32]),
            "o_expm1": (f32, [f32]),
            "o_selu": (f32, [f32]),
            "o_sigmoid": (f32, [f32]),
            "o_set_dot_model": (None, [i32, i32, i32, i32]),
            "o_get_dot_model": (None, [vp]),
            "o_dot": (f32, [f32, vp, i32, vp, i32]),
            "o_fused_sum": (f32, [vp, vp, vp, i32, i32, i32]),
            "o_grid_encode": (None, [vp, i32, f32, f32, vp]),
            "o_mlp_forward": (None, [vp, i32, vp, vp]),
            "o_mlp_raw": (None, [i32, vp, vp, vp, vp, vp]),
            "o_rgb565": (u16, [vp]),
            "o_unorm8": (u8, [f32]),
            "o_expand565": (None, [u16, vp]),
            "o_palette_bc1": (None, [vp, vp, vp]),
            "o_palette_bc4": (None, [u8, u8, vp]),
            "o_argmin_bc1": (i32, [vp, vp]),
            "o_argmin_bc4": (i32, [f32, vp]),
            "o_encode_bc1": (u64, [vp, vp]),
            "o_encode_bc4": (u64, [vp, vp]),
            "o_quantize_weight": (i32, [f32, i32, i32]),
            "o_encode_ref_bc1": (u64, [vp, i32]),
            "o_encode_ref_bc4": (u64, [vp, i32]),
            "o_encode_ref_texture": (None, [vp, i32, i32, i32, i32, vp, i32]),
            "o_encode_bc1_naive": (u64, [vp, vp]),
            "o_encode_bc4_naive": (u64, [vp, vp]),
            "o_decode_block": (None, [u64, i32, vp]),
            "o_decode_material": (None, [vp, i32, i32, i32, i32, vp, i32]),
            "o_mlp_outputs": (None, [vp, i32, i32, i32, i32, vp, vp, i32]),
            "o_pack": (None, [i32, vp, vp, vp, i32, i32, i32, i32, vp, i32]),
            "o_decode_bc": (None, [vp, i32, i32, i32, vp]),
            "o_psnr": (C.c_double, [vp, vp, sz]),
            "o_bruteforce_bc4": (u64, [vp, vp]),
            "o_block_sq_error": (C.c_double, [u64, i32, vp]),
            "o_storage_bytes": (u64, [i32] * 10),
            "o_exp_max_relerr": (C.c_double, [f32, f32, i32, i32]),
            "o_set_act_model": (None, [i32]),
            "o_get_act_model": (i32, []),
            "o_set_operand_model": (None, [i32]),
            "o_f64_to_f16": (u16, [C.c_double]),
            "o_h16_fma": (u16, [u16, u16, u16]),
            "o_h16_mul": (u16, [u16, u16]),
            "o_h16_sub": (u16, [u16, u16]),
            "o_selu_half": (u16, [f32]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


class Model:
    """A parsed `.ntbc` model held by the oracle."""

    def __init__(self, blob: bytes):
        self._buf = np.frombuffer(blob, np.uint8).copy()
        h = C.c_void_p()
        rc = lib().o_model_parse(_p(self._buf), self._buf.size, C.byref(h))
        if rc != 0:
            raise ValueError(f"oracle: bad model blob (rc={rc})")
        self.h = h
        info = np.zeros(17, np.int32)
        lib().o_model_info(h, _p(info))
        self.n_tex = int(info[0])
        self.fmts = [int(x) for x in info[1:1 + self.n_tex]]
        self.hidden, self.n_e, self.n_c = int(info[9]), int(info[10]), int(info[11])
        self.block_levels, self.texel_levels = int(info[12]), int(info[14])
        self.naive = bool(info[16])

    def __del__(self):
        try:
            lib().o_model_free(self.h)
        except Exception:
            pass

    def decode_material(self, W, H, row_begin=0, row_end=None, nthreads=0) -> np.ndarray:
        row_end = H // 4 if row_end is None else row_end
        out = np.zeros((self.n_tex, row_end - row_begin, W // 4), np.uint64)
        lib().o_decode_material(self.h, W, H, row_begin, row_end, _p(out), nthreads)
        return out

    def mlp_outputs(self, W, H, row_begin=0, row_end=None, nthreads=0):
        row_end = H // 4 if row_end is None else row_end
        rows = row_end - row_begin
        ep = np.zeros((rows, W // 4, self.n_e), np.float32)
        col = np.zeros((rows * 4, W, self.n_c), np.float32)
        lib().o_mlp_outputs(self.h, W, H, row_begin, row_end, _p(ep), _p(col), nthreads)
        return ep, col

    def grid_encode(self, which: int, p: float, q: float) -> np.ndarray:
        n = self.block_levels * 2 if which == 0 else self.texel_levels * 2
        out = np.zeros(n, np.float32)
        lib().o_grid_encode(self.h, which, p, q, _p(out))
        return out

    def mlp_forward(self, which: int, x: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float32)
        out = np.zeros(self.n_e if which == 0 else self.n_c, np.float32)
        lib().o_mlp_forward(self.h, which, _p(x), _p(out))
        return out


def pack(fmts, ep: np.ndarray, col: np.ndarray, W, H, row_begin=0, row_end=None, nthreads=0):
    row_end = H // 4 if row_end is None else row_end
    f = np.asarray(fmts, np.int32)
    ep = np.ascontiguousarray(ep, np.float32)
    col = np.ascontiguousarray(col, np.float32)
    out = np.zeros((len(fmts), row_end - row_begin, W // 4), np.uint64)
    lib().o_pack(len(fmts), _p(f), _p(ep), _p(col), W, H, row_begin, row_end, _p(out), nthreads)
    return out


def decode_bc(blocks: np.ndarray, fmt: int, W: int, H: int) -> np.ndarray:
    b = np.ascontiguousarray(blocks, np.uint64)
    out = np.zeros((H, W, 3 if fmt == BC1 else 1), np.float32)
    lib().o_decode_bc(_p(b), fmt, W, H, _p(out))
    return out


def f32_to_f16(x: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x, np.float32)
    out = np.zeros(x.shape, np.uint16)
    lib().o_f32_to_f16_n(_p(x), _p(out), x.size)
    return out


def psnr(a: np.ndarray, b: np.ndarray) -> float:
    a = np.ascontiguousarray(a, np.float32)
    b = np.ascontiguousarray(b, np.float32)
    return float(lib().o_psnr(_p(a), _p(b), a.size))


def set_dot_model(mode: int, chunk: int = 16, p_bits: int = 100, rmode: int = 0):
    lib().o_set_dot_model(mode, chunk, p_bits, rmode)


def get_dot_model():
    o = np.zeros(4, np.int32)
    lib().o_get_dot_model(_p(o))
    return tuple(int(x) for x in o)


def set_act_model(plain: int):
    lib().o_set_act_model(int(plain))


def set_operand_model(split: int):
    """0 = contract H (binary16 layer inputs, the kernels' default); 1 = contract F (binary32 activations,
    hi/lo split operands; the library's ntbc_set_contract(m, 1))."""
    lib().o_set_operand_model(int(split))


class contract_f:
    """Context manager: the oracle computes contract F (its pinned or plain arithmetic as set otherwise)."""

    def __enter__(self):
        set_operand_model(1)
        return self

    def __exit__(self, *exc):
        set_operand_model(0)
        return False


class contract_p:
    """Context manager: the oracle computes contract P: the hidden selu in
    binary16 arithmetic (R9-P, `o_selu_half`), everything else pinned as in contract H."""

    def __enter__(self):
        self._act = int(lib().o_get_act_model())
        set_act_model(3)
        return self

    def __exit__(self, *exc):
        set_act_model(self._act)
        return False


class plain_definitions:
    """Context manager: the oracle computes the PLAIN definitions (every dot product exact and rounded
    once, selu / sigmoid in float64 with libm, one rounding) instead of the pinned op sequences the
    kernels execute (R9, R10).  The binary16 operand rounding of P:322 / P:331 stays."""

    def __enter__(self):
        self._dot = get_dot_model()
        self._act = int(lib().o_get_act_model())
        set_dot_model(0)
        set_act_model(1)
        return self

    def __exit__(self, *exc):
        set_dot_model(*self._dot)
        set_act_model(self._act)
        return False


def mlp_raw(weights, biases, x) -> np.ndarray:
    """weights: list of fp16 [in][out]; biases: list of fp16 [out]; x: fp32 [in]."""
    n = len(weights)
    dims = np.array([weights[0].shape[0]] + [w.shape[1] for w in weights], np.int32)
    ws = [np.ascontiguousarray(w, np.float16) for w in weights]
    bs = [np.ascontiguousarray(b, np.float16) for b in biases]
    wp = (C.c_void_p * n)(*[w.ctypes.data for w in ws])
    bp = (C.c_void_p * n)(*[b.ctypes.data for b in bs])
    x = np.ascontiguousarray(x, np.float32)
    out = np.zeros(dims[-1], np.float32)
    lib().o_mlp_raw(n, _p(dims), wp, bp, _p(x), _p(out))
    return out


def encode_bc1(ep6, texels16x3) -> int:
    e = np.ascontiguousarray(ep6, np.float32)
    t = np.ascontiguousarray(texels16x3, np.float32).reshape(-1)
    return int(lib().o_encode_bc1(_p(e), _p(t)))


def encode_bc4(ep2, texels16) -> int:
    e = np.ascontiguousarray(ep2, np.float32)
    t = np.ascontiguousarray(texels16, np.float32).reshape(-1)
    return int(lib().o_encode_bc4(_p(e), _p(t)))


def rgb565(e3) -> int:
    e = np.ascontiguousarray(e3, np.float32)
    return int(lib().o_rgb565(_p(e)))


def expand565(c: int) -> np.ndarray:
    out = np.zeros(3, np.float32)
    lib().o_expand565(int(c), _p(out))
    return out


def encode_ref_block(texels, fmt: int, n_refine: int = 2) -> int:
    """Reference BC encoder of one 4x4 block (SPEC encode_block_reference; 16x3 for BC1, 16 for BC4)."""
    t = np.ascontiguousarray(texels, np.float32).reshape(-1)
    f = lib().o_encode_ref_bc1 if fmt == 1 else lib().o_encode_ref_bc4
    return int(f(_p(t), int(n_refine)))


def encode_ref_texture(tex, n_refine: int = 2, nthreads: int = 0) -> np.ndarray:
    """fp32 [H][W][C] texture (C = 3 -> BC1, 1 -> BC4) -> uint64 [H/4][W/4] blocks."""
    t = np.ascontiguousarray(tex, np.float32)
    H, W = t.shape[:2]
    C = t.shape[2] if t.ndim == 3 else 1
    out = np.zeros((H // 4, W // 4), np.uint64)
    lib().o_encode_ref_texture(_p(t), W, H, C, int(n_refine), _p(out), nthreads)
    return out


def quantize_weight(w: float, fmt: int, mode8: bool = True) -> int:
    """Naive approach: linear palette index of the nearest palette weight (ties -> lower n)."""
    return int(lib().o_quantize_weight(float(w), int(fmt), int(bool(mode8))))


def encode_bc1_naive(ep6, weights16) -> int:
    e = np.ascontiguousarray(ep6, np.float32)
    w = np.ascontiguousarray(weights16, np.float32).reshape(-1)
    return int(lib().o_encode_bc1_naive(_p(e), _p(w)))


def encode_bc4_naive(ep2, weights16) -> int:
    e = np.ascontiguousarray(ep2, np.float32)
    w = np.ascontiguousarray(weights16, np.float32).reshape(-1)
    return int(lib().o_encode_bc4_naive(_p(e), _p(w)))


def decode_block(blk: int, fmt: int) -> np.ndarray:
    out = np.zeros(48 if fmt == BC1 else 16, np.float32)
    lib().o_decode_block(blk, fmt, _p(out))
    return out.reshape(16, 3) if fmt == BC1 else out


def palette_bc1(e0, e1) -> np.ndarray:
    a = np.ascontiguousarray(e0, np.float32)
    b = np.ascontiguousarray(e1, np.float32)
    out = np.zeros((4, 3), np.float32)
    lib().o_palette_bc1(_p(a), _p(b), _p(out))
    return out


def palette_bc4(E0: int, E1: int) -> np.ndarray:
    out = np.zeros(8, np.float32)
    lib().o_palette_bc4(E0, E1, _p(out))
    return out


def fused_sum(acc, a16: np.ndarray, b16: np.ndarray, p_bits: int, rmode: int) -> float:
    a = np.ascontiguousarray(a16, np.float16)
    b = np.ascontiguousarray(b16, np.float16)
    if acc is None:
        return float(lib().o_fused_sum(None, _p(a), _p(b), a.size, p_bits, rmode))
    accv = np.array([acc], np.float32)
    return float(lib().o_fused_sum(_p(accv), _p(a), _p(b), a.size, p_bits, rmode))


def bruteforce_bc4(texels16):
    t = np.ascontiguousarray(texels16, np.float32)
    err = np.zeros(1, np.float64)
    blk = int(lib().o_bruteforce_bc4(_p(t), _p(err)))
    return blk, float(err[0])


def block_sq_error(blk: int, fmt: int, texels) -> float:
    t = np.ascontiguousarray(texels, np.float32).reshape(-1)
    return float(lib().o_block_sq_error(blk, fmt, _p(t)))
