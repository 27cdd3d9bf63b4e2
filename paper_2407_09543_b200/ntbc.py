"""Thin ctypes binding of libntbc.so (include/ntbc.h): argument marshalling only.

Every step of the hot path runs in the CUDA kernels of libntbc.so.  There is no
CPU fallback: if the library is missing this module raises at import time.
PyTorch supplies device memory (tensors) and streams; pointers are passed as
integers.  Names follow the C ABI (ntbc_<name> -> <name>).
"""
from __future__ import annotations

import ctypes as C
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# NTBC_LIB selects another in-tree build of the same library (A/B measurements of kernel variants)
LIB_PATH = os.path.join(_HERE, os.environ.get("NTBC_LIB", "libntbc.so"))
BC1, BC4 = 1, 4

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
                      "(there is no CPU fallback)")

_lib = C.CDLL(LIB_PATH)
_vp, _i, _sz = C.c_void_p, C.c_int, C.c_size_t


class _Info(C.Structure):
    _fields_ = [("n_textures", C.c_int), ("fmt", C.c_int * 8), ("hidden", C.c_int), ("n_hidden", C.c_int),
                ("n_endpoint_out", C.c_int), ("n_color_out", C.c_int), ("block_levels", C.c_int),
                ("block_coarsest", C.c_int), ("texel_levels", C.c_int), ("texel_coarsest", C.c_int),
                ("features", C.c_int), ("variant", C.c_int), ("device_bytes", C.c_size_t)]


_SIGS = {
    "ntbc_load_model": (_i, [_vp, _sz, _i, C.POINTER(_vp)]),
    "ntbc_model_upload_async": (_i, [_vp, _vp, _sz, _vp]),
    "ntbc_model_get_info": (_i, [_vp, C.POINTER(_Info)]),
    "ntbc_free_model": (None, [_vp]),
    "ntbc_decode_material": (_i, [_vp, _i, _i, _i, _i, _i, _vp, _vp]),
    "ntbc_decode_material_host": (_i, [_vp, _i, _vp, _vp, _i, _i, _vp, _vp]),
    "ntbc_decode_bc": (_i, [_vp, _i, _i, _i, _vp, _vp]),
    "ntbc_encode_bc": (_i, [_vp, _i, _i, _i, _i, _vp, _vp]),
    "ntbc_debug_host_timeline": (_i, [_vp, _vp, _i]),
    "ntbc_train_param_count": (C.c_longlong, [_vp]),
    "ntbc_train_endpoint_param_count": (C.c_longlong, [_vp]),
    "ntbc_train_endpoint_step": (_i, [_vp, _vp, _vp, _vp, _vp, _i, _vp, _vp, _vp, _i, _i, _i, C.c_float, C.c_float,
                                      C.c_float, _vp, _vp]),
    "ntbc_train_colour_step": (_i, [_vp, _vp, _vp, _vp, _vp, _i, _vp, _vp, _vp, _i, _i, _i, C.c_float, C.c_float,
                                    C.c_float, _vp, _vp]),
    "ntbc_debug_mlp": (_i, [_vp, _i, _i, _i, _i, _vp, _vp, _vp]),
    "ntbc_debug_features": (_i, [_vp, _i, _i, _i, _i, _vp, _vp, _vp]),
    "ntbc_pack": (_i, [_i, _vp, _vp, _vp, _i, _i, _i, _i, _vp, _vp]),
    "ntbc_debug_mma": (_i, [_vp, _vp, _vp, _vp, _i, _i, _vp]),
    "ntbc_peer_export": (_i, [_vp, _vp]),
    "ntbc_peer_open": (_i, [_vp, _i, C.POINTER(_vp)]),
    "ntbc_peer_close": (_i, [_vp]),
    "ntbc_launch_count": (C.c_uint64, []),
    "ntbc_debug_time_fused": (_i, [_vp, _vp]),
    "ntbc_set_contract": (_i, [_vp, _i]),
    "ntbc_last_error": (C.c_char_p, []),
}
for _name, (_res, _args) in _SIGS.items():
    _fn = getattr(_lib, _name)
    _fn.restype = _res
    _fn.argtypes = _args

EXPORTED = tuple(_SIGS)


class NtbcError(RuntimeError):
    pass


def _check(rc: int):
    if rc != 0:
        raise NtbcError(f"ntbc error {rc}: {_lib.ntbc_last_error().decode()}")


def _stream(stream) -> int:
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def _ptr(t) -> int:
    return 0 if t is None else t.data_ptr()


class Model:
    """A model loaded on one device (ntbc_load_model)."""

    def __init__(self, blob: bytes, device: int = 0):
        self._h = _vp()
        buf = C.create_string_buffer(blob, len(blob))
        _check(_lib.ntbc_load_model(buf, len(blob), device, C.byref(self._h)))
        self.device = device
        info = _Info()
        _check(_lib.ntbc_model_get_info(self._h, C.byref(info)))
        self.n_tex = info.n_textures
        self.fmts = [info.fmt[i] for i in range(info.n_textures)]
        self.hidden = info.hidden
        self.n_e, self.n_c = info.n_endpoint_out, info.n_color_out
        self.device_bytes = info.device_bytes
        self.naive = bool(info.variant)

    @property
    def handle(self):
        return self._h

    def upload_async(self, pinned_blob: torch.Tensor, stream=None):
        _check(_lib.ntbc_model_upload_async(self._h, pinned_blob.data_ptr(), pinned_blob.numel(), _stream(stream)))

    def free(self):
        if self._h:
            _lib.ntbc_free_model(self._h)
            self._h = _vp()

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def _handles(models):
    arr = (_vp * len(models))(*[m.handle.value for m in models])
    return arr


def alloc_outputs(models, width: int, height: int, row_begin: int = 0, row_end: int | None = None, device=None):
    row_end = height // 4 if row_end is None else row_end
    dev = torch.device("cuda", models[0].device) if device is None else device
    n = sum(m.n_tex for m in models)
    return [torch.empty((row_end - row_begin, width // 4), dtype=torch.int64, device=dev) for _ in range(n)]


def decode_material(models, width: int, height: int, outs=None, row_begin: int = 0, row_end: int | None = None,
                    stream=None, out_ptrs=None):
    """ntbc_decode_material: returns one int64 [rows][W/4] tensor of BC words per texture.
    out_ptrs: raw device pointers (one per texture) instead of tensors, e.g. rank 0's buffer mapped
    with peer_open (the fused peer-memory gather); then nothing is returned."""
    row_end = height // 4 if row_end is None else row_end
    if out_ptrs is not None:
        ptrs = (_vp * len(out_ptrs))(*out_ptrs)
        _check(_lib.ntbc_decode_material(_handles(models), len(models), width, height, row_begin, row_end, ptrs,
                                         _stream(stream)))
        return None
    if outs is None:
        outs = alloc_outputs(models, width, height, row_begin, row_end)
    ptrs = (_vp * len(outs))(*[o.data_ptr() for o in outs])
    _check(_lib.ntbc_decode_material(_handles(models), len(models), width, height, row_begin, row_end, ptrs,
                                     _stream(stream)))
    return outs


def decode_material_host(models, pinned_blobs, width: int, height: int, host_outs, stream=None):
    """ntbc_decode_material_host: pinned host blobs in, pinned host BC words out (async on stream)."""
    blobs = (_vp * len(models))(*[b.data_ptr() for b in pinned_blobs])
    sizes = (_sz * len(models))(*[b.numel() for b in pinned_blobs])
    outs = (_vp * len(host_outs))(*[o.data_ptr() for o in host_outs])
    _check(_lib.ntbc_decode_material_host(_handles(models), len(models), blobs, sizes, width, height, outs,
                                          _stream(stream)))


def debug_host_timeline(model):
    """Event times (ms) of the model's last ntbc_decode_material_host call (needs NTBC_TIMELINE=1)."""
    out = (C.c_float * 13)()
    _check(_lib.ntbc_debug_host_timeline(model.handle, out, 13))
    return list(out)


def encode_bc(texels: torch.Tensor, fmt: int, width: int, height: int, n_refine: int = 2, out=None, stream=None):
    """ntbc_encode_bc: reference BC1/BC4 encoder (fp32 [H][W][3|1] device texels -> int64 [H/4][W/4])."""
    if out is None:
        out = torch.empty((height // 4, width // 4), dtype=torch.int64, device=texels.device)
    _check(_lib.ntbc_encode_bc(texels.data_ptr(), fmt, width, height, n_refine, out.data_ptr(), _stream(stream)))
    return out


class _TrainArch(C.Structure):
    _fields_ = [("n_textures", C.c_int), ("fmt", C.c_int * 8), ("hidden", C.c_int), ("levels", C.c_int),
                ("coarsest", C.c_int), ("qat", C.c_int)]


def _train_arch(fmts, hidden, levels, coarsest, qat=False):
    a = _TrainArch()
    a.qat = int(bool(qat))
    a.n_textures = len(fmts)
    for i, f in enumerate(fmts):
        a.fmt[i] = f
    a.hidden, a.levels, a.coarsest = hidden, levels, coarsest
    return a


def train_param_count(fmts, hidden=64, levels=8, coarsest=16) -> int:
    n = int(_lib.ntbc_train_param_count(C.byref(_train_arch(fmts, hidden, levels, coarsest))))
    if n < 0:
        raise NtbcError(-1, "unsupported training architecture")
    return n


def train_colour_step(fmts, params, grads, adam_m, adam_v, step, xy, cref, eref, width, height,
                      temperature=0.01, lr_grid=0.01, lr_mlp=0.005, hidden=64, levels=8, coarsest=16,
                      loss=None, stream=None, qat=False):
    """ntbc_train_colour_step on device fp32 tensors (params/grads/adam_m/adam_v: flat; xy int32 [B][2])."""
    if loss is None:
        loss = torch.zeros(1, dtype=torch.float32, device=params.device)
    arch = _train_arch(fmts, hidden, levels, coarsest, qat)
    _check(_lib.ntbc_train_colour_step(C.byref(arch), params.data_ptr(), grads.data_ptr(), adam_m.data_ptr(),
                                       adam_v.data_ptr(), step, xy.data_ptr(), cref.data_ptr(), eref.data_ptr(),
                                       xy.shape[0], width, height, temperature, lr_grid, lr_mlp, loss.data_ptr(),
                                       _stream(stream)))
    return loss


def train_endpoint_param_count(fmts, hidden=64, levels=7, coarsest=16) -> int:
    n = int(_lib.ntbc_train_endpoint_param_count(C.byref(_train_arch(fmts, hidden, levels, coarsest))))
    if n < 0:
        raise NtbcError(-1, "unsupported training architecture")
    return n


def train_endpoint_step(fmts, params, grads, adam_m, adam_v, step, bxy, cref16, eref, blocks_w, blocks_h,
                        temperature=0.01, lr_grid=0.01, lr_mlp=0.005, hidden=64, levels=7, coarsest=16,
                        loss=None, stream=None, qat=False):
    """ntbc_train_endpoint_step: bxy int32 [B][2] block coords, cref16 [B][16][N_c], eref [B][N_e]."""
    if loss is None:
        loss = torch.zeros(1, dtype=torch.float32, device=params.device)
    arch = _train_arch(fmts, hidden, levels, coarsest, qat)
    _check(_lib.ntbc_train_endpoint_step(C.byref(arch), params.data_ptr(), grads.data_ptr(), adam_m.data_ptr(),
                                         adam_v.data_ptr(), step, bxy.data_ptr(), cref16.data_ptr(), eref.data_ptr(),
                                         bxy.shape[0], blocks_w, blocks_h, temperature, lr_grid, lr_mlp,
                                         loss.data_ptr(), _stream(stream)))
    return loss


def decode_bc(blocks: torch.Tensor, fmt: int, width: int, height: int, out=None, stream=None):
    ch = 3 if fmt == BC1 else 1
    if out is None:
        out = torch.empty((height, width, ch), dtype=torch.float32, device=blocks.device)
    _check(_lib.ntbc_decode_bc(blocks.data_ptr(), fmt, width, height, out.data_ptr(), _stream(stream)))
    return out


def debug_mlp(model: Model, width: int, height: int, row_begin: int = 0, row_end: int | None = None, stream=None):
    row_end = height // 4 if row_end is None else row_end
    rows = row_end - row_begin
    dev = torch.device("cuda", model.device)
    ep = torch.empty((rows, width // 4, model.n_e), dtype=torch.float32, device=dev)
    col = torch.empty((rows * 4, width, model.n_c), dtype=torch.float32, device=dev)
    _check(_lib.ntbc_debug_mlp(model.handle, width, height, row_begin, row_end, ep.data_ptr(), col.data_ptr(),
                               _stream(stream)))
    return ep, col


def debug_features(model: Model, width: int, height: int, row_begin: int = 0, row_end: int | None = None,
                   stream=None):
    """fp32 grid features (16 per block / texel) of block rows [row_begin, row_end)."""
    row_end = height // 4 if row_end is None else row_end
    rows = row_end - row_begin
    dev = torch.device("cuda", model.device)
    bf = torch.zeros((rows, width // 4, 16), dtype=torch.float32, device=dev)
    tf = torch.zeros((rows * 4, width, 16), dtype=torch.float32, device=dev)
    _check(_lib.ntbc_debug_features(model.handle, width, height, row_begin, row_end, bf.data_ptr(), tf.data_ptr(),
                                    _stream(stream)))
    return bf, tf


def pack(fmts, endpoints: torch.Tensor, colors: torch.Tensor, width: int, height: int, row_begin: int = 0,
         row_end: int | None = None, outs=None, stream=None):
    row_end = height // 4 if row_end is None else row_end
    if outs is None:
        outs = [torch.empty((row_end - row_begin, width // 4), dtype=torch.int64, device=endpoints.device)
                for _ in fmts]
    f = (C.c_int * len(fmts))(*fmts)
    ptrs = (_vp * len(outs))(*[o.data_ptr() for o in outs])
    _check(_lib.ntbc_pack(len(fmts), f, endpoints.data_ptr(), colors.data_ptr(), width, height, row_begin, row_end,
                          ptrs, _stream(stream)))
    return outs


def debug_mma(A: torch.Tensor, B: torch.Tensor, Cin, K: int, N: int, stream=None):
    D = torch.empty((128, N), dtype=torch.float32, device=A.device)
    _check(_lib.ntbc_debug_mma(A.data_ptr(), B.data_ptr(), _ptr(Cin), D.data_ptr(), K, N, _stream(stream)))
    return D


PEER_HANDLE_BYTES = 72


def peer_export(t: torch.Tensor) -> bytes:
    """ntbc_peer_export: CUDA-IPC handle (+ offset) of a device tensor's memory, to send to other ranks."""
    buf = C.create_string_buffer(PEER_HANDLE_BYTES)
    _check(_lib.ntbc_peer_export(t.data_ptr(), buf))
    return buf.raw


def peer_open(handle: bytes, device: int) -> int:
    """ntbc_peer_open: map another process's exported memory on `device`; returns a raw device pointer."""
    if len(handle) != PEER_HANDLE_BYTES:
        raise ValueError("bad peer handle")
    p = _vp()
    _check(_lib.ntbc_peer_open(C.create_string_buffer(handle, PEER_HANDLE_BYTES), device, C.byref(p)))
    return p.value


def peer_close(ptr: int):
    _check(_lib.ntbc_peer_close(ptr))


def launch_count() -> int:
    return int(_lib.ntbc_launch_count())


def time_fused(start_event=None, end_event=None):
    """ntbc_debug_time_fused: record torch.cuda.Event `start_event` / `end_event` right before / after every
    fused-kernel launch of this thread (None, None clears)."""
    a = start_event.cuda_event if start_event is not None else None
    b = end_event.cuda_event if end_event is not None else None
    _check(_lib.ntbc_debug_time_fused(a, b))


def set_contract(model, contract: int):
    """ntbc_set_contract: 0 = H (binary16 activations, the paper's), 1 = F (binary32 activations, hi/lo operands),
    2 = P (H with the selu evaluated in binary16 arithmetic on f16x2 lanes)."""
    _check(_lib.ntbc_set_contract(model._h, int(contract)))
