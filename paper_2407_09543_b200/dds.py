"""DDS container for BC1/BC4 surfaces (host I/O plumbing; SPEC dds_write / dds_read).

Standard 128-byte preamble ("DDS " + 124-byte DDS_HEADER), fourCC "DXT1" (BC1) or "ATI1" (BC4),
DDSD_LINEARSIZE set, one mip level; the block words follow little-endian, row-major -- exactly the
layout ntbc_decode_material writes, so a decoded surface is written without any conversion."""
from __future__ import annotations

import struct

import numpy as np

_DDSD_CAPS, _DDSD_HEIGHT, _DDSD_WIDTH, _DDSD_PIXELFORMAT, _DDSD_LINEARSIZE = 0x1, 0x2, 0x4, 0x1000, 0x80000
_DDPF_FOURCC, _DDSCAPS_TEXTURE = 0x4, 0x1000
_FOURCC = {1: b"DXT1", 4: b"ATI1"}


def dds_bytes(blocks, fmt: int, width: int, height: int) -> bytes:
    """blocks: uint64/int64 [height/4][width/4] BC words (numpy or a CPU tensor)."""
    if fmt not in _FOURCC:
        raise ValueError(f"unsupported format {fmt}")
    words = np.ascontiguousarray(np.asarray(blocks).view(np.uint64)).reshape(-1)
    if width % 4 or height % 4 or words.size != (width // 4) * (height // 4):
        raise ValueError("block count does not match width x height")
    flags = _DDSD_CAPS | _DDSD_HEIGHT | _DDSD_WIDTH | _DDSD_PIXELFORMAT | _DDSD_LINEARSIZE
    pixfmt = struct.pack("<II4sIIIII", 32, _DDPF_FOURCC, _FOURCC[fmt], 0, 0, 0, 0, 0)
    hdr = struct.pack("<IIIIIII", 124, flags, height, width, words.size * 8, 0, 1) + b"\0" * 44 + pixfmt
    hdr += struct.pack("<IIIII", _DDSCAPS_TEXTURE, 0, 0, 0, 0)
    assert len(hdr) == 124
    return b"DDS " + hdr + words.astype("<u8").tobytes()


def write_dds(path: str, blocks, fmt: int, width: int, height: int) -> None:
    with open(path, "wb") as f:
        f.write(dds_bytes(blocks, fmt, width, height))


def read_dds(data: bytes):
    """-> (blocks uint64 [H/4][W/4], fmt, width, height); raises ValueError on a bad container."""
    if len(data) < 128 or data[:4] != b"DDS " or struct.unpack_from("<I", data, 4)[0] != 124:
        raise ValueError("bad DDS magic / header size")
    height, width = struct.unpack_from("<II", data, 12)
    fourcc = data[84:88]
    fmt = {v: k for k, v in _FOURCC.items()}.get(fourcc)
    if fmt is None:
        raise ValueError(f"unsupported fourCC {fourcc!r}")
    n = (width // 4) * (height // 4)
    if len(data) < 128 + 8 * n:
        raise ValueError("truncated payload")
    blocks = np.frombuffer(data, "<u8", n, 128).astype(np.uint64).reshape(height // 4, width // 4)
    return blocks, fmt, width, height
