"""Host-side packed layout (numpy): the reference's on-disk / in-memory list format.

pack_list / unpack_list follow layout.hpp:50-68 (LSB-first subcode packing into 8/16-bit words)
and layout.hpp:105-176 (transposed blocks of block_len codes, rows contiguous, tail slots padded
with all-ones words).  Used to prepare inputs for the C ABI, which consumes exactly this format.
"""
from __future__ import annotations

import numpy as np

from ._lib import QadcError, QadcSpec


def pack_list(spec: QadcSpec, codes: np.ndarray) -> np.ndarray:
    codes = np.ascontiguousarray(codes, dtype=np.uint8).reshape(-1, spec.m)
    n = codes.shape[0]
    g, rows, bl = spec.g, spec.groups, spec.block_len
    for k in range(g):
        if n and int(codes[:, k::g].max()) >= (1 << spec.widths[k]):
            raise QadcError(6, f"pack_group: index exceeds {spec.widths[k]} bits")  # layout.hpp:55-57
    wdt = np.uint8 if spec.word_width == 8 else np.dtype("<u2")
    words = np.zeros((n, rows), dtype=np.uint32)
    c = codes.reshape(n, rows, g).astype(np.uint32)
    for k in range(g):
        words |= c[:, :, k] << np.uint32(spec.offsets[k])
    nblocks = (n + bl - 1) // bl
    out = np.full((nblocks, rows, bl), 0xFFFF if spec.word_width == 16 else 0xFF, dtype=wdt)
    if n:
        flat = out.reshape(nblocks, rows, bl)
        idx = np.arange(n)
        flat[idx // bl, :, idx % bl] = words.astype(wdt)
    return out.reshape(-1).view(np.uint8)


def unpack_list(spec: QadcSpec, packed: np.ndarray, n: int) -> np.ndarray:
    g, rows, bl = spec.g, spec.groups, spec.block_len
    wdt = np.uint8 if spec.word_width == 8 else np.dtype("<u2")
    nblocks = (n + bl - 1) // bl
    words = np.ascontiguousarray(packed, dtype=np.uint8).view(wdt)[: nblocks * rows * bl].reshape(nblocks, rows, bl)
    idx = np.arange(n)
    w = words[idx // bl, :, idx % bl].astype(np.uint32)  # [n, rows]
    out = np.empty((n, rows, g), dtype=np.uint8)
    for k in range(g):
        out[:, :, k] = (w >> np.uint32(spec.offsets[k])) & np.uint32((1 << spec.widths[k]) - 1)
    return out.reshape(n, rows * g)
