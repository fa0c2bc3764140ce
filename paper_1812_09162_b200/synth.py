"""Seeded synthetic inputs with the shapes BASELINE.json names (stand-ins for SIFT/Deep-like data;
no dataset items are reproduced).  Data preparation only -- none of this is on the timed path.

* ``gaussian_mixture``  d-dim float32 from a mixture of 1024 isotropic Gaussians (sigma=1,
                        centres ~ N(0, 25 I)).
* ``train_codebook``    per-subspace Lloyd k-means (plain numpy; the codebook is an INPUT to the
                        path, any reasonable trainer will do -- the reference's own trainer is
                        exercised through the oracle in the tests).
* ``random_packed``     uniform random codes written straight in the packed layout (config 4).
"""
from __future__ import annotations

import numpy as np

from ._lib import QadcSpec

N_COMPONENTS = 1024


def mixture_centres(d: int, seed: int = 1) -> np.ndarray:
    return (np.random.default_rng(seed).standard_normal((N_COMPONENTS, d)) * 5.0).astype(np.float32)


def gaussian_mixture(n: int, d: int, seed: int, centres: np.ndarray | None = None) -> np.ndarray:
    centres = mixture_centres(d) if centres is None else centres
    rng = np.random.default_rng(seed)
    which = rng.integers(0, centres.shape[0], size=n)
    out = rng.standard_normal((n, d), dtype=np.float32)
    out += centres[which]
    return out


def _kmeans(x: np.ndarray, k: int, iters: int, rng) -> np.ndarray:
    c = x[rng.choice(x.shape[0], size=k, replace=False)].astype(np.float64)
    x64 = x.astype(np.float64)
    xx = (x64 * x64).sum(1)
    for _ in range(iters):
        d = xx[:, None] - 2.0 * x64 @ c.T + (c * c).sum(1)[None, :]
        a = d.argmin(1)
        for j in range(k):
            m = a == j
            if m.any():
                c[j] = x64[m].mean(0)
            else:
                c[j] = x64[rng.integers(x.shape[0])]
    return c.astype(np.float32)


def train_codebook(spec: QadcSpec, samples: np.ndarray, iters: int = 10, seed: int = 5) -> np.ndarray:
    """Flat codebook (spec.cb_floats floats): per subquantizer a k_j x dim_alloc[j] row-major matrix."""
    rng = np.random.default_rng(seed)
    parts = []
    for j in range(spec.m):
        off, ds = spec.dim_off[j], spec.dim_alloc[j]
        parts.append(_kmeans(samples[:, off:off + ds], 1 << spec.bits[j], iters, rng).reshape(-1))
    return np.concatenate(parts)


def random_codes(spec: QadcSpec, n: int, seed: int = 6) -> np.ndarray:
    rng = np.random.default_rng(seed)
    out = np.empty((n, spec.m), dtype=np.uint8)
    for j in range(spec.m):
        out[:, j] = rng.integers(0, 1 << spec.bits[j], size=n, dtype=np.uint8 if spec.bits[j] < 8 else np.uint16)
    return out


def random_packed(spec: QadcSpec, n: int, seed: int = 6) -> np.ndarray:
    """Uniform random subcodes directly in packed form.  Valid whenever every bit pattern of a word is a
    legal group ({4,4}, {6,5,5}, {6,6,4}, {8,8}, {8}: widths sum to the word width)."""
    assert sum(spec.widths[k] for k in range(spec.g)) == spec.word_width
    bl, rows, wb = spec.block_len, spec.groups, spec.word_width // 8
    nblocks = (n + bl - 1) // bl
    rng = np.random.default_rng(seed)
    out = rng.integers(0, 256, size=nblocks * rows * bl * wb, dtype=np.uint8)
    tail = nblocks * bl - n
    if tail:  # padding slots are all-ones (layout.hpp:117)
        last = out[(nblocks - 1) * rows * bl * wb:].reshape(rows, bl, wb)
        last[:, bl - tail:, :] = 0xFF
    return out
