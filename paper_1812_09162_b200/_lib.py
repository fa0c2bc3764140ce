"""ctypes loader for libqadc_b200.so (the C ABI declared in include/qadc.h).

The shared library is built in-tree by ``paper_1812_09162_b200/csrc/Makefile`` (nvcc, sm_100a).
Loading never falls back to anything else: a missing library raises, and every compute
entry point fails with QADC_ERR_CUDA when no CUDA device is usable.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
SO_PATH = Path(os.environ.get("QADC_LIB_PATH", PKG / "libqadc_b200.so"))  # override: A/B runs of two builds
HEADER = ROOT / "include" / "qadc.h"

QADC_MAX_SUBS = 64
QADC_MAX_GROUP = 16
QADC_MAX_R = 16384

ERR_KINDS = {3: "invalid_spec", 4: "training", 5: "input", 6: "corruption", 7: "config", 8: "io", 9: "calibration",
             20: "cuda"}


class QadcError(RuntimeError):
    """Mirror of the reference's exception taxonomy (errors.hpp:9-46) keyed by the ABI status class."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"[{ERR_KINDS.get(code, code)}] {msg}")
        self.code = code
        self.kind = ERR_KINDS.get(code, str(code))


class QadcSpec(C.Structure):
    _fields_ = [
        ("dims", C.c_uint32), ("m", C.c_uint32), ("g", C.c_uint32), ("groups", C.c_uint32),
        ("word_width", C.c_uint32), ("block_len", C.c_uint32), ("exact", C.c_uint32),
        ("total_entries", C.c_uint32), ("cb_floats", C.c_uint32),
        ("widths", C.c_uint8 * QADC_MAX_GROUP), ("offsets", C.c_uint8 * QADC_MAX_GROUP),
        ("bits", C.c_uint8 * QADC_MAX_SUBS), ("dim_alloc", C.c_uint32 * QADC_MAX_SUBS),
        ("dim_off", C.c_uint32 * QADC_MAX_SUBS), ("ent_off", C.c_uint32 * QADC_MAX_SUBS),
        ("cb_off", C.c_uint32 * QADC_MAX_SUBS),
    ]

    @property
    def q_max(self) -> int:
        return 255 if self.word_width == 8 else 65535

    def bits_list(self):
        return [int(self.bits[j]) for j in range(self.m)]

    def dim_alloc_list(self):
        return [int(self.dim_alloc[j]) for j in range(self.m)]


class QadcSearchParams(C.Structure):
    _fields_ = [("probes", C.c_uint32), ("r", C.c_uint32), ("t", C.c_uint32), ("flags", C.c_uint32)]


class QadcStats(C.Structure):
    _fields_ = [
        ("kernel_launches", C.c_uint64), ("scan_launches", C.c_uint64), ("pairs_scanned", C.c_uint64),
        ("candidates", C.c_uint64), ("overflow_retries", C.c_uint64), ("segments", C.c_uint64),
        ("scan_variant", C.c_uint32), ("query_tile", C.c_uint32),
        ("ms_lut", C.c_float), ("ms_scan", C.c_float), ("ms_select", C.c_float),
    ]


def build(force: bool = False, verbose: bool = False) -> Path:
    """Compile every CUDA source for sm_100a into the in-tree shared library."""
    srcs = list((PKG / "csrc").glob("*.cu")) + list((PKG / "csrc").glob("*.cuh")) + [HEADER]
    stale = force or not SO_PATH.exists() or any(s.stat().st_mtime > SO_PATH.stat().st_mtime for s in srcs)
    if stale:
        cmd = ["make", "-C", str(PKG / "csrc"), "-j8"]
        subprocess.check_call(cmd, stdout=None if verbose else subprocess.DEVNULL)
    return SO_PATH


_LIB = None


def lib() -> C.CDLL:
    global _LIB
    if _LIB is None:
        if not SO_PATH.exists():
            raise FileNotFoundError(
                f"{SO_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                "(there is no fallback implementation)")
        L = C.CDLL(str(SO_PATH))
        L.qadc_version.restype = C.c_char_p
        L.qadc_last_error.restype = C.c_char_p
        L.qadc_variant_name.restype = C.c_char_p
        L.qadc_variant_name.argtypes = [C.c_uint32]
        L.qadc_packed_bytes.restype = C.c_uint64
        L.qadc_packed_bytes.argtypes = [C.POINTER(QadcSpec), C.c_uint64]
        L.qadc_close.restype = None
        L.qadc_close.argtypes = [C.c_void_p]
        L.qadc_multi_close.restype = None
        L.qadc_multi_close.argtypes = [C.c_void_p]
        _LIB = L
    return _LIB


def check(rc: int) -> None:
    if rc != 0:
        raise QadcError(rc, lib().qadc_last_error().decode(errors="replace"))


def exported_symbols_declared_in_header() -> list[str]:
    """Every function name declared in include/qadc.h (used by the ABI export test)."""
    import re
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(qadc_[a-z0-9_]+)\s*\(", text)))
