"""ctypes front-end for the CPU oracle (TEST INFRASTRUCTURE ONLY).

Two interchangeable libraries export the same ``orc_*`` C API (qadc_oracle.h):

* ``port``      -- oracle/_build/libqadc_oracle.so, the plain-C restatement
                   (oracle/qadc_oracle.c);
* ``reference`` -- oracle/_ref/libpqscan_ref.so, a shim that calls the
                   unmodified reference headers (oracle/ref_shim.cpp).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` legs may import this module.  Nothing here reads
/root/reference at run time.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
PORT_SO = HERE / "_build" / "libqadc_oracle.so"
REF_SO = HERE / "_ref" / "libpqscan_ref.so"

ORC_MAX_SUBS = 64
ORC_MAX_GROUP = 16

ERR_NAMES = {3: "invalid_spec", 4: "training", 5: "input", 6: "corruption", 7: "config", 8: "io", 9: "calibration"}


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{ERR_NAMES.get(code, code)}] {msg}")
        self.code = code
        self.kind = ERR_NAMES.get(code, str(code))


class OrcSpec(C.Structure):
    _fields_ = [
        ("dims", C.c_uint32),
        ("m", C.c_uint32),
        ("g", C.c_uint32),
        ("groups", C.c_uint32),
        ("word_width", C.c_uint32),
        ("block_len", C.c_uint32),
        ("exact", C.c_uint32),
        ("total_entries", C.c_uint32),
        ("cb_floats", C.c_uint32),
        ("widths", C.c_uint8 * ORC_MAX_GROUP),
        ("offsets", C.c_uint8 * ORC_MAX_GROUP),
        ("bits", C.c_uint8 * ORC_MAX_SUBS),
        ("dim_alloc", C.c_uint32 * ORC_MAX_SUBS),
        ("dim_off", C.c_uint32 * ORC_MAX_SUBS),
        ("ent_off", C.c_uint32 * ORC_MAX_SUBS),
        ("cb_off", C.c_uint32 * ORC_MAX_SUBS),
    ]

    # convenience views
    @property
    def q_max(self) -> int:
        return 255 if self.word_width == 8 else 65535

    @property
    def qdtype(self):
        return np.uint8 if self.word_width == 8 else np.uint16

    def bits_list(self):
        return [int(self.bits[j]) for j in range(self.m)]

    def dim_alloc_list(self):
        return [int(self.dim_alloc[j]) for j in range(self.m)]


def build(force: bool = False) -> None:
    """Compile the port (always possible) and, when /root/reference is present, the reference shim."""
    if force or not PORT_SO.exists() or PORT_SO.stat().st_mtime < (HERE / "qadc_oracle.c").stat().st_mtime:
        subprocess.check_call(["make", "-C", str(HERE), "port"], stdout=subprocess.DEVNULL)
    ref_inc = Path(os.environ.get("QADC_REFERENCE_INCLUDE", "/root/reference/proj/include"))
    if (ref_inc / "pqscan").is_dir():
        if force or not REF_SO.exists() or REF_SO.stat().st_mtime < (HERE / "ref_shim.cpp").stat().st_mtime:
            subprocess.check_call(["make", "-C", str(HERE), "ref", f"REF={ref_inc}"], stdout=subprocess.DEVNULL)
        # the C++ integration test (reference types -> include/qadc.hpp -> libqadc_b200.so); make skips it
        # quietly when the product library has not been built yet
        subprocess.check_call(["make", "-C", str(HERE), "integration", f"REF={ref_inc}"], stdout=subprocess.DEVNULL)


def _p(a, ctype):
    return a.ctypes.data_as(C.POINTER(ctype)) if a is not None else None


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


class Oracle:
    """Thin numpy wrapper over one of the two oracle libraries."""

    def __init__(self, kind: str = "port"):
        path = PORT_SO if kind == "port" else REF_SO
        if not path.exists():
            build()
        if not path.exists():
            raise FileNotFoundError(f"oracle library {path} is not built")
        self.kind = kind
        self.lib = C.CDLL(str(path))
        L = self.lib
        L.orc_impl_name.restype = C.c_char_p
        L.orc_last_error.restype = C.c_char_p
        L.orc_packed_bytes.restype = C.c_uint64
        L.orc_packed_bytes.argtypes = [C.POINTER(OrcSpec), C.c_uint64]
        L.orc_min_total.restype = C.c_float
        L.orc_prefix_float.restype = C.c_uint64
        if kind == "reference":
            L.ref_auto_family.restype = C.c_char_p
            L.ref_simd_caps.restype = C.c_char_p
        assert L.orc_impl_name().decode() == kind

    # -- helpers ---------------------------------------------------------
    def _check(self, rc: int):
        if rc != 0:
            raise OracleError(rc, self.lib.orc_last_error().decode())

    @staticmethod
    def available(kind: str) -> bool:
        return (PORT_SO if kind == "port" else REF_SO).exists()

    # -- spec / layout -----------------------------------------------------
    def spec(self, dims: int, text: str) -> OrcSpec:
        s = OrcSpec()
        self._check(self.lib.orc_spec_parse(C.c_uint32(dims), text.encode(), C.byref(s)))
        return s

    def packed_bytes(self, s: OrcSpec, n: int) -> int:
        return int(self.lib.orc_packed_bytes(C.byref(s), C.c_uint64(n)))

    def pack_list(self, s: OrcSpec, codes: np.ndarray) -> np.ndarray:
        codes = np.ascontiguousarray(codes, dtype=np.uint8).reshape(-1, s.m)
        n = codes.shape[0]
        out = np.empty(self.packed_bytes(s, n), dtype=np.uint8)
        self._check(self.lib.orc_pack_list(C.byref(s), _p(codes, C.c_uint8), C.c_uint64(n), _p(out, C.c_uint8)))
        return out

    def unpack_list(self, s: OrcSpec, packed: np.ndarray, n: int) -> np.ndarray:
        packed = np.ascontiguousarray(packed, dtype=np.uint8)
        out = np.empty((n, s.m), dtype=np.uint8)
        self._check(self.lib.orc_unpack_list(C.byref(s), _p(packed, C.c_uint8), C.c_uint64(n), _p(out, C.c_uint8)))
        return out

    def encode(self, s: OrcSpec, codebook: np.ndarray, vectors: np.ndarray) -> np.ndarray:
        cb, v = _f32(codebook), _f32(vectors).reshape(-1, s.dims)
        out = np.empty((v.shape[0], s.m), dtype=np.uint8)
        self._check(self.lib.orc_encode(C.byref(s), _p(cb, C.c_float), _p(v, C.c_float), C.c_uint64(v.shape[0]),
                                        _p(out, C.c_uint8)))
        return out

    def ivf_assign_encode(self, s: OrcSpec, codebook, coarse, vectors):
        cb, co, v = _f32(codebook), _f32(coarse).reshape(-1, s.dims), _f32(vectors).reshape(-1, s.dims)
        assign = np.empty(v.shape[0], dtype=np.uint32)
        codes = np.empty((v.shape[0], s.m), dtype=np.uint8)
        self._check(self.lib.orc_ivf_assign_encode(C.byref(s), _p(cb, C.c_float), _p(co, C.c_float),
                                                   C.c_uint32(co.shape[0]), _p(v, C.c_float), C.c_uint64(v.shape[0]),
                                                   _p(assign, C.c_uint32), _p(codes, C.c_uint8)))
        return assign, codes

    # -- tables ------------------------------------------------------------
    def compute_tables(self, s: OrcSpec, codebook: np.ndarray, query: np.ndarray) -> np.ndarray:
        cb, q = _f32(codebook), _f32(query)
        if q.size != s.dims:
            raise OracleError(5, "compute_tables: query has wrong dimension")
        out = np.empty(s.total_entries, dtype=np.float32)
        self._check(self.lib.orc_compute_tables(C.byref(s), _p(cb, C.c_float), _p(q, C.c_float), _p(out, C.c_float)))
        return out

    def min_total(self, s: OrcSpec, lut: np.ndarray):
        lut = _f32(lut)
        pm = np.empty(s.m, dtype=np.float32)
        tot = self.lib.orc_min_total(C.byref(s), _p(lut, C.c_float), _p(pm, C.c_float))
        return np.float32(tot), pm

    def prefix_float(self, s: OrcSpec, packed: np.ndarray, count: int, lut: np.ndarray, limit: int) -> np.ndarray:
        packed, lut = np.ascontiguousarray(packed, dtype=np.uint8), _f32(lut)
        out = np.empty(max(1, min(limit, count)), dtype=np.float32)
        n = self.lib.orc_prefix_float(C.byref(s), _p(packed, C.c_uint8), C.c_uint64(count), _p(lut, C.c_float),
                                      C.c_uint64(limit), _p(out, C.c_float))
        return out[:n]

    def calibrate(self, s: OrcSpec, lut: np.ndarray, prefix: np.ndarray, r: int):
        lut, prefix = _f32(lut), _f32(prefix)
        dmin, dmax = C.c_float(), C.c_float()
        self._check(self.lib.orc_calibrate(C.byref(s), _p(lut, C.c_float), _p(prefix, C.c_float),
                                           C.c_uint64(prefix.size), C.c_uint32(r), C.byref(dmin), C.byref(dmax)))
        return np.float32(dmin.value), np.float32(dmax.value)

    def quantize(self, s: OrcSpec, lut: np.ndarray, d_min, d_max, width: int):
        lut = _f32(lut)
        q = np.empty(s.total_entries, dtype=np.uint8 if width == 8 else np.uint16)
        pm = np.empty(s.m, dtype=np.float32)
        delta, own = C.c_float(), C.c_float()
        self._check(self.lib.orc_quantize(C.byref(s), _p(lut, C.c_float), C.c_float(float(d_min)),
                                          C.c_float(float(d_max)), C.c_uint32(width), q.ctypes.data_as(C.c_void_p),
                                          _p(pm, C.c_float), C.byref(delta), C.byref(own)))
        return q, pm, np.float32(delta.value), np.float32(own.value)

    # -- scan ----------------------------------------------------------------
    def scan_quantized(self, s: OrcSpec, packed, count: int, qlut, *, rows=None, width=None, ids=None, base_id=0,
                       acc_init=0, cap=100, heap_in=None, family=0):
        packed = np.ascontiguousarray(packed, dtype=np.uint8)
        width = s.word_width if width is None else width
        qlut = np.ascontiguousarray(qlut, dtype=np.uint8 if width == 8 else np.uint16)
        rows = s.groups if rows is None else rows
        ids_a = None if ids is None else np.ascontiguousarray(ids, dtype=np.uint32)
        hin_d = hin_i = None
        n_in = 0
        if heap_in is not None and len(heap_in):
            hin_d = np.ascontiguousarray([d for d, _ in heap_in], dtype=np.uint32)
            hin_i = np.ascontiguousarray([i for _, i in heap_in], dtype=np.uint32)
            n_in = len(heap_in)
        od = np.empty(max(cap, 1), dtype=np.uint32)
        oi = np.empty(max(cap, 1), dtype=np.uint32)
        n_out = C.c_uint32(0)
        self._check(self.lib.orc_scan_quantized(
            C.byref(s), _p(packed, C.c_uint8), C.c_uint64(count), C.c_uint32(rows), qlut.ctypes.data_as(C.c_void_p),
            C.c_uint32(width), _p(ids_a, C.c_uint32), C.c_uint32(base_id), C.c_uint32(acc_init), C.c_uint32(cap),
            _p(hin_d, C.c_uint32), _p(hin_i, C.c_uint32), C.c_uint32(n_in), _p(od, C.c_uint32), _p(oi, C.c_uint32),
            C.byref(n_out), C.c_int(family)))
        return od[:n_out.value].copy(), oi[:n_out.value].copy()

    def adc_sums(self, s: OrcSpec, packed, count: int, qlut, first: int, n: int, acc_init=0, width=None):
        packed = np.ascontiguousarray(packed, dtype=np.uint8)
        width = s.word_width if width is None else width
        qlut = np.ascontiguousarray(qlut, dtype=np.uint8 if width == 8 else np.uint16)
        out = np.empty(n, dtype=np.uint32)
        self._check(self.lib.orc_adc_sums(C.byref(s), _p(packed, C.c_uint8), C.c_uint64(count),
                                          qlut.ctypes.data_as(C.c_void_p), C.c_uint32(width), C.c_uint32(acc_init),
                                          C.c_uint64(first), C.c_uint64(n), _p(out, C.c_uint32)))
        return out

    # -- search ----------------------------------------------------------------
    def flat_search(self, s: OrcSpec, codebook, packed, count: int, queries, r=100, t=400, family=0, threads=1,
                    debug=False):
        cb, q = _f32(codebook), _f32(queries).reshape(-1, s.dims)
        packed = np.ascontiguousarray(packed, dtype=np.uint8)
        nq = q.shape[0]
        ids = np.zeros((nq, r), dtype=np.uint32)
        dists = np.zeros((nq, r), dtype=np.float32)
        counts = np.zeros(nq, dtype=np.uint32)
        qlut = params = None
        if debug:
            qlut = np.zeros((nq, s.total_entries), dtype=s.qdtype)
            params = np.zeros((nq, 4), dtype=np.float32)
        self._check(self.lib.orc_flat_search(
            C.byref(s), _p(cb, C.c_float), _p(packed, C.c_uint8), C.c_uint64(count), _p(q, C.c_float),
            C.c_uint32(nq), C.c_uint32(r), C.c_uint32(t), C.c_int(family), C.c_int(threads), _p(ids, C.c_uint32),
            _p(dists, C.c_float), _p(counts, C.c_uint32),
            qlut.ctypes.data_as(C.c_void_p) if debug else None, _p(params, C.c_float)))
        if debug:
            return ids, dists, counts, qlut, params
        return ids, dists, counts

    def probe_order(self, dims: int, coarse, query, a: int) -> np.ndarray:
        coarse, query = _f32(coarse).reshape(-1, dims), _f32(query)
        k = coarse.shape[0]
        out = np.empty(min(a, k), dtype=np.uint32)
        self._check(self.lib.orc_probe_order(C.c_uint32(dims), _p(coarse, C.c_float), C.c_uint32(k),
                                             _p(query, C.c_float), C.c_uint32(a), _p(out, C.c_uint32)))
        return out

    def ivf_search(self, s: OrcSpec, codebook, coarse, packed, list_byte_off, list_id_off, list_count, ids, queries,
                   probes=1, r=100, t=400, family=0, threads=1):
        cb, q = _f32(codebook), _f32(queries).reshape(-1, s.dims)
        coarse = _f32(coarse).reshape(-1, s.dims)
        packed = np.ascontiguousarray(packed, dtype=np.uint8)
        lbo = np.ascontiguousarray(list_byte_off, dtype=np.uint64)
        lio = np.ascontiguousarray(list_id_off, dtype=np.uint64)
        lc = np.ascontiguousarray(list_count, dtype=np.uint64)
        ids_a = np.ascontiguousarray(ids, dtype=np.uint32)
        nq = q.shape[0]
        out_ids = np.zeros((nq, r), dtype=np.uint32)
        out_d = np.zeros((nq, r), dtype=np.float32)
        counts = np.zeros(nq, dtype=np.uint32)
        self._check(self.lib.orc_ivf_search(
            C.byref(s), _p(cb, C.c_float), _p(coarse, C.c_float), C.c_uint32(coarse.shape[0]), _p(packed, C.c_uint8),
            _p(lbo, C.c_uint64), _p(lio, C.c_uint64), _p(lc, C.c_uint64), _p(ids_a, C.c_uint32), _p(q, C.c_float),
            C.c_uint32(nq), C.c_uint32(probes), C.c_uint32(r), C.c_uint32(t), C.c_int(family), C.c_int(threads),
            _p(out_ids, C.c_uint32), _p(out_d, C.c_float), _p(counts, C.c_uint32)))
        return out_ids, out_d, counts

    # -- handle-based search (index built once; used by bench.py's CPU baseline) ----------------
    def flat_open(self, s: OrcSpec, codebook, packed, count: int):
        self.lib.orc_flat_create.restype = C.c_void_p
        keep = (_f32(codebook), np.ascontiguousarray(packed, dtype=np.uint8))
        h = self.lib.orc_flat_create(C.byref(s), _p(keep[0], C.c_float), _p(keep[1], C.c_uint8), C.c_uint64(count))
        if not h:
            raise OracleError(1, self.lib.orc_last_error().decode())
        return {"h": C.c_void_p(h), "keep": keep, "dims": s.dims, "ivf": False}

    def ivf_open(self, s: OrcSpec, codebook, coarse, packed, list_byte_off, list_id_off, list_count, ids):
        self.lib.orc_ivf_create.restype = C.c_void_p
        keep = (_f32(codebook), _f32(coarse).reshape(-1, s.dims), np.ascontiguousarray(packed, dtype=np.uint8),
                np.ascontiguousarray(list_byte_off, dtype=np.uint64), np.ascontiguousarray(list_id_off, dtype=np.uint64),
                np.ascontiguousarray(list_count, dtype=np.uint64), np.ascontiguousarray(ids, dtype=np.uint32))
        h = self.lib.orc_ivf_create(C.byref(s), _p(keep[0], C.c_float), _p(keep[1], C.c_float),
                                    C.c_uint32(keep[1].shape[0]), _p(keep[2], C.c_uint8), _p(keep[3], C.c_uint64),
                                    _p(keep[4], C.c_uint64), _p(keep[5], C.c_uint64), _p(keep[6], C.c_uint32))
        if not h:
            raise OracleError(1, self.lib.orc_last_error().decode())
        return {"h": C.c_void_p(h), "keep": keep, "dims": s.dims, "ivf": True}

    def search_h(self, handle, queries, probes=1, r=100, t=400, family=0, threads=1):
        q = _f32(queries).reshape(-1, handle["dims"])
        nq = q.shape[0]
        ids = np.zeros((nq, r), dtype=np.uint32)
        dists = np.zeros((nq, r), dtype=np.float32)
        counts = np.zeros(nq, dtype=np.uint32)
        if handle["ivf"]:
            rc = self.lib.orc_ivf_search_h(handle["h"], _p(q, C.c_float), C.c_uint32(nq), C.c_uint32(probes),
                                           C.c_uint32(r), C.c_uint32(t), C.c_int(family), C.c_int(threads),
                                           _p(ids, C.c_uint32), _p(dists, C.c_float), _p(counts, C.c_uint32))
        else:
            rc = self.lib.orc_flat_search_h(handle["h"], _p(q, C.c_float), C.c_uint32(nq), C.c_uint32(r), C.c_uint32(t),
                                            C.c_int(family), C.c_int(threads), _p(ids, C.c_uint32),
                                            _p(dists, C.c_float), _p(counts, C.c_uint32))
        self._check(rc)
        return ids, dists, counts

    def close_h(self, handle):
        (self.lib.orc_ivf_destroy if handle["ivf"] else self.lib.orc_flat_destroy)(handle["h"])

    # -- reference-only helpers ---------------------------------------------
    def train_codebook(self, s: OrcSpec, vectors, iters=25, seed=0) -> np.ndarray:
        assert self.kind == "reference"
        v = _f32(vectors).reshape(-1, s.dims)
        out = np.empty(s.cb_floats, dtype=np.float32)
        self._check(self.lib.ref_train_codebook(C.byref(s), _p(v, C.c_float), C.c_uint64(v.shape[0]),
                                                C.c_uint32(iters), C.c_uint64(seed), _p(out, C.c_float)))
        return out

    def kmeans(self, points, k: int, iters=25, seed=0):
        assert self.kind == "reference"
        p = _f32(points)
        n, dim = p.shape
        cent = np.empty((k, dim), dtype=np.float32)
        asg = np.empty(n, dtype=np.uint32)
        self._check(self.lib.ref_kmeans(_p(p, C.c_float), C.c_uint64(n), C.c_uint32(dim), C.c_uint32(k),
                                        C.c_uint32(iters), C.c_uint64(seed), _p(cent, C.c_float),
                                        _p(asg, C.c_uint32)))
        return cent, asg

    def ivf_build(self, vectors, spec_text: str, k_coarse: int, iters=8, seed=0):
        """The reference's IvfIndex::build (index.hpp:179-230) -> dict of its codebook, centroids, lists and ids."""
        assert self.kind == "reference"
        v = _f32(vectors)
        n, dims = v.shape
        self.lib.ref_ivf_build.restype = C.c_void_p
        h = self.lib.ref_ivf_build(_p(v, C.c_float), C.c_uint64(n), C.c_uint32(dims), spec_text.encode(),
                                   C.c_uint32(k_coarse), C.c_uint32(iters), C.c_uint64(seed))
        if not h:
            raise OracleError(1, self.lib.orc_last_error().decode())
        h = C.c_void_p(h)
        sizes = np.zeros(3, dtype=np.uint64)
        self.lib.ref_ivf_built_sizes(h, _p(sizes, C.c_uint64))
        out = dict(codebook=np.empty(int(sizes[0]), np.float32), coarse=np.empty((k_coarse, dims), np.float32),
                   packed=np.empty(int(sizes[1]), np.uint8), list_byte_off=np.empty(k_coarse, np.uint64),
                   list_id_off=np.empty(k_coarse, np.uint64), list_count=np.empty(k_coarse, np.uint64),
                   ids=np.empty(int(sizes[2]), np.uint32))
        self.lib.ref_ivf_built_get(h, _p(out["codebook"], C.c_float), _p(out["coarse"], C.c_float),
                                   _p(out["packed"], C.c_uint8), _p(out["list_byte_off"], C.c_uint64),
                                   _p(out["list_id_off"], C.c_uint64), _p(out["list_count"], C.c_uint64),
                                   _p(out["ids"], C.c_uint32))
        self.lib.ref_ivf_built_free(h)
        return out

    def save_flat(self, s: OrcSpec, codebook, packed, count: int, path: str):
        assert self.kind == "reference"
        cb, pk = _f32(codebook), np.ascontiguousarray(packed, dtype=np.uint8)
        self._check(self.lib.ref_save_flat(C.byref(s), _p(cb, C.c_float), _p(pk, C.c_uint8), C.c_uint64(count),
                                           str(path).encode()))

    def save_ivf(self, s: OrcSpec, codebook, coarse, packed, list_byte_off, list_id_off, list_count, ids, path: str):
        assert self.kind == "reference"
        cb, co = _f32(codebook), _f32(coarse).reshape(-1, s.dims)
        pk = np.ascontiguousarray(packed, dtype=np.uint8)
        lbo, lio = np.ascontiguousarray(list_byte_off, dtype=np.uint64), np.ascontiguousarray(list_id_off, dtype=np.uint64)
        lc, idv = np.ascontiguousarray(list_count, dtype=np.uint64), np.ascontiguousarray(ids, dtype=np.uint32)
        self._check(self.lib.ref_save_ivf(C.byref(s), _p(cb, C.c_float), _p(co, C.c_float), C.c_uint32(co.shape[0]),
                                          _p(pk, C.c_uint8), _p(lbo, C.c_uint64), _p(lio, C.c_uint64), _p(lc, C.c_uint64),
                                          _p(idv, C.c_uint32), str(path).encode()))

    def auto_family(self, s: OrcSpec) -> str:
        assert self.kind == "reference"
        return self.lib.ref_auto_family(C.byref(s)).decode()

    def simd_caps(self) -> str:
        assert self.kind == "reference"
        return self.lib.ref_simd_caps().decode()
