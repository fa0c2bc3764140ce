"""Host-side mirror of the reference's search interface over the C ABI.

Names and argument meaning follow the reference (``pqscan``): ``allocate_dims`` /
``PqSpec`` (pqspec.hpp), ``SearchParams`` / ``SearchResult`` / ``FlatIndex`` / ``IvfIndex``
(index.hpp) and the ``QuantizedScanFn`` plugin point (simd/kernels.hpp:49-50).  All
computation happens in libqadc_b200.so's CUDA kernels; these classes only marshal
numpy / torch buffers.  Errors raise :class:`QadcError` whose ``kind`` is the reference's
exception class name (input / config / calibration / ...).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from .layout import pack_list
from ._lib import QadcError, QadcSearchParams, QadcSpec, QadcStats, check, lib

KERNEL_FAMILY = "b200-smem-lut"  # reported in SearchResult.kernel (the reference reports its SIMD family)


def _p(a, ctype):
    return a.ctypes.data_as(C.POINTER(ctype)) if a is not None else None


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def allocate_dims(total_dims: int, spec_string: str) -> QadcSpec:
    """parse_spec_string + allocate_dims + PackingScheme::for_spec (pqspec.hpp:24-55, 119-171)."""
    s = QadcSpec()
    check(lib().qadc_spec_parse(C.c_uint32(total_dims), spec_string.encode(), C.byref(s)))
    return s


def packed_bytes(spec: QadcSpec, n: int) -> int:
    return int(lib().qadc_packed_bytes(C.byref(spec), C.c_uint64(n)))


@dataclass
class SearchParams:
    """index.hpp:20-32.  ``fma_unquantize`` reproduces the reference's default -march=native build,
    which contracts ``q*delta + d_min`` into one FMA; off matches the pinned (-ffp-contract=off) oracle."""
    probes: int = 1
    r: int = 100
    t: int = 400
    fma_unquantize: bool = False
    rerank: bool = False  # exact re-ranking of the final top-R by float ADC (index.hpp:24)

    def c(self) -> QadcSearchParams:
        for name in ("probes", "r", "t"):
            v = getattr(self, name)
            if v < 0 or v > 0xFFFFFFFF:
                raise QadcError(5, f"search: {name} out of range")
        return QadcSearchParams(self.probes, self.r, self.t, (1 if self.fma_unquantize else 0) | (2 if self.rerank else 0))


@dataclass
class SearchResult:
    """index.hpp:34-39 for a batch: row q holds ``counts[q]`` valid entries, ascending (distance, id)."""
    ids: np.ndarray
    dists: np.ndarray
    counts: np.ndarray
    kernel: str = KERNEL_FAMILY
    scalar_fallback: bool = False

    def query(self, q: int):
        n = int(self.counts[q])
        return self.ids[q, :n], self.dists[q, :n]


class _Index:
    def __init__(self):
        self._h = C.c_void_p()
        self.spec: QadcSpec | None = None
        self.device = 0

    def close(self):
        if self._h:
            lib().qadc_close(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- search ---------------------------------------------------------------
    def search(self, queries, params: SearchParams | None = None) -> SearchResult:
        """FlatIndex::search / IvfIndex::search (index.hpp:110, 276) for a batch of host queries."""
        params = params or SearchParams()
        q = _f32(queries)
        if q.ndim == 1:
            q = q.reshape(1, -1)
        if q.ndim != 2 or q.shape[1] != self.spec.dims:
            raise QadcError(5, "search: query has wrong dimension")  # index.hpp:112
        nq, r = q.shape[0], max(int(params.r), 1)
        ids = np.empty((nq, r), dtype=np.uint32)
        dists = np.empty((nq, r), dtype=np.float32)
        counts = np.zeros(nq, dtype=np.uint32)
        cp = params.c()
        check(lib().qadc_search_batch(self._h, _p(q, C.c_float), C.c_uint32(nq), C.byref(cp), _p(ids, C.c_uint32),
                                      _p(dists, C.c_float), _p(counts, C.c_uint32)))
        return SearchResult(ids, dists, counts)

    def search_device(self, d_queries, params: SearchParams, d_ids, d_dists, d_counts, d_keys=None, d_map=None,
                      stream=None):
        """Device-buffer variant: arguments are torch CUDA tensors (float32 [nq,dims]; uint32-as-int32 / float32
        [nq,r]; int32 [nq]; optional int64 [nq,r] keys and float32 [nq,2] map).  Runs on ``stream`` (an int
        cudaStream_t, e.g. ``torch.cuda.current_stream().cuda_stream``)."""
        nq = int(d_queries.shape[0])
        if nq and int(d_queries.shape[1]) != self.spec.dims:
            raise QadcError(5, "search: query has wrong dimension")
        cp = params.c()
        ptr = lambda t: C.c_void_p(t.data_ptr()) if t is not None else None  # noqa: E731
        check(lib().qadc_search_batch_device(self._h, ptr(d_queries), C.c_uint32(nq), C.byref(cp), ptr(d_ids),
                                             ptr(d_dists), ptr(d_counts), ptr(d_keys), ptr(d_map),
                                             C.c_void_p(stream or 0)))

    def stats(self) -> QadcStats:
        st = QadcStats()
        check(lib().qadc_get_stats(self._h, C.byref(st)))
        return st

    def set_option(self, name: str, value: int):
        check(lib().qadc_set_option(self._h, name.encode(), C.c_int64(value)))


class FlatIndex(_Index):
    """FlatIndex (index.hpp:73-157): exhaustive search over one packed list.

    ``packed`` is the reference's PackedList byte stream (layout.hpp:135-160) for ``count`` codes.
    For a database shard pass ``base_id`` (id of the shard's first code) and ``calib_packed`` /
    ``calib_count`` (the PackedList of the first codes of the WHOLE list) so that every shard
    derives the same quantization map (index.hpp:124-129)."""

    def __init__(self, spec: QadcSpec, codebook, packed, count: int, base_id: int = 0, calib_packed=None,
                 calib_count: int = 0, device: int = 0, global_count: int = 0):
        super().__init__()
        self.spec = spec
        self.device = device
        self.count = int(count)
        cb = _f32(codebook).reshape(-1)
        if cb.size != spec.cb_floats:
            raise QadcError(5, "codebook: table count does not match spec")  # codebook.hpp:40
        pk = np.ascontiguousarray(packed, dtype=np.uint8).reshape(-1)
        if pk.size < packed_bytes(spec, count):
            raise QadcError(5, "packed list is shorter than its code count requires")
        cpk = None
        if calib_packed is not None:
            cpk = np.ascontiguousarray(calib_packed, dtype=np.uint8).reshape(-1)
            if cpk.size < packed_bytes(spec, calib_count):
                raise QadcError(5, "calibration list is shorter than its code count requires")
        check(lib().qadc_flat_open(C.byref(spec), _p(cb, C.c_float), _p(pk, C.c_uint8), C.c_uint64(count),
                                   C.c_uint32(base_id), _p(cpk, C.c_uint8), C.c_uint64(calib_count if cpk is not None else 0),
                                   C.c_uint64(global_count), C.c_int(device), C.byref(self._h)))

    def size(self) -> int:
        return self.count

    # -- parity / debug entry points -----------------------------------------------
    def tables(self, queries, params: SearchParams | None = None):
        """(float LUTs, quantized LUTs, calib{d_min,d_max,delta,own_d_min}) as the search derives them."""
        params = params or SearchParams()
        q = _f32(queries).reshape(-1, self.spec.dims)
        nq, E = q.shape[0], self.spec.total_entries
        luts = np.empty((nq, E), dtype=np.float32)
        qluts = np.empty((nq, E), dtype=np.uint8 if self.spec.word_width == 8 else np.uint16)
        calib = np.empty((nq, 4), dtype=np.float32)
        cp = params.c()
        check(lib().qadc_flat_tables(self._h, _p(q, C.c_float), C.c_uint32(nq), C.byref(cp), _p(luts, C.c_float),
                                     qluts.ctypes.data_as(C.c_void_p), _p(calib, C.c_float)))
        return luts, qluts, calib

    def adc_sums(self, qlut, first: int, n: int, acc_init: int = 0, width: int | None = None) -> np.ndarray:
        width = self.spec.word_width if width is None else width
        q = np.ascontiguousarray(qlut, dtype=np.uint8 if width == 8 else np.uint16)
        out = np.empty(n, dtype=np.uint32)
        check(lib().qadc_flat_adc_sums(self._h, q.ctypes.data_as(C.c_void_p), C.c_uint32(width), C.c_uint32(acc_init),
                                       C.c_uint64(first), C.c_uint64(n), _p(out, C.c_uint32)))
        return out

    def download_codes(self, first: int, n: int) -> np.ndarray:
        out = np.empty((n, self.spec.m), dtype=np.uint8)
        check(lib().qadc_flat_download_codes(self._h, C.c_uint64(first), C.c_uint64(n), _p(out, C.c_uint8)))
        return out


class MultiGpuFlatIndex:
    """One process, several GPUs: FlatIndex sharded over ``ndev`` devices behind one handle (qadc_flat_open_sharded):
    block-aligned shards with base ids, replicated calibration head, one NCCL all_gather + merge per batch."""

    def __init__(self, spec: QadcSpec, codebook, packed, count: int, ndev: int = 1, devices=None):
        self.spec, self.count, self._h = spec, int(count), C.c_void_p()
        cb = _f32(codebook).reshape(-1)
        if cb.size != spec.cb_floats:
            raise QadcError(5, "codebook: table count does not match spec")
        pk = np.ascontiguousarray(packed, dtype=np.uint8).reshape(-1)
        if pk.size < packed_bytes(spec, count):
            raise QadcError(5, "packed list is shorter than its code count requires")
        dv = None if devices is None else np.ascontiguousarray(devices, dtype=np.int32)
        check(lib().qadc_flat_open_sharded(C.byref(spec), _p(cb, C.c_float), _p(pk, C.c_uint8), C.c_uint64(count),
                                           C.c_int(ndev), _p(dv, C.c_int), C.byref(self._h)))

    def info(self):
        ndev, count, nccl = C.c_int(), C.c_uint64(), C.c_int()
        check(lib().qadc_multi_info(self._h, C.byref(ndev), C.byref(count), C.byref(nccl)))
        return dict(ndev=ndev.value, count=int(count.value), uses_nccl=bool(nccl.value))

    def search(self, queries, params: SearchParams | None = None) -> SearchResult:
        params = params or SearchParams()
        q = _f32(queries).reshape(-1, self.spec.dims)
        nq, r = q.shape[0], max(int(params.r), 1)
        ids = np.empty((nq, r), dtype=np.uint32)
        dists = np.empty((nq, r), dtype=np.float32)
        counts = np.zeros(nq, dtype=np.uint32)
        cp = params.c()
        check(lib().qadc_multi_search_batch(self._h, _p(q, C.c_float), C.c_uint32(nq), C.byref(cp), _p(ids, C.c_uint32),
                                            _p(dists, C.c_float), _p(counts, C.c_uint32)))
        return SearchResult(ids, dists, counts)

    def close(self):
        if self._h:
            lib().qadc_multi_close(self._h)
            self._h = C.c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


class MultiGpuIvfIndex(MultiGpuFlatIndex):
    """One process, several GPUs: IvfIndex with every list split over ``ndev`` devices behind one handle
    (qadc_ivf_open_sharded): replicated list heads, one NCCL all_gather + merge per batch."""

    def __init__(self, spec: QadcSpec, codebook, coarse, packed, list_byte_off, list_id_off, list_count, ids,
                 ndev: int = 1, devices=None):
        self.spec, self._h = spec, C.c_void_p()
        cb = _f32(codebook).reshape(-1)
        if cb.size != spec.cb_floats:
            raise QadcError(5, "codebook: table count does not match spec")
        co = _f32(coarse).reshape(-1, spec.dims)
        k = co.shape[0]
        pk = np.ascontiguousarray(packed, dtype=np.uint8).reshape(-1)
        boff = np.ascontiguousarray(list_byte_off, dtype=np.uint64)
        ioff = np.ascontiguousarray(list_id_off, dtype=np.uint64)
        cnt = np.ascontiguousarray(list_count, dtype=np.uint64)
        idv = np.ascontiguousarray(ids, dtype=np.uint32)
        if not (len(boff) == len(ioff) == len(cnt) == k):
            raise QadcError(5, "ivf: one offset / count per coarse centroid is required")
        self.count = int(cnt.sum())
        dv = None if devices is None else np.ascontiguousarray(devices, dtype=np.int32)
        check(lib().qadc_ivf_open_sharded(C.byref(spec), _p(cb, C.c_float), _p(co, C.c_float), C.c_uint32(k),
                                          _p(pk, C.c_uint8), _p(boff, C.c_uint64), _p(ioff, C.c_uint64), _p(cnt, C.c_uint64),
                                          _p(idv, C.c_uint32), C.c_int(ndev), _p(dv, C.c_int), C.byref(self._h)))

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class IvfIndex(_Index):
    """IvfIndex (index.hpp:166-177): coarse partition + per-cell packed lists of residual codes."""

    def __init__(self, spec: QadcSpec, codebook, coarse, packed, list_byte_off, list_id_off, list_count, ids,
                 device: int = 0, calib_packed=None, calib_byte_off=None, calib_count=None, global_list_count=None):
        """For a shard (every list split across ranks) pass ``calib_*``: the PackedLists of the first
        min(count, t_max) codes of the UNSHARDED lists, so that every rank derives the same quantization map,
        and ``global_list_count`` (lengths of the unsharded lists): a search whose t exceeds a truncated head
        is refused (config)."""
        super().__init__()
        self.spec = spec
        self.device = device
        cb = _f32(codebook).reshape(-1)
        if cb.size != spec.cb_floats:
            raise QadcError(5, "codebook: table count does not match spec")
        co = _f32(coarse).reshape(-1, spec.dims)
        self.k_cells = co.shape[0]
        pk = np.ascontiguousarray(packed, dtype=np.uint8).reshape(-1)
        lbo = np.ascontiguousarray(list_byte_off, dtype=np.uint64)
        lio = np.ascontiguousarray(list_id_off, dtype=np.uint64)
        lc = np.ascontiguousarray(list_count, dtype=np.uint64)
        idv = np.ascontiguousarray(ids, dtype=np.uint32)
        if not (lbo.size == lio.size == lc.size == self.k_cells):
            raise QadcError(6, "ivf: list/id section mismatch")  # index.hpp:173
        if int(lc.sum()) != idv.size:
            raise QadcError(6, "ivf: list code count != id count")  # index.hpp:175
        self.total = int(lc.sum())
        cpk = cbo = cc = glc = None
        if calib_packed is not None:
            cpk = np.ascontiguousarray(calib_packed, dtype=np.uint8).reshape(-1)
            cbo = np.ascontiguousarray(calib_byte_off, dtype=np.uint64)
            cc = np.ascontiguousarray(calib_count, dtype=np.uint64)
            if global_list_count is None:
                raise QadcError(5, "ivf: global_list_count is required with calibration heads")
            glc = np.ascontiguousarray(global_list_count, dtype=np.uint64)
            if not (cbo.size == cc.size == glc.size == self.k_cells):
                raise QadcError(6, "ivf: calibration head section mismatch")
        check(lib().qadc_ivf_open(C.byref(spec), _p(cb, C.c_float), _p(co, C.c_float), C.c_uint32(self.k_cells),
                                  _p(pk, C.c_uint8), _p(lbo, C.c_uint64), _p(lio, C.c_uint64), _p(lc, C.c_uint64),
                                  _p(idv, C.c_uint32), _p(cpk, C.c_uint8), _p(cbo, C.c_uint64), _p(cc, C.c_uint64),
                                  _p(glc, C.c_uint64), C.c_int(device), C.byref(self._h)))

    def size(self) -> int:
        return self.total

    def cells(self) -> int:
        return self.k_cells

    def probe_order(self, queries, a: int) -> np.ndarray:
        """IvfIndex::probe_order (index.hpp:247-265) for a batch."""
        q = _f32(queries).reshape(-1, self.spec.dims)
        a = min(a, self.k_cells)
        out = np.empty((q.shape[0], a), dtype=np.uint32)
        check(lib().qadc_ivf_probe_order(self._h, _p(q, C.c_float), C.c_uint32(q.shape[0]), C.c_uint32(a),
                                         _p(out, C.c_uint32)))
        return out


def open_index(path: str, device: int = 0):
    """load_flat_index / load_ivf_index (io.hpp:286-326) straight onto the GPU: opens a QFLT or QIVF container written
    by the reference and returns a :class:`FlatIndex` or :class:`IvfIndex`."""
    h = C.c_void_p()
    check(lib().qadc_open_file(str(path).encode(), C.c_int(device), C.byref(h)))
    kind, spec, count, cells = C.c_int(), QadcSpec(), C.c_uint64(), C.c_uint32()
    check(lib().qadc_index_info(h, C.byref(kind), C.byref(spec), C.byref(count), C.byref(cells)))
    obj = object.__new__(FlatIndex if kind.value == 0 else IvfIndex)
    _Index.__init__(obj)
    obj._h, obj.spec, obj.device = h, spec, device
    if kind.value == 0:
        obj.count = int(count.value)
    else:
        obj.total, obj.k_cells = int(count.value), int(cells.value)
    return obj


def scan_list(spec: QadcSpec, packed, count: int, qlut, *, rows=None, width=None, ids=None, base_id=0, acc_init=0,
              cap=100, heap_in=None, device=0):
    """The QuantizedScanFn contract (simd/kernels.hpp:49-50, scan_scalar.hpp:34-64) on the GPU.

    Scans one PackedList with caller-supplied quantized tables into a bounded heap that may be
    pre-seeded with ``heap_in`` [(dist, id), ...]; returns the heap's ``sorted()`` as (dists, ids)."""
    packed = np.ascontiguousarray(packed, dtype=np.uint8).reshape(-1)
    width = spec.word_width if width is None else width
    qlut = np.ascontiguousarray(qlut, dtype=np.uint8 if width == 8 else np.uint16)
    rows = spec.groups if rows is None else rows
    ids_a = None if ids is None else np.ascontiguousarray(ids, dtype=np.uint32)
    hd = hi = None
    n_in = 0
    if heap_in is not None and len(heap_in):
        hd = np.ascontiguousarray([d for d, _ in heap_in], dtype=np.uint32)
        hi = np.ascontiguousarray([i for _, i in heap_in], dtype=np.uint32)
        n_in = len(heap_in)
    od = np.empty(max(cap, 1), dtype=np.uint32)
    oi = np.empty(max(cap, 1), dtype=np.uint32)
    n_out = C.c_uint32(0)
    check(lib().qadc_scan_list(C.byref(spec), _p(packed, C.c_uint8), C.c_uint64(count), C.c_uint32(rows),
                               qlut.ctypes.data_as(C.c_void_p), C.c_uint32(width), _p(ids_a, C.c_uint32),
                               C.c_uint32(base_id), C.c_uint32(acc_init), C.c_uint32(cap), _p(hd, C.c_uint32),
                               _p(hi, C.c_uint32), C.c_uint32(n_in), _p(od, C.c_uint32), _p(oi, C.c_uint32),
                               C.byref(n_out), C.c_int(device)))
    return od[:n_out.value].copy(), oi[:n_out.value].copy()


def encode(spec: QadcSpec, codebook, vectors, device: int = 0) -> np.ndarray:
    """encode (codebook.hpp:94-118) on the GPU: nearest centroid per slice, double accumulators,
    ties toward the lowest index."""
    cb = _f32(codebook).reshape(-1)
    v = _f32(vectors).reshape(-1, spec.dims)
    out = np.empty((v.shape[0], spec.m), dtype=np.uint8)
    check(lib().qadc_encode(C.byref(spec), _p(cb, C.c_float), _p(v, C.c_float), C.c_uint64(v.shape[0]),
                            _p(out, C.c_uint8), C.c_int(device)))
    return out


def ivf_assign_encode(spec: QadcSpec, codebook, coarse, vectors, device: int = 0):
    """The data-dependent half of IvfIndex::build (index.hpp:195-227) on the GPU: nearest coarse centroid (double
    accumulator, ties to the lowest cell, kmeans.hpp:178-190), fp32 residual (index.hpp:200), residual encode.
    Returns (assign[n] u32, codes[n, m] u8)."""
    cb = _f32(codebook).reshape(-1)
    co = _f32(coarse).reshape(-1, spec.dims)
    v = _f32(vectors).reshape(-1, spec.dims)
    assign = np.empty(v.shape[0], dtype=np.uint32)
    codes = np.empty((v.shape[0], spec.m), dtype=np.uint8)
    check(lib().qadc_ivf_assign_encode(C.byref(spec), _p(cb, C.c_float), _p(co, C.c_float), C.c_uint32(co.shape[0]),
                                       _p(v, C.c_float), C.c_uint64(v.shape[0]), _p(assign, C.c_uint32),
                                       _p(codes, C.c_uint8), C.c_int(device)))
    return assign, codes


def build_ivf_lists(spec: QadcSpec, codebook, coarse, vectors, device: int = 0) -> dict:
    """IVF lists for `vectors` under trained `coarse` centroids and a residual `codebook`, laid out as
    IvfIndex::build does (index.hpp:219-227): each cell's members in ascending vector index, one PackedList per
    cell, ids = vector indices.  Everything runs on the GPU behind the C ABI (qadc_ivf_build_lists): assignment,
    residuals, encode, a stable grouping by cell and the packing into the reference's transposed blocks.  The dict's
    keys are IvfIndex's constructor arguments (+ ``assign``)."""
    cb = _f32(codebook).reshape(-1)
    co = _f32(coarse).reshape(-1, spec.dims)
    v = _f32(vectors).reshape(-1, spec.dims)
    n, k_cells = v.shape[0], co.shape[0]
    L = lib()
    L.qadc_ivf_build_packed_bound.restype = C.c_uint64
    cap = int(L.qadc_ivf_build_packed_bound(C.byref(spec), C.c_uint64(n), C.c_uint32(k_cells)))
    counts = np.zeros(k_cells, dtype=np.uint64)
    byte_off = np.zeros(k_cells, dtype=np.uint64)
    id_off = np.zeros(k_cells, dtype=np.uint64)
    ids = np.zeros(n, dtype=np.uint32)
    assign = np.zeros(n, dtype=np.uint32)
    packed = np.zeros(max(cap, 1), dtype=np.uint8)
    nbytes = C.c_uint64(0)
    check(L.qadc_ivf_build_lists(C.byref(spec), _p(cb, C.c_float), _p(co, C.c_float), C.c_uint32(k_cells),
                                 _p(v, C.c_float), C.c_uint64(n), _p(counts, C.c_uint64), _p(byte_off, C.c_uint64),
                                 _p(id_off, C.c_uint64), _p(ids, C.c_uint32), _p(packed, C.c_uint8), C.c_uint64(cap),
                                 C.byref(nbytes), _p(assign, C.c_uint32), C.c_int(device)))
    return dict(packed=packed[: nbytes.value].copy(), list_byte_off=byte_off, list_id_off=id_off, list_count=counts,
                ids=ids, assign=assign)


def merge_topk_device(d_keys, nshards: int, nq: int, r: int, d_map, d_ids, d_dists, d_counts, device: int,
                      fma_unquantize=False, stream=None):
    """Multi-GPU exchange step: merge gathered per-shard key lists [nshards, nq, r] (torch CUDA tensors)."""
    ptr = lambda t: C.c_void_p(t.data_ptr()) if t is not None else None  # noqa: E731
    check(lib().qadc_merge_topk_device(ptr(d_keys), C.c_uint32(nshards), C.c_uint32(nq), C.c_uint32(r), ptr(d_map),
                                       C.c_uint32(1 if fma_unquantize else 0), ptr(d_ids), ptr(d_dists),
                                       ptr(d_counts), C.c_int(device), C.c_void_p(stream or 0)))
