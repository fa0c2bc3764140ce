"""Pins the CPU oracle (oracle/qadc_oracle.c) before anything trusts it.

(a) known-answer vectors held inline by the reference's own tests (cited file:line under
    /root/reference/proj/tests), (b) golden fixtures produced by the unmodified reference
    (oracle/make_golden.py -> tests/golden/), (c) live differential runs against oracle/_ref
    when it is present.  Bit-exact everywhere (integer/byte work; float LUTs compare bitwise
    because both builds pin -ffp-contract=off).
"""
import numpy as np
import pytest

from oracle.pyoracle import OracleError

FLAT = ["flat_pq16x4.npz", "flat_irr655.npz", "flat_irr664.npz", "flat_irr555.npz", "flat_split88.npz",
        "flat_split8.npz", "flat_pq16x4_short.npz", "flat_irr655_short.npz"]
IVF = ["ivf_irr655.npz", "ivf_pq16x4.npz"]


# ---------------------------------------------------------------- (a) KATs --

def test_kat_block_len_and_word_width(port):
    # T/test_layout.cpp:18-26
    for dims, text, bl, ww in [(128, "16x{4,4}", 16, 8), (128, "12x{6,6,4}", 32, 16), (120, "12x{5,5,5}", 32, 16),
                               (128, "8x{8,8}", 32, 16), (128, "8x{8}", 64, 8)]:
        s = port.spec(dims, text)
        assert (s.block_len, s.word_width) == (bl, ww)


def test_kat_pack_bit_order(port):
    # T/test_layout.cpp:28-39: (0xA,0x3) -> 0x3A ; 0xFFFF -> (63,63,15) ; zeros -> 0x0000
    s44 = port.spec(8, "2x{4,4}")
    pk = port.pack_list(s44, np.array([[0xA, 0x3]], np.uint8))
    assert pk[0] == 0x3A and np.all(pk[1:] == 0xFF)  # padding is all-ones (T/test_layout.cpp:96-98)
    s664 = port.spec(16, "3x{6,6,4}")
    pk = port.pack_list(s664, np.array([[0, 0, 0]], np.uint8))
    assert pk[0] == 0 and pk[1] == 0
    ones = np.full(port.packed_bytes(s664, 1), 0xFF, np.uint8)
    assert port.unpack_list(s664, ones, 1).tolist() == [[63, 63, 15]]


def test_kat_pack_overflow_is_corruption(port):
    # T/test_layout.cpp:41-45
    s44 = port.spec(8, "2x{4,4}")
    with pytest.raises(OracleError) as e:
        port.pack_list(s44, np.array([[0x10, 0x3]], np.uint8))
    assert e.value.kind == "corruption"


@pytest.mark.parametrize("n", [0, 1, 15, 16, 17, 100])
def test_kat_pack_list_sizes(port, n):
    # T/test_layout.cpp:151-163
    s = port.spec(128, "16x{4,4}")
    assert port.packed_bytes(s, n) == ((n + 15) // 16) * 8 * 16
    s = port.spec(96, "12x{6,5,5}")
    assert port.packed_bytes(s, n) == ((n + 31) // 32) * 4 * 32 * 2


def test_kat_spec_allocation_examples(port):
    # T/test_pqspec.cpp:39-91: 128 / 12x{6,6,4} -> 12,12,8 ; 96 -> 9,9,6
    assert port.spec(128, "12x{6,6,4}").dim_alloc_list()[:3] == [12, 12, 8]
    assert port.spec(96, "12x{6,6,4}").dim_alloc_list()[:3] == [9, 9, 6]
    # SURVEY.md section 0.6 probes of allocate_dims
    assert port.spec(96, "12x{6,5,5}").dim_alloc_list() == [10, 8, 8, 10, 7, 7, 9, 7, 7, 9, 7, 7]
    assert port.spec(128, "12x{6,5,5}").dim_alloc_list() == [12, 10, 10] * 4
    for bad in ["x{4,4}", "16x{4,4", "16x{}", "16x{9}", "16x{4,}", "5x{4,4}", "16x{4,3}"]:
        with pytest.raises(OracleError) as e:
            port.spec(128, bad)
        assert e.value.kind == "invalid_spec"


def test_kat_compute_tables_1d(port):
    # T/test_distance.cpp:14-32: 1-D centroids {0,10,1e3...}, query 4 -> [16, 36]
    s = port.spec(1, "1x{8}")
    cb = np.full(256, 1e3, np.float32)
    cb[0], cb[1] = 0.0, 10.0
    lut = port.compute_tables(s, cb, np.array([4.0], np.float32))
    assert lut[0] == 16.0 and lut[1] == 36.0
    with pytest.raises(OracleError):  # T/test_distance.cpp:49-53
        port.compute_tables(s, cb, np.array([1.0, 2.0], np.float32))


def test_kat_calibrate_bounds(port):
    # T/test_distance.cpp:84-109: tables {1,9},{2,8},{3,7}; prefix {9,3,7,1,5}, R=3 -> d_min 6, d_max 5
    # three 2-entry tables do not form a legal packing group; embed them in the first two entries of a
    # 3x{6,5,5} LUT whose other entries are large
    s = port.spec(24, "3x{6,5,5}")
    lut = np.full(s.total_entries, 100.0, np.float32)
    for j, (a, b) in enumerate([(1.0, 9.0), (2.0, 8.0), (3.0, 7.0)]):
        lut[s.ent_off[j]], lut[s.ent_off[j] + 1] = a, b
    dmin, dmax = port.calibrate(s, lut, np.array([9, 3, 7, 1, 5], np.float32), 3)
    assert dmin == 6.0 and dmax == 5.0
    dmin, dmax = port.calibrate(s, lut, np.full(10, 4.25, np.float32), 7)
    assert dmax == 4.25
    for r in (3, 0):
        with pytest.raises(OracleError) as e:
            port.calibrate(s, lut, np.array([1, 2], np.float32), r)
        assert e.value.kind == "calibration"


def test_kat_quantize_identity_and_degenerate(port):
    # T/test_distance.cpp:111-119: width 8, d_min 0, d_max 255, distances 0..255 -> identity, delta 1
    s = port.spec(1, "1x{8}")
    q, pmin, delta, own = port.quantize(s, np.arange(256, dtype=np.float32), 0.0, 255.0, 8)
    assert delta == 1.0 and q.tolist() == list(range(256))
    # T/test_distance.cpp:167-177: d_max == d_min -> minima to 0, the rest to q_max
    s2 = port.spec(24, "3x{6,5,5}")
    lut = np.full(s2.total_entries, 50.0, np.float32)
    lut[s2.ent_off[0]:s2.ent_off[0] + 3] = [3.0, 5.0, 3.0]
    lut[s2.ent_off[1]:s2.ent_off[1] + 3] = [1.0, 2.0, 9.0]
    lut[s2.ent_off[2]] = 0.0
    q, pmin, delta, own = port.quantize(s2, lut, 4.0, 4.0, 16)
    assert delta == 0.0
    assert q[s2.ent_off[0]:s2.ent_off[0] + 3].tolist() == [0, 65535, 0]
    assert q[s2.ent_off[1]:s2.ent_off[1] + 3].tolist() == [0, 65535, 65535]
    with pytest.raises(OracleError) as e:
        port.quantize(s2, lut, 5.0, 4.0, 16)
    assert e.value.kind == "calibration"


def test_kat_saturating_adc(port):
    # T/test_distance.cpp:192-208: zero entries -> 0 ; 200 + 200 at width 8 -> 255
    s = port.spec(4, "2x{8}")
    qlut = np.concatenate([np.full(256, 7, np.uint8), np.full(256, 9, np.uint8)])
    qlut[4], qlut[256 + 5] = 0, 0
    pk = port.pack_list(s, np.array([[4, 5]], np.uint8))
    assert port.adc_sums(s, pk, 1, qlut, 0, 1).tolist() == [0]
    qlut = np.full(512, 200, np.uint8)
    pk = port.pack_list(s, np.array([[0, 0]], np.uint8))
    assert port.adc_sums(s, pk, 1, qlut, 0, 1).tolist() == [255]


def test_kat_heap_order(port):
    # T/test_heap_scan.cpp:11-42: keeps the R lexicographically smallest (dist, id); equal distance keeps lower id
    s = port.spec(4, "2x{8}")
    qlut = np.zeros(512, np.uint8)
    empty = np.zeros(0, np.uint8)
    d, i = port.scan_quantized(s, empty, 0, qlut, cap=3, heap_in=[(50, 1), (10, 2), (30, 3), (40, 4), (60, 5)])
    assert i.tolist() == [2, 3, 4] and d.tolist() == [10, 30, 40]
    d, i = port.scan_quantized(s, empty, 0, qlut, cap=1, heap_in=[(5, 10), (5, 3), (5, 7)])
    assert i.tolist() == [3]
    d, i = port.scan_quantized(s, empty, 0, qlut, cap=1, heap_in=[(5, 3), (5, 10)])
    assert i.tolist() == [3]
    with pytest.raises(OracleError) as e:  # T/test_heap_scan.cpp:56-58
        port.scan_quantized(s, empty, 0, qlut, cap=0)
    assert e.value.kind == "config"


def test_kat_scan_mismatch_is_config_error(port):
    # T/test_heap_scan.cpp:147-158: width != word width, rows*g != table count
    s = port.spec(128, "16x{4,4}")
    codes = np.zeros((5, 16), np.uint8)
    pk = port.pack_list(s, codes)
    with pytest.raises(OracleError) as e:
        port.scan_quantized(s, pk, 5, np.zeros(256, np.uint16), width=16)
    assert e.value.kind == "config"
    with pytest.raises(OracleError) as e:
        port.scan_quantized(s, pk, 5, np.zeros(256, np.uint8), rows=4)
    assert e.value.kind == "config"


def test_kat_all_zero_tables_keep_first_ids(port):
    # T/test_kernels.cpp:79-105: all-zero tables -> the first R ids at distance 0
    s = port.spec(128, "16x{4,4}")
    rng = np.random.default_rng(5)
    codes = rng.integers(0, 16, size=(100, 16)).astype(np.uint8)
    pk = port.pack_list(s, codes)
    d, i = port.scan_quantized(s, pk, 100, np.zeros(256, np.uint8), cap=10, base_id=7)
    assert d.tolist() == [0] * 10 and i.tolist() == list(range(7, 17))


def test_search_param_validation(port):
    # index.hpp:27-31 via T/test_index.cpp:46-55
    s = port.spec(64, "16x{4,4}")
    cb = np.zeros(s.cb_floats, np.float32)
    pk = port.pack_list(s, np.zeros((4, 16), np.uint8))
    q = np.zeros((1, 64), np.float32)
    for r, t in [(0, 400), (100, 50)]:
        with pytest.raises(OracleError) as e:
            port.flat_search(s, cb, pk, 4, q, r=r, t=t)
        assert e.value.kind == "input"
    ids, dists, counts = port.flat_search(s, cb, np.zeros(0, np.uint8), 0, q)  # empty DB -> empty result
    assert counts.tolist() == [0]


# ------------------------------------------------------- (b) golden fixtures --

@pytest.mark.parametrize("name", FLAT)
def test_golden_flat(port, golden, name):
    g = golden(name)
    s = port.spec(int(g["dims"]), str(g["spec"]))
    n = int(g["count"])
    assert np.array_equal(port.pack_list(s, g["codes"]), g["packed"])
    assert np.array_equal(port.unpack_list(s, g["packed"], n), g["codes"])
    assert np.array_equal(port.encode(s, g["codebook"], np.zeros((0, s.dims), np.float32)), np.zeros((0, s.m)))
    for qi, q in enumerate(g["queries"]):
        lut = port.compute_tables(s, g["codebook"], q)
        assert lut.tobytes() == g["luts"][qi].tobytes()
        pre = port.prefix_float(s, g["packed"], n, lut, int(g["t"]))
        assert pre.tobytes() == g["prefix"][qi].tobytes()
        r_eff = min(int(g["r"]), len(pre))
        dmin, dmax = port.calibrate(s, lut, pre, r_eff)
        assert (dmin, dmax) == (g["params"][qi][0], g["params"][qi][1])
        qlut, pmin, delta, own = port.quantize(s, lut, dmin, dmax, s.word_width)
        assert np.array_equal(qlut, g["qlut"][qi])
        assert (delta, own) == (g["params"][qi][2], g["params"][qi][3])
        assert np.array_equal(port.adc_sums(s, g["packed"], n, qlut, 0, n), g["sums"][qi])
    ids, dists, counts, qlut, params = port.flat_search(s, g["codebook"], g["packed"], n, g["queries"],
                                                        r=int(g["r"]), t=int(g["t"]), threads=2, debug=True)
    assert np.array_equal(counts, g["counts"])
    assert np.array_equal(ids, g["ids"]) and dists.tobytes() == g["dists"].tobytes()
    assert np.array_equal(qlut, g["qlut"]) and params.tobytes() == g["params"].tobytes()


def test_golden_scan_cases(port, golden):
    g = golden("scan_cases.npz")
    for c in range(int(g["n_cases"])):
        p = f"c{c}_"
        s = port.spec(int(g[p + "dims"]), str(g[p + "spec"]))
        ids = g[p + "ids"] if g[p + "ids"].size else None
        pre = [(int(d), int(i)) for d, i in g[p + "pre"]]
        od, oi = port.scan_quantized(s, g[p + "packed"], int(g[p + "n"]), g[p + "qlut"], ids=ids,
                                     base_id=int(g[p + "base"]), acc_init=int(g[p + "init"]), cap=int(g[p + "cap"]),
                                     heap_in=pre)
        assert np.array_equal(od, g[p + "out_d"]) and np.array_equal(oi, g[p + "out_i"]), str(g[p + "spec"])


@pytest.mark.parametrize("name", IVF)
def test_golden_ivf(port, golden, name):
    g = golden(name)
    s = port.spec(int(g["dims"]), str(g["spec"]))
    probes_mid = int(g["probe_list"][1])
    for qi, q in enumerate(g["queries"]):
        assert np.array_equal(port.probe_order(s.dims, g["coarse"], q, probes_mid), g["order"][qi])
    for pr in g["probe_list"]:
        ids, dists, counts = port.ivf_search(s, g["codebook"], g["coarse"], g["packed"], g["list_byte_off"],
                                             g["list_id_off"], g["list_count"], g["list_ids"], g["queries"],
                                             probes=int(pr), r=int(g["r"]), t=int(g["t"]), threads=2)
        assert np.array_equal(counts, g[f"counts_p{pr}"])
        assert np.array_equal(ids, g[f"ids_p{pr}"]) and dists.tobytes() == g[f"dists_p{pr}"].tobytes()


# ------------------------------------------- (c) live differential vs the reference --

@pytest.mark.parametrize("dims,text", [(128, "16x{4,4}"), (96, "12x{6,5,5}"), (128, "8x{8,8}"), (128, "8x{8}"),
                                       (128, "12x{6,6,4}"), (120, "12x{5,5,5}"), (64, "4x{4,4,4,4}")])
def test_live_differential_flat(port, ref, dims, text):
    rng = np.random.default_rng(hash(text) % 1000)
    sp, sr = port.spec(dims, text), ref.spec(dims, text)
    assert bytes(sp) == bytes(sr)
    cb = (rng.normal(size=sp.cb_floats) * 3).astype(np.float32)
    for n in (1, 31, 33, 700, 5000):
        codes = np.stack([rng.integers(0, 1 << b, size=n) for b in sp.bits_list()], 1).astype(np.uint8)
        pk = port.pack_list(sp, codes)
        assert np.array_equal(pk, ref.pack_list(sr, codes))
        queries = (rng.normal(size=(5, dims)) * 3).astype(np.float32)
        a = port.flat_search(sp, cb, pk, n, queries, r=100, t=400, debug=True)
        for fam in (0, 1):
            b = ref.flat_search(sr, cb, pk, n, queries, r=100, t=400, family=fam, debug=True)
            for x, y in zip(a, b):
                assert x.tobytes() == y.tobytes()


def test_live_differential_scan_fn(port, ref):
    """selftest.hpp:40-127 methodology: random tables / occupancy / pre-seeded heaps / bias / id modes."""
    rng = np.random.default_rng(11)
    fams = [("{4,4}", [2, 4, 6, 8, 10, 16, 32]), ("{6,6,4}", [3, 6, 12, 24]), ("{6,5,5}", [3, 6, 12, 24]),
            ("{5,5,5}", [3, 6, 12, 24]), ("{8,8}", [2, 4, 8, 16]), ("{8}", [1, 2, 4, 8, 16])]
    for pat, ms in fams:
        for _ in range(60):
            m = int(ms[rng.integers(len(ms))])
            s = port.spec(16 * m, f"{m}x{pat}")
            qmax = s.q_max
            if rng.integers(4) == 0:
                qlut = (qmax - rng.integers(0, qmax // 4 + 1, size=s.total_entries)).astype(s.qdtype)
            else:
                qlut = rng.integers(0, qmax + 1, size=s.total_entries).astype(s.qdtype)
            n = int(1 + rng.integers(s.block_len * 3))
            codes = np.stack([rng.integers(0, 1 << b, size=n) for b in s.bits_list()], 1).astype(np.uint8)
            pk = port.pack_list(s, codes)
            kw = dict(cap=int(1 + rng.integers(24)), acc_init=int(rng.integers(qmax + 2)) if rng.integers(4) == 0 else 0,
                      base_id=int(rng.integers(100000)),
                      ids=rng.integers(0, 1000000, size=n).astype(np.uint32) if rng.integers(2) else None,
                      heap_in=[(int(rng.integers(qmax + 1)), 2000000 + i) for i in range(int(rng.integers(4)))])
            a = port.scan_quantized(s, pk, n, qlut, **kw)
            for fam in (0, 1):
                b = ref.scan_quantized(s, pk, n, qlut, family=fam, **kw)
                assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


@pytest.mark.parametrize("dims,text,k_cells,n", [(64, "16x{4,4}", 24, 9000), (48, "12x{6,5,5}", 40, 12000),
                                                   (64, "8x{8,8}", 9, 2500), (32, "4x{8}", 15, 3000), (48, "6x{6,6,4}", 50, 700)])
def test_live_differential_ivf(port, ref, dims, text, k_cells, n):
    """The port's IvfIndex::search (shared quantization map + per-cell bias, index.hpp:276-341) against the unmodified
    reference, live: random coarse centroids and residual codebooks, ragged lists incl. empty / 1-code / shorter than t
    and R, probes 1 .. > K, both kernel families (normative scalar and the reference's auto SIMD choice), ids, distance
    bits and counts; and the probe order of every query (index.hpp:247-265), ties included."""
    rng = np.random.default_rng(k_cells * 1000 + n)
    sp, sr = port.spec(dims, text), ref.spec(dims, text)
    cb = (rng.normal(size=sp.cb_floats) * 1.5).astype(np.float32)
    coarse = (rng.normal(size=(k_cells, dims)) * 3).astype(np.float32)
    coarse[k_cells - 1] = coarse[0]  # an exact tie in the probe order: the lower cell first
    assign = rng.integers(0, k_cells, size=n)
    assign[assign == 3] = 4          # cell 3 stays empty
    assign[:1] = 5
    codes = np.stack([rng.integers(0, 1 << b, size=n) for b in sp.bits_list()], 1).astype(np.uint8)
    packed, ids, boff, ioff, counts = [], [], [], [], []
    b = i = 0
    for c in range(k_cells):
        members = np.nonzero(assign == c)[0].astype(np.uint32)
        pk = port.pack_list(sp, codes[members])
        boff.append(b); ioff.append(i); counts.append(len(members)); packed.append(pk); ids.append(members)
        b += pk.size; i += len(members)
    packed = np.concatenate(packed) if b else np.zeros(0, np.uint8)
    ids = np.concatenate(ids)
    args = (packed, np.array(boff, np.uint64), np.array(ioff, np.uint64), np.array(counts, np.uint64), ids)
    queries = (rng.normal(size=(7, dims)) * 3).astype(np.float32)
    queries[0] = coarse[0]
    for q in queries:
        for a in (1, 3, k_cells, k_cells + 5):
            assert np.array_equal(port.probe_order(dims, coarse, q, a), ref.probe_order(dims, coarse, q, a))
    for probes, r, t in [(1, 10, 20), (3, 100, 400), (k_cells // 2, 50, 50), (k_cells + 3, 300, 1000)]:
        want = port.ivf_search(sp, cb, coarse, *args, queries, probes=probes, r=r, t=t, threads=2)
        for fam in (0, 1):
            got = ref.ivf_search(sr, cb, coarse, *args, queries, probes=probes, r=r, t=t, family=fam, threads=2)
            for x, y in zip(want, got):
                assert x.tobytes() == y.tobytes(), (probes, r, t, fam)


# ------------------------------------------------------------------ rerank (N4) --

@pytest.mark.parametrize("name", FLAT + IVF)
def test_golden_rerank(port, golden, name):
    """SearchParams::rerank (index.hpp:53-67, 148-152, 377-386): same set, ordered by exact float ADC."""
    g = golden(name)
    s = port.spec(int(g["dims"]), str(g["spec"]))
    if name.startswith("flat"):
        ids, dists, counts = port.flat_search(s, g["codebook"], g["packed"], int(g["count"]), g["queries"],
                                              r=int(g["r"]), t=int(g["t"]), family=0x100)
        base = g["ids"]
    else:
        pr = int(g["probe_list"][1])
        ids, dists, counts = port.ivf_search(s, g["codebook"], g["coarse"], g["packed"], g["list_byte_off"],
                                             g["list_id_off"], g["list_count"], g["list_ids"], g["queries"], probes=pr,
                                             r=int(g["r"]), t=int(g["t"]), family=0x100)
        base = g[f"ids_p{pr}"]
    assert np.array_equal(ids, g["ids_rr"]) and dists.tobytes() == g["dists_rr"].tobytes()
    for qi in range(len(ids)):
        c = int(counts[qi])
        assert set(ids[qi, :c].tolist()) == set(base[qi, :c].tolist())  # T/test_index.cpp:318-322
        assert np.all(np.diff(dists[qi, :c]) >= 0)                        # T/test_index.cpp:325


def test_ivf_id_out_of_range_is_corruption(port, golden):
    g = golden("ivf_pq16x4.npz")  # index.hpp:372
    s = port.spec(int(g["dims"]), str(g["spec"]))
    bad = g["list_ids"].copy()
    bad[3] = bad.size + 5
    with pytest.raises(OracleError) as e:
        port.ivf_search(s, g["codebook"], g["coarse"], g["packed"], g["list_byte_off"], g["list_id_off"],
                        g["list_count"], bad, g["queries"], probes=2)
    assert e.value.kind == "corruption"


def _lists_equal(g, built, spec_pack, codes_by_cell=None):
    k = len(g["list_count"])
    for c in range(k):
        cnt, i0, b0 = int(g["list_count"][c]), int(g["list_id_off"][c]), int(g["list_byte_off"][c])
        assert cnt == int(built["list_count"][c])
        assert np.array_equal(g["ids"][i0:i0 + cnt], built["ids"][int(built["list_id_off"][c]):][:cnt])
        nb = spec_pack(cnt)
        assert np.array_equal(g["packed"][b0:b0 + nb], built["packed"][int(built["list_byte_off"][c]):][:nb])


@pytest.mark.parametrize("name", ["ivfbuild_pq8x4.npz", "ivfbuild_irr655.npz"])
def test_golden_ivf_build_lists(port, golden, name):
    """The port's assignment + residual encode, grouped and packed as index.hpp:219-227 does, reproduces the lists
    IvfIndex::build itself produced from the same vectors, centroids and codebook (fixture written by the reference)."""
    g = golden(name)
    s = port.spec(int(g["dims"]), str(g["spec"]))
    assign, codes = port.ivf_assign_encode(s, g["codebook"], g["coarse"], g["vectors"])
    k = len(g["list_count"])
    order = np.argsort(assign, kind="stable").astype(np.uint32)
    counts = np.bincount(assign, minlength=k).astype(np.uint64)
    id_off = np.concatenate([[0], np.cumsum(counts)[:-1]]).astype(np.uint64)
    parts, boff, b = [], [], 0
    for c in range(k):
        boff.append(b)
        pk = port.pack_list(s, codes[order[int(id_off[c]):int(id_off[c] + counts[c])]]) if counts[c] else np.zeros(0, np.uint8)
        parts.append(pk)
        b += pk.size
    built = dict(packed=np.concatenate(parts), list_byte_off=np.array(boff, np.uint64), list_id_off=id_off,
                 list_count=counts, ids=order)
    per_block = s.block_len * s.groups * (s.word_width // 8)
    _lists_equal(g, built, lambda cnt: (cnt + s.block_len - 1) // s.block_len * per_block)


def test_live_ivf_assign_encode(port, ref):
    rng = np.random.default_rng(9)
    dims, text, k = 32, "8x{4,4}", 300
    s = port.spec(dims, text)
    cb = (rng.standard_normal(s.cb_floats)).astype(np.float32)
    coarse = (rng.standard_normal((k, dims)) * 3).astype(np.float32)
    coarse[257] = coarse[3]  # exact tie: the lower cell wins
    v = (rng.standard_normal((500, dims)) * 3).astype(np.float32)
    v[0] = coarse[3]
    a, c = port.ivf_assign_encode(s, cb, coarse, v)
    a2, c2 = ref.ivf_assign_encode(s, cb, coarse, v)
    assert a[0] == 3 and np.array_equal(a, a2) and np.array_equal(c, c2)
