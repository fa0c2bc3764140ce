"""GPU parity tests proper: the CUDA path, called through the C ABI, against (1) the committed golden
fixtures produced by the unmodified reference and (2) the CPU oracle on the same seeded inputs.
Bit-exact everywhere: float LUTs and distances compare bitwise, integers exactly."""
import numpy as np
import pytest

import paper_1812_09162_b200 as qb
from paper_1812_09162_b200.synth import gaussian_mixture, random_codes

pytestmark = pytest.mark.gpu

FLAT = ["flat_pq16x4.npz", "flat_irr655.npz", "flat_irr664.npz", "flat_irr555.npz", "flat_split88.npz",
        "flat_split8.npz", "flat_pq16x4_short.npz", "flat_irr655_short.npz"]


@pytest.fixture(scope="module", autouse=True)
def _lib_loaded():
    qb.build()
    assert qb.lib().qadc_device_count() > 0, "GPU tests need a CUDA device"


def bits_equal(a, b):
    return a.shape == b.shape and a.tobytes() == b.tobytes()


@pytest.mark.parametrize("name", FLAT)
def test_golden_flat(golden, name):
    g = golden(name)
    s = qb.allocate_dims(int(g["dims"]), str(g["spec"]))
    n, r, t = int(g["count"]), int(g["r"]), int(g["t"])
    with qb.FlatIndex(s, g["codebook"], g["packed"], n) as idx:
        assert np.array_equal(idx.download_codes(0, n), g["codes"])  # layout bijection
        p = qb.SearchParams(r=r, t=t)
        luts, qluts, calib = idx.tables(g["queries"], p)
        assert bits_equal(luts, g["luts"])
        assert bits_equal(calib, g["params"])
        assert np.array_equal(qluts, g["qlut"])
        for qi in range(len(g["queries"])):
            assert np.array_equal(idx.adc_sums(g["qlut"][qi], 0, n), g["sums"][qi])
        res = idx.search(g["queries"], p)
        assert np.array_equal(res.counts, g["counts"])
        for qi in range(len(g["queries"])):
            c = int(g["counts"][qi])
            assert np.array_equal(res.ids[qi, :c], g["ids"][qi, :c])
            assert bits_equal(res.dists[qi, :c], g["dists"][qi, :c])
        assert idx.stats().kernel_launches > 0


def test_golden_scan_cases(golden):
    g = golden("scan_cases.npz")
    for c in range(int(g["n_cases"])):
        p = f"c{c}_"
        s = qb.allocate_dims(int(g[p + "dims"]), str(g[p + "spec"]))
        ids = g[p + "ids"] if g[p + "ids"].size else None
        pre = [(int(d), int(i)) for d, i in g[p + "pre"]]
        od, oi = qb.scan_list(s, g[p + "packed"], int(g[p + "n"]), g[p + "qlut"], ids=ids, base_id=int(g[p + "base"]),
                              acc_init=int(g[p + "init"]), cap=int(g[p + "cap"]), heap_in=pre)
        assert np.array_equal(od, g[p + "out_d"]) and np.array_equal(oi, g[p + "out_i"]), str(g[p + "spec"])


def test_scan_fn_differential(port):
    """selftest.hpp:40-127 methodology against the oracle: random tables (uniform / saturation-heavy), block
    counts and occupancies, pre-seeded heaps, accumulator bias, both id modes."""
    rng = np.random.default_rng(2024)
    fams = [("{4,4}", [2, 4, 6, 8, 10, 16, 32]), ("{6,6,4}", [3, 6, 12, 24]), ("{6,5,5}", [3, 6, 12, 24]),
            ("{5,5,5}", [3, 6, 12, 24]), ("{8,8}", [2, 4, 8, 16]), ("{8}", [1, 2, 4, 8, 16])]
    for pat, ms in fams:
        for _ in range(12):
            m = int(ms[rng.integers(len(ms))])
            s = qb.allocate_dims(16 * m, f"{m}x{pat}")
            so = port.spec(16 * m, f"{m}x{pat}")
            qmax = s.q_max
            dt = np.uint8 if s.word_width == 8 else np.uint16
            if rng.integers(4) == 0:
                qlut = (qmax - rng.integers(0, qmax // 4 + 1, size=s.total_entries)).astype(dt)
            else:
                qlut = rng.integers(0, qmax + 1, size=s.total_entries).astype(dt)
            n = int(1 + rng.integers(s.block_len * 3))
            if rng.integers(3) == 0:
                n = int(1 + rng.integers(20000))
            codes = random_codes(s, n, seed=int(rng.integers(1 << 30)))
            pk = qb.pack_list(s, codes)
            kw = dict(cap=int(1 + rng.integers(24)),
                      acc_init=int(rng.integers(qmax + 2)) if rng.integers(4) == 0 else 0,
                      base_id=int(rng.integers(100000)),
                      ids=rng.integers(0, 1000000, size=n).astype(np.uint32) if rng.integers(2) else None,
                      heap_in=[(int(rng.integers(qmax + 1)), 2000000 + i) for i in range(int(rng.integers(4)))])
            a = port.scan_quantized(so, pk, n, qlut, **kw)
            b = qb.scan_list(s, pk, n, qlut, **kw)
            assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]), (pat, m, n, kw["cap"])


@pytest.mark.parametrize("variant", [12, 13, 14])
def test_tensor_core_scan_through_scan_fn_contract(port, monkeypatch, variant):
    """The tcgen05 one-hot GEMM scan (scan_tc.cu, variants 12 = dense and 13 = 2:4 sparse) forced onto the QuantizedScanFn entry point
    (QADC_FORCE_VARIANT): the same differential as above for 16x{4,4} -- ragged list lengths (sub-tile and stage
    tails), saturation-heavy tables, pre-seeded heaps, accumulator bias up to q_max + 1 (folded into the threshold
    K step), both id modes, heaps that never fill (rows without a threshold take the exact re-evaluation), and the
    all-zero / all-saturated corner tables of T/test_kernels.cpp:79-105, 135-159."""
    monkeypatch.setenv("QADC_FORCE_VARIANT", str(variant))
    rng = np.random.default_rng(4242)
    s, so = qb.allocate_dims(128, "16x{4,4}"), port.spec(128, "16x{4,4}")
    for trial in range(40):
        if rng.integers(4) == 0:
            qlut = (255 - rng.integers(0, 64, size=256)).astype(np.uint8)
        elif rng.integers(3) == 0:
            qlut = rng.integers(0, 24, size=256).astype(np.uint8)        # small sums: dense admissions, many ties
        else:
            qlut = rng.integers(0, 256, size=256).astype(np.uint8)
        n = int([1, 127, 128, 129, 1023, 1024, 1025, 5000, 20000, 70001][trial % 10] + rng.integers(0, 3))
        pk = qb.pack_list(s, random_codes(s, n, seed=int(rng.integers(1 << 30))))
        kw = dict(cap=int([1, 7, 24, 100, 1000][trial % 5]),
                  acc_init=int(rng.integers(257)) if rng.integers(3) == 0 else 0,
                  base_id=int(rng.integers(100000)),
                  ids=rng.integers(0, 1000000, size=n).astype(np.uint32) if rng.integers(2) else None,
                  heap_in=[(int(rng.integers(256)), 2000000 + i) for i in range(int(rng.integers(4)))])
        a = port.scan_quantized(so, pk, n, qlut, **kw)
        b = qb.scan_list(s, pk, n, qlut, **kw)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]), (trial, n, kw["cap"], kw["acc_init"])
    n = 30000
    pk = qb.pack_list(s, random_codes(s, n, seed=3))
    d, i = qb.scan_list(s, pk, n, np.zeros(256, np.uint8), cap=10, base_id=7)
    assert d.tolist() == [0] * 10 and i.tolist() == list(range(7, 17))
    d, i = qb.scan_list(s, pk, n, np.full(256, 255, np.uint8), cap=5, heap_in=[(9, 1), (8, 2), (7, 3), (6, 4), (5, 5)])
    assert i.tolist() == [5, 4, 3, 2, 1]
    d, i = qb.scan_list(s, pk, n, np.full(256, 255, np.uint8), cap=5)
    assert d.tolist() == [255] * 5 and i.tolist() == [0, 1, 2, 3, 4]


def test_scan_list_config_errors():
    # scan_scalar.hpp:23-27, 38-39; heap.hpp:27-28
    s = qb.allocate_dims(128, "16x{4,4}")
    pk = qb.pack_list(s, np.zeros((5, 16), np.uint8))
    for kw, q in [(dict(width=16), np.zeros(256, np.uint16)), (dict(rows=4), np.zeros(256, np.uint8)),
                  (dict(cap=0), np.zeros(256, np.uint8))]:
        with pytest.raises(qb.QadcError) as e:
            qb.scan_list(s, pk, 5, q, **kw)
        assert e.value.kind == "config"


def test_all_zero_and_saturated_tables(port):
    # T/test_kernels.cpp:79-105 (all-zero tables keep the first R ids) and :135-159 (saturated never displace)
    s = qb.allocate_dims(128, "16x{4,4}")
    n = 30000
    pk = qb.pack_list(s, random_codes(s, n, seed=3))
    d, i = qb.scan_list(s, pk, n, np.zeros(256, np.uint8), cap=10, base_id=7)
    assert d.tolist() == [0] * 10 and i.tolist() == list(range(7, 17))
    d, i = qb.scan_list(s, pk, n, np.full(256, 255, np.uint8), cap=5, heap_in=[(9, 1), (8, 2), (7, 3), (6, 4), (5, 5)])
    assert i.tolist() == [5, 4, 3, 2, 1]
    d, i = qb.scan_list(s, pk, n, np.full(256, 255, np.uint8), cap=5)
    assert d.tolist() == [255] * 5 and i.tolist() == [0, 1, 2, 3, 4]


def test_whole_vs_chunked_scan(port):
    # T/test_kernels.cpp:107-133: scanning a list in chunks with base_id == scanning it whole (sharding correctness)
    rng = np.random.default_rng(9)
    for dims, text in [(128, "16x{4,4}"), (96, "12x{6,5,5}")]:
        s = qb.allocate_dims(dims, text)
        n = 3 * 960
        codes = random_codes(s, n, seed=4)
        qlut = rng.integers(0, s.q_max + 1, size=s.total_entries).astype(np.uint8 if s.word_width == 8 else np.uint16)
        whole = qb.scan_list(s, qb.pack_list(s, codes), n, qlut, cap=20)
        heap = []
        for c in range(3):
            part = codes[c * 960:(c + 1) * 960]
            d, i = qb.scan_list(s, qb.pack_list(s, part), 960, qlut, cap=20, base_id=c * 960, heap_in=heap)
            heap = list(zip(d.tolist(), i.tolist()))
        assert [h[0] for h in heap] == whole[0].tolist() and [h[1] for h in heap] == whole[1].tolist()


SPECS = [(128, "16x{4,4}"), (96, "12x{6,5,5}"), (128, "8x{8,8}"), (128, "8x{8}"), (128, "12x{6,6,4}"),
         (120, "12x{5,5,5}"), (128, "12x{6,5,5}"), (64, "32x{4,4}"), (64, "4x{4,4,4,4}"), (96, "24x{6,5,5}"),
         (96, "24x{6,6,4}"), (128, "16x{8,8}")]  # incl. the paper's 128-bit configurations


@pytest.mark.parametrize("dims,text", SPECS)
def test_flat_search_vs_oracle(port, dims, text):
    """FlatIndex::search end to end (T/test_index.cpp:57-89): ids AND unquantized distances exact."""
    rng = np.random.default_rng(abs(hash(text)) % 10000)
    s, so = qb.allocate_dims(dims, text), port.spec(dims, text)
    cb = (rng.standard_normal(s.cb_floats) * 2).astype(np.float32)
    n, nq = 60000, 70
    codes = random_codes(s, n, seed=12)
    pk = qb.pack_list(s, codes)
    queries = (rng.standard_normal((nq, dims)) * 2).astype(np.float32)
    ref = port.flat_search(so, cb, pk, n, queries, r=100, t=400, threads=8, debug=True)
    with qb.FlatIndex(s, cb, pk, n) as idx:
        luts, qluts, calib = idx.tables(queries)
        assert np.array_equal(qluts, ref[3]) and bits_equal(calib, ref[4])
        res = idx.search(queries)
        assert np.array_equal(res.counts, ref[2])
        assert np.array_equal(res.ids, ref[0]) and bits_equal(res.dists, ref[1])
        # R >= N and tiny r / t edge cases (T/test_index.cpp:24-55)
        for r, t in [(1, 1), (7, 9), (1000, 1000)]:
            sub = queries[:5]
            ref2 = port.flat_search(so, cb, pk[:qb.packed_bytes(s, 300)], 300, sub, r=r, t=t)
            with qb.FlatIndex(s, cb, pk[:qb.packed_bytes(s, 300)], 300) as small:
                got = small.search(sub, qb.SearchParams(r=r, t=t))
                assert np.array_equal(got.counts, ref2[2])
                for qi in range(5):
                    c = int(ref2[2][qi])
                    assert np.array_equal(got.ids[qi, :c], ref2[0][qi, :c]) and bits_equal(got.dists[qi, :c], ref2[1][qi, :c])


@pytest.mark.parametrize("dims,text,n,r,t", [(64, "16x{4,4}", 30_000, 1500, 2000), (48, "12x{6,5,5}", 20_000, 7000, 9000),
                                            (64, "8x{8}", 9_000, 16384, 16384)])
def test_large_r_and_t_vs_oracle(port, dims, text, n, r, t):
    """R and t far above the paper's 100 / 400 (the reference bounds neither, index.hpp:27-31; the device top-R stage
    goes to QADC_MAX_R = QADC_MAX_T = 16384): heaps that stay unfilled for most of the list, candidate-buffer retries,
    R > N; flat and IVF."""
    rng = np.random.default_rng(r)
    s, so = qb.allocate_dims(dims, text), port.spec(dims, text)
    cb = (rng.standard_normal(s.cb_floats) * 2).astype(np.float32)
    pk = qb.pack_list(s, random_codes(s, n, seed=r))
    queries = (rng.standard_normal((6, dims)) * 2).astype(np.float32)
    want = port.flat_search(so, cb, pk, n, queries, r=r, t=t, threads=6)
    with qb.FlatIndex(s, cb, pk, n) as idx:
        got = idx.search(queries, qb.SearchParams(r=r, t=t))
        with pytest.raises(qb.QadcError) as e:
            idx.search(queries, qb.SearchParams(r=16385, t=16385))
        assert e.value.kind == "config"
    assert np.array_equal(got.counts, want[2])
    for qi in range(len(queries)):
        c = int(want[2][qi])
        assert np.array_equal(got.ids[qi, :c], want[0][qi, :c]) and bits_equal(got.dists[qi, :c], want[1][qi, :c])
    k_cells = 12
    coarse = (rng.standard_normal((k_cells, dims)) * 3).astype(np.float32)
    packed, boff, ioff, counts, ids = _ivf_lists(rng, s, k_cells, n)
    rr, tt = min(r, 3000), min(t, 4000)
    want = port.ivf_search(so, cb, coarse, packed, boff, ioff, counts, ids, queries, probes=5, r=rr, t=tt, threads=6)
    with qb.IvfIndex(s, cb, coarse, packed, boff, ioff, counts, ids) as idx:
        got = idx.search(queries, qb.SearchParams(probes=5, r=rr, t=tt))
    assert np.array_equal(got.counts, want[2])
    for qi in range(len(queries)):
        c = int(want[2][qi])
        assert np.array_equal(got.ids[qi, :c], want[0][qi, :c]) and bits_equal(got.dists[qi, :c], want[1][qi, :c])


def test_search_errors_and_empty():
    s = qb.allocate_dims(64, "16x{4,4}")
    cb = np.zeros(s.cb_floats, np.float32)
    pk = qb.pack_list(s, np.zeros((40, 16), np.uint8))
    with qb.FlatIndex(s, cb, pk, 40) as idx:
        q = np.zeros((2, 64), np.float32)
        for p in (qb.SearchParams(r=0), qb.SearchParams(r=100, t=50)):
            with pytest.raises(qb.QadcError) as e:
                idx.search(q, p)
            assert e.value.kind == "input"
        with pytest.raises(qb.QadcError) as e:
            idx.search(np.zeros((2, 63), np.float32))
        assert e.value.kind == "input"
        res = idx.search(q)  # degenerate: all-zero codebook -> delta == 0, every distance 0, first ids win
        assert res.counts.tolist() == [40, 40] and res.ids[0, :40].tolist() == list(range(40))
    with qb.FlatIndex(s, cb, np.zeros(0, np.uint8), 0) as empty:
        res = empty.search(np.zeros((3, 64), np.float32))
        assert res.counts.tolist() == [0, 0, 0]
    bad = cb.copy()
    bad[3] = np.nan
    with pytest.raises(qb.QadcError) as e:
        qb.FlatIndex(s, bad, pk, 40)
    assert e.value.kind == "corruption"


def test_candidate_overflow_retry(port):
    """Adversarial order (distances strictly improving along the list) floods the candidate buffer; the
    library must detect the overflow and redo the batch with a larger buffer, still exact."""
    s, so = qb.allocate_dims(16, "2x{8}"), port.spec(16, "2x{8}")
    n = 40000
    codes = np.zeros((n, 2), np.uint8)
    codes[:, 0] = (255 - (np.arange(n) * 256 // n)).astype(np.uint8)  # decreasing first subcode
    codes[:, 1] = 0
    pk = qb.pack_list(s, codes)
    qlut = np.concatenate([np.arange(256) // 2, np.zeros(256)]).astype(np.uint8)
    a = port.scan_quantized(so, pk, n, qlut, cap=50)
    b = qb.scan_list(s, pk, n, qlut, cap=50)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_encode_vs_oracle(port):
    rng = np.random.default_rng(5)
    for dims, text in [(128, "16x{4,4}"), (96, "12x{6,5,5}"), (64, "8x{8}")]:
        s, so = qb.allocate_dims(dims, text), port.spec(dims, text)
        cb = (rng.standard_normal(s.cb_floats) * 2).astype(np.float32)
        # duplicate a centroid so that exact ties occur (lowest index must win, T/test_kmeans_codebook.cpp:108-118)
        d0 = s.dim_alloc[0]
        cb[d0:2 * d0] = cb[0:d0]
        v = (rng.standard_normal((3000, dims)) * 2).astype(np.float32)
        v[0, :d0] = cb[0:d0]
        assert np.array_equal(qb.encode(s, cb, v), port.encode(so, cb, v))


def test_large_seeded_property_round_trip(port):
    """Size-independent properties at a larger size (1M codes x 256 queries on 16x{4,4}): every returned
    (distance, id) must equal the oracle's quantized ADC sum of that code under the oracle's tables, be
    sorted by (distance, id), and the R-th distance must bound a uniform sample of the list."""
    rng = np.random.default_rng(77)
    dims, text = 128, "16x{4,4}"
    s, so = qb.allocate_dims(dims, text), port.spec(dims, text)
    centres = None
    train = gaussian_mixture(20000, dims, seed=4)
    from paper_1812_09162_b200.synth import train_codebook
    cb = train_codebook(s, train, iters=4)
    n, nq = 1_000_000, 256
    codes = random_codes(s, n, seed=6)
    pk = qb.pack_list(s, codes)
    queries = gaussian_mixture(nq, dims, seed=3)
    with qb.FlatIndex(s, cb, pk, n) as idx:
        res = idx.search(queries)
        luts, qluts, calib = idx.tables(queries)
    assert np.all(res.counts == 100)
    sample = rng.choice(n, size=20000, replace=False)
    for qi in range(0, nq, 16):
        lut = port.compute_tables(so, cb, queries[qi])
        pre = port.prefix_float(so, pk, n, lut, 400)
        dmin, dmax = port.calibrate(so, lut, pre, 100)
        qlut, _, delta, own = port.quantize(so, lut, dmin, dmax, 8)
        assert np.array_equal(qlut, qluts[qi])
        sums = qlut.astype(np.uint32).reshape(16, 16)[np.arange(16)[None, :], codes[res.ids[qi]].astype(np.int64)].sum(1)
        sums = np.minimum(sums, 255)
        want = (sums.astype(np.float32) * delta + own).astype(np.float32)
        assert bits_equal(res.dists[qi], want)
        keys = sums.astype(np.int64) << 32 | res.ids[qi].astype(np.int64)
        assert np.all(np.diff(keys) > 0)
        ssum = np.minimum(qlut.astype(np.uint32).reshape(16, 16)[np.arange(16)[None, :], codes[sample].astype(np.int64)].sum(1), 255)
        skeys = ssum.astype(np.int64) << 32 | sample.astype(np.int64)
        inside = np.isin(sample, res.ids[qi])
        assert np.all(skeys[~inside] > keys[-1])
    # and the full oracle on a few queries
    ref = port.flat_search(so, cb, pk, n, queries[:4], r=100, t=400, threads=4)
    assert np.array_equal(res.ids[:4], ref[0]) and bits_equal(res.dists[:4], ref[1])


# ------------------------------------------------------------------------- IVF --

def _ivf_lists(rng, s, k_cells, n, empty=()):
    """Random IVF partition: list sizes, packed lists (reference layout, concatenated), ids."""
    assign = rng.integers(0, k_cells, size=n)
    for c in empty:
        assign[assign == c] = (c + 1) % k_cells
    codes = random_codes(s, n, seed=int(rng.integers(1 << 30)))
    packed, ids, boff, ioff, counts = [], [], [], [], []
    b = i = 0
    for c in range(k_cells):
        members = np.nonzero(assign == c)[0].astype(np.uint32)
        rng.shuffle(members)
        pk = qb.pack_list(s, codes[members]) if len(members) else np.zeros(0, np.uint8)
        boff.append(b); ioff.append(i); counts.append(len(members))
        packed.append(pk); ids.append(members)
        b += pk.size; i += len(members)
    return (np.concatenate(packed), np.array(boff, np.uint64), np.array(ioff, np.uint64),
            np.array(counts, np.uint64), np.concatenate(ids).astype(np.uint32))


@pytest.mark.parametrize("name", ["ivf_irr655.npz", "ivf_pq16x4.npz"])
def test_golden_ivf(golden, name):
    g = golden(name)
    s = qb.allocate_dims(int(g["dims"]), str(g["spec"]))
    with qb.IvfIndex(s, g["codebook"], g["coarse"], g["packed"], g["list_byte_off"], g["list_id_off"],
                     g["list_count"], g["list_ids"]) as idx:
        probes_mid = int(g["probe_list"][1])
        assert np.array_equal(idx.probe_order(g["queries"], probes_mid), g["order"])
        for pr in g["probe_list"]:
            res = idx.search(g["queries"], qb.SearchParams(probes=int(pr), r=int(g["r"]), t=int(g["t"])))
            assert np.array_equal(res.counts, g[f"counts_p{pr}"])
            for qi in range(len(g["queries"])):
                c = int(res.counts[qi])
                assert np.array_equal(res.ids[qi, :c], g[f"ids_p{pr}"][qi, :c]), (name, int(pr), qi)
                assert bits_equal(res.dists[qi, :c], g[f"dists_p{pr}"][qi, :c])


@pytest.mark.parametrize("dims,text,k_cells,n,probes", [(128, "12x{6,5,5}", 64, 150000, 8), (64, "16x{4,4}", 40, 60000, 5),
                                                        (64, "8x{8,8}", 16, 30000, 16), (48, "12x{6,6,4}", 300, 90000, 32)])
def test_ivf_search_vs_oracle(port, dims, text, k_cells, n, probes):
    """IvfIndex::search (shared map + per-cell bias + explicit ids) against the oracle, including empty cells,
    lists shorter than t and R, and probes > non-empty cells."""
    rng = np.random.default_rng(abs(hash((text, k_cells))) % 10000)
    s, so = qb.allocate_dims(dims, text), port.spec(dims, text)
    cb = (rng.standard_normal(s.cb_floats) * 1.5).astype(np.float32)
    coarse = (rng.standard_normal((k_cells, dims)) * 3).astype(np.float32)
    packed, boff, ioff, counts, ids = _ivf_lists(rng, s, k_cells, n, empty=(1, k_cells - 2))
    queries = (rng.standard_normal((50, dims)) * 3).astype(np.float32)
    with qb.IvfIndex(s, cb, coarse, packed, boff, ioff, counts, ids) as idx:
        for pr, r, t in [(probes, 100, 400), (1, 10, 10), (k_cells + 5, 100, 5000)]:
            want = port.ivf_search(so, cb, coarse, packed, boff, ioff, counts, ids, queries, probes=pr, r=r, t=t, threads=8)
            got = idx.search(queries, qb.SearchParams(probes=pr, r=r, t=t))
            assert np.array_equal(got.counts, want[2]), (pr, r, t)
            for qi in range(len(queries)):
                c = int(want[2][qi])
                assert np.array_equal(got.ids[qi, :c], want[0][qi, :c]), (pr, r, t, qi)
                assert bits_equal(got.dists[qi, :c], want[1][qi, :c])
        a = min(probes, k_cells)
        order = idx.probe_order(queries, a)
        for qi in range(0, 50, 7):
            assert np.array_equal(order[qi], port.probe_order(dims, coarse, queries[qi], a))
        with pytest.raises(qb.QadcError) as e:
            idx.search(queries, qb.SearchParams(probes=0))
        assert e.value.kind == "input"


def test_ivf_all_lists_empty_or_tiny(port):
    dims, text = 64, "16x{4,4}"
    s, so = qb.allocate_dims(dims, text), port.spec(dims, text)
    rng = np.random.default_rng(4)
    cb = rng.standard_normal(s.cb_floats).astype(np.float32)
    coarse = rng.standard_normal((8, dims)).astype(np.float32)
    queries = rng.standard_normal((6, dims)).astype(np.float32)
    z64 = np.zeros(8, np.uint64)
    with qb.IvfIndex(s, cb, coarse, np.zeros(0, np.uint8), z64, z64, z64, np.zeros(0, np.uint32)) as idx:
        res = idx.search(queries, qb.SearchParams(probes=3))
        assert res.counts.tolist() == [0] * 6
    packed, boff, ioff, counts, ids = _ivf_lists(rng, s, 8, 30)
    with qb.IvfIndex(s, cb, coarse, packed, boff, ioff, counts, ids) as idx:
        want = port.ivf_search(so, cb, coarse, packed, boff, ioff, counts, ids, queries, probes=8, r=100, t=400)
        got = idx.search(queries, qb.SearchParams(probes=8))
        assert np.array_equal(got.counts, want[2])
        for qi in range(6):
            c = int(want[2][qi])
            assert np.array_equal(got.ids[qi, :c], want[0][qi, :c]) and bits_equal(got.dists[qi, :c], want[1][qi, :c])


# ------------------------------------------------------------------ sharded (1 GPU) --

@pytest.mark.parametrize("dims,text,n,world", [(128, "16x{4,4}", 100000, 4), (96, "12x{6,5,5}", 50000, 3), (128, "8x{8,8}", 300, 8)])
def test_sharded_device_path_equals_unsharded(port, dims, text, n, world):
    """The multi-GPU data path on one device: every 'rank' is a FlatIndex over its block-aligned shard opened
    with base_id and the global calibration head; their device key lists are stacked as all_gather would and
    merged by the CUDA merge kernel.  Ranks run one after the other (nothing waits on another kernel)."""
    import torch
    from paper_1812_09162_b200.dist import global_head, shard_ranges, slice_packed
    rng = np.random.default_rng(3)
    s, so = qb.allocate_dims(dims, text), port.spec(dims, text)
    cb = (rng.standard_normal(s.cb_floats) * 2).astype(np.float32)
    packed = qb.pack_list(s, random_codes(s, n, seed=8))
    queries = (rng.standard_normal((33, dims)) * 2).astype(np.float32)
    r, t = 100, 400
    want = port.flat_search(so, cb, packed, n, queries, r=r, t=t, threads=8)
    dev = torch.device("cuda", 0)
    d_q = torch.from_numpy(queries).to(dev)
    head, head_n = global_head(s, packed, n)
    if n > 1000:  # a head shorter than the list serves t <= its length only; beyond that: refused, never clamped
        short, short_n = global_head(s, packed, n, t_max=256)
        for gc in (n, 0):  # 0 = whole-list length unknown: treated as truncated
            with qb.FlatIndex(s, cb, slice_packed(s, packed, shard_ranges(n, world, s.block_len)[1]), 64, base_id=64,
                              calib_packed=short, calib_count=short_n, global_count=gc) as shard:
                with pytest.raises(qb.QadcError) as e:
                    shard.search(queries, qb.SearchParams(r=r, t=t))
                assert e.value.kind == "config"
                assert shard.search(queries, qb.SearchParams(r=r, t=256)).counts.max() <= r
    keys = torch.empty((world, len(queries), r), dtype=torch.int64, device=dev)
    qmap = torch.empty((len(queries), 2), dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream().cuda_stream
    params = qb.SearchParams(r=r, t=t)
    for rank, rg in enumerate(shard_ranges(n, world, s.block_len)):
        with qb.FlatIndex(s, cb, slice_packed(s, packed, rg), rg.count, base_id=rg.start, calib_packed=head,
                          calib_count=head_n, global_count=n) as shard:
            shard.search_device(d_q, params, None, None, None, d_keys=keys[rank], d_map=qmap, stream=stream)
            torch.cuda.synchronize()
    d_ids = torch.empty((len(queries), r), dtype=torch.int32, device=dev)
    d_dists = torch.empty((len(queries), r), dtype=torch.float32, device=dev)
    d_counts = torch.empty((len(queries),), dtype=torch.int32, device=dev)
    qb.merge_topk_device(keys, world, len(queries), r, qmap, d_ids, d_dists, d_counts, 0, stream=stream)
    torch.cuda.synchronize()
    counts = d_counts.cpu().numpy().astype(np.uint32)
    ids = d_ids.cpu().numpy().view(np.uint32)
    dists = d_dists.cpu().numpy()
    assert np.array_equal(counts, want[2])
    for qi in range(len(queries)):
        c = int(want[2][qi])
        assert np.array_equal(ids[qi, :c], want[0][qi, :c]) and bits_equal(dists[qi, :c], want[1][qi, :c])


# ------------------------------------------------ reference-side C++ binding (qadc.hpp) --

def test_one_process_multi_gpu_handle(port):
    """qadc_flat_open_sharded / qadc_multi_search_batch (the C++ single-process host: shards with base ids, replicated
    calibration head, ncclAllGather, merge) on the devices of this box: same result as the plain FlatIndex and the
    oracle; the exchange goes through NCCL whenever libnccl can be loaded; bad device lists are input errors."""
    import torch  # noqa: F401  (loads the NCCL build the process shares)
    rng = np.random.default_rng(12)
    ndev = qb.lib().qadc_device_count()
    for dims, text, n in [(128, "16x{4,4}", 120_000), (96, "12x{6,5,5}", 33_333), (64, "8x{8}", 100)]:
        s, so = qb.allocate_dims(dims, text), port.spec(dims, text)
        cb = (rng.standard_normal(s.cb_floats) * 2).astype(np.float32)
        pk = qb.pack_list(s, random_codes(s, n, seed=31))
        queries = (rng.standard_normal((50, dims)) * 2).astype(np.float32)
        want = port.flat_search(so, cb, pk, n, queries, r=100, t=400, threads=8)
        with qb.MultiGpuFlatIndex(s, cb, pk, n, ndev=ndev) as idx:
            info = idx.info()
            assert info["ndev"] == ndev and info["count"] == n and info["uses_nccl"]
            for _ in range(2):
                got = idx.search(queries, qb.SearchParams(r=100, t=400))
                assert np.array_equal(got.counts, want[2])
                for qi in range(len(queries)):
                    c = int(want[2][qi])
                    assert np.array_equal(got.ids[qi, :c], want[0][qi, :c]) and bits_equal(got.dists[qi, :c], want[1][qi, :c])
            with pytest.raises(qb.QadcError) as e:
                idx.search(queries, qb.SearchParams(r=100, t=400, rerank=True))
            assert e.value.kind == "config"
    for bad in ([0, 0], [ndev], [-1]):
        with pytest.raises(qb.QadcError) as e:
            qb.MultiGpuFlatIndex(s, cb, pk, n, ndev=len(bad), devices=bad)
        assert e.value.kind == "input"


def test_cpp_integration_binary():
    """The reference's own C++ types (FlatIndex, IvfIndex, QuantizedScanFn, CandidateHeap) against the GPU path
    through include/qadc.hpp.  The binary is compiled in the build container against the unmodified reference
    headers (oracle/Makefile `integration`) and travels with the snapshot; it is absent only if that build never ran."""
    import subprocess
    from pathlib import Path
    exe = Path(__file__).resolve().parent.parent / "oracle" / "_ref" / "integration_test"
    if not exe.exists():
        pytest.skip("oracle/_ref/integration_test was not built (no reference tree at build time)")
    import os
    for extra in ({}, {"QADC_MULTI_SAME_DEVICE_TEST": "1"}):  # second run: the sharded handles split 3 ways on one device
        out = subprocess.run([str(exe), "25"], capture_output=True, text=True, timeout=900, env={**os.environ, **extra})
        assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]
        assert "INTEGRATION OK" in out.stdout


def test_one_process_sharding_arithmetic_on_one_device(port, monkeypatch):
    """qadc_flat_open_sharded / qadc_ivf_open_sharded with ndev = 3 on ONE device (test hook
    QADC_MULTI_SAME_DEVICE_TEST: duplicate ordinals allowed, the exchange is a device-to-device copy instead of
    ncclAllGather): block-aligned ranges with base ids, every IVF list split three ways, replicated calibration heads,
    gather order and merge -- same result as the oracle, incl. lists shorter than a block and t beyond short lists."""
    monkeypatch.setenv("QADC_MULTI_SAME_DEVICE_TEST", "1")
    rng = np.random.default_rng(77)
    for dims, text, n in [(128, "16x{4,4}", 100_003), (96, "12x{6,5,5}", 20_000), (64, "8x{8}", 70)]:
        s, so = qb.allocate_dims(dims, text), port.spec(dims, text)
        cb = (rng.standard_normal(s.cb_floats) * 2).astype(np.float32)
        pk = qb.pack_list(s, random_codes(s, n, seed=5))
        queries = (rng.standard_normal((33, dims)) * 2).astype(np.float32)
        want = port.flat_search(so, cb, pk, n, queries, r=50, t=300, threads=8)
        with qb.MultiGpuFlatIndex(s, cb, pk, n, ndev=3, devices=[0, 0, 0]) as idx:
            assert idx.info() == dict(ndev=3, count=n, uses_nccl=False)
            got = idx.search(queries, qb.SearchParams(r=50, t=300))
        assert np.array_equal(got.counts, want[2]) and np.array_equal(got.ids, want[0]) and bits_equal(got.dists, want[1])
    dims, text, k_cells, n = 64, "12x{6,5,5}", 24, 30_000
    s, so = qb.allocate_dims(dims, text), port.spec(dims, text)
    cb = (rng.standard_normal(s.cb_floats) * 1.5).astype(np.float32)
    coarse = (rng.standard_normal((k_cells, dims)) * 3).astype(np.float32)
    assign = rng.integers(0, k_cells - 2, size=n)  # two empty lists
    assign[:5] = k_cells - 2                        # and one of five codes
    codes = random_codes(s, n, seed=8)
    packed, ids, boff, ioff, counts = [], [], [], [], []
    b = i = 0
    for c in range(k_cells):
        members = np.nonzero(assign == c)[0].astype(np.uint32)
        lp = qb.pack_list(s, codes[members])
        boff.append(b); ioff.append(i); counts.append(len(members)); packed.append(lp); ids.append(members)
        b += lp.size; i += len(members)
    packed, ids = np.concatenate(packed), np.concatenate(ids)
    queries = (rng.standard_normal((40, dims)) * 3).astype(np.float32)
    for probes, r, t in [(5, 60, 250), (24, 100, 2000)]:
        want = port.ivf_search(so, cb, coarse, packed, boff, ioff, counts, ids, queries, probes=probes, r=r, t=t, threads=8)
        with qb.MultiGpuIvfIndex(s, cb, coarse, packed, boff, ioff, counts, ids, ndev=3, devices=[0, 0, 0]) as idx:
            assert idx.info()["ndev"] == 3 and idx.info()["count"] == n
            got = idx.search(queries, qb.SearchParams(probes=probes, r=r, t=t))
        assert np.array_equal(got.counts, want[2])
        for qi in range(len(queries)):
            c = int(want[2][qi])
            assert np.array_equal(got.ids[qi, :c], want[0][qi, :c]) and bits_equal(got.dists[qi, :c], want[1][qi, :c])


@pytest.mark.parametrize("world", [2, 5])
def test_sharded_ivf_equals_unsharded(port, world):
    """IVF sharding on one device: every list split across `world` ranks, heads replicated for calibration;
    per-rank key lists merged by the CUDA merge kernel must equal the unsharded IvfIndex::search."""
    import torch
    from paper_1812_09162_b200.dist import shard_ivf_lists
    dims, text, k_cells, n = 64, "12x{6,5,5}", 30, 40000
    rng = np.random.default_rng(21)
    s, so = qb.allocate_dims(dims, text), port.spec(dims, text)
    cb = (rng.standard_normal(s.cb_floats) * 1.5).astype(np.float32)
    coarse = (rng.standard_normal((k_cells, dims)) * 3).astype(np.float32)
    packed, boff, ioff, counts, ids = _ivf_lists(rng, s, k_cells, n, empty=(3,))
    queries = (rng.standard_normal((24, dims)) * 3).astype(np.float32)
    probes, r, t = 7, 60, 300
    want = port.ivf_search(so, cb, coarse, packed, boff, ioff, counts, ids, queries, probes=probes, r=r, t=t, threads=8)
    dev = torch.device("cuda", 0)
    d_q = torch.from_numpy(queries).to(dev)
    keys = torch.empty((world, len(queries), r), dtype=torch.int64, device=dev)
    qmap = torch.empty((len(queries), 2), dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream().cuda_stream
    params = qb.SearchParams(probes=probes, r=r, t=t)
    for rank in range(world):
        kw = shard_ivf_lists(s, packed, boff, ioff, counts, ids, rank, world, t_max=512)
        with qb.IvfIndex(s, cb, coarse, kw["packed"], kw["list_byte_off"], kw["list_id_off"], kw["list_count"],
                         kw["ids"], calib_packed=kw["calib_packed"], calib_byte_off=kw["calib_byte_off"],
                         calib_count=kw["calib_count"], global_list_count=kw["global_list_count"]) as shard:
            if rank == 0:  # t beyond a truncated head is refused, never clamped (dist.py:49)
                with pytest.raises(qb.QadcError) as e:
                    shard.search_device(d_q, qb.SearchParams(probes=probes, r=r, t=513), None, None, None,
                                        d_keys=keys[rank], d_map=qmap, stream=stream)
                assert e.value.kind == "config"
            shard.search_device(d_q, params, None, None, None, d_keys=keys[rank], d_map=qmap, stream=stream)
            torch.cuda.synchronize()
    d_ids = torch.empty((len(queries), r), dtype=torch.int32, device=dev)
    d_dists = torch.empty((len(queries), r), dtype=torch.float32, device=dev)
    d_counts = torch.empty((len(queries),), dtype=torch.int32, device=dev)
    qb.merge_topk_device(keys, world, len(queries), r, qmap, d_ids, d_dists, d_counts, 0, stream=stream)
    torch.cuda.synchronize()
    counts_g = d_counts.cpu().numpy().astype(np.uint32)
    ids_g = d_ids.cpu().numpy().view(np.uint32)
    dists_g = d_dists.cpu().numpy()
    assert np.array_equal(counts_g, want[2])
    for qi in range(len(queries)):
        c = int(want[2][qi])
        assert np.array_equal(ids_g[qi, :c], want[0][qi, :c]) and bits_equal(dists_g[qi, :c], want[1][qi, :c])


def test_ivf_probe_order_massive_ties(port):
    """2100 coarse centroids of which 2080 coincide: every distance ties, the fast probe selection overflows its
    candidate buffer and must fall back to the radix path; order is still (distance, cell) exact."""
    dims, text, k_cells = 32, "8x{4,4}", 2100
    rng = np.random.default_rng(31)
    s, so = qb.allocate_dims(dims, text), port.spec(dims, text)
    cb = rng.standard_normal(s.cb_floats).astype(np.float32)
    coarse = np.tile(rng.standard_normal((1, dims)).astype(np.float32), (k_cells, 1))
    coarse[:20] = rng.standard_normal((20, dims)).astype(np.float32) * 0.1
    packed, boff, ioff, counts, ids = _ivf_lists(rng, s, k_cells, 6000)
    queries = rng.standard_normal((5, dims)).astype(np.float32)
    with qb.IvfIndex(s, cb, coarse, packed, boff, ioff, counts, ids) as idx:
        for a in (7, 64, 256):
            order = idx.probe_order(queries, a)
            for qi in range(5):
                assert np.array_equal(order[qi], port.probe_order(dims, coarse, queries[qi], a))
        want = port.ivf_search(so, cb, coarse, packed, boff, ioff, counts, ids, queries, probes=40, r=20, t=100)
        got = idx.search(queries, qb.SearchParams(probes=40, r=20, t=100))
        assert np.array_equal(got.counts, want[2])
        for qi in range(5):
            c = int(want[2][qi])
            assert np.array_equal(got.ids[qi, :c], want[0][qi, :c]) and bits_equal(got.dists[qi, :c], want[1][qi, :c])


# ------------------------------------------------------------------ rerank (N4) --

@pytest.mark.parametrize("name", FLAT)
def test_golden_flat_rerank(golden, name):
    g = golden(name)
    s = qb.allocate_dims(int(g["dims"]), str(g["spec"]))
    with qb.FlatIndex(s, g["codebook"], g["packed"], int(g["count"])) as idx:
        res = idx.search(g["queries"], qb.SearchParams(r=int(g["r"]), t=int(g["t"]), rerank=True))
    assert np.array_equal(res.counts, g["counts"])
    for qi in range(len(g["queries"])):
        c = int(res.counts[qi])
        assert np.array_equal(res.ids[qi, :c], g["ids_rr"][qi, :c]) and bits_equal(res.dists[qi, :c], g["dists_rr"][qi, :c])


@pytest.mark.parametrize("name", ["ivf_irr655.npz", "ivf_pq16x4.npz"])
def test_golden_ivf_rerank(golden, name):
    g = golden(name)
    s = qb.allocate_dims(int(g["dims"]), str(g["spec"]))
    pr = int(g["probe_list"][1])
    with qb.IvfIndex(s, g["codebook"], g["coarse"], g["packed"], g["list_byte_off"], g["list_id_off"],
                     g["list_count"], g["list_ids"]) as idx:
        res = idx.search(g["queries"], qb.SearchParams(probes=pr, r=int(g["r"]), t=int(g["t"]), rerank=True))
    for qi in range(len(g["queries"])):
        c = int(res.counts[qi])
        assert np.array_equal(res.ids[qi, :c], g["ids_rr"][qi, :c]) and bits_equal(res.dists[qi, :c], g["dists_rr"][qi, :c])
    bad = g["list_ids"].copy()
    bad[3] = bad.size + 5
    with pytest.raises(qb.QadcError) as e:  # index.hpp:372
        qb.IvfIndex(s, g["codebook"], g["coarse"], g["packed"], g["list_byte_off"], g["list_id_off"], g["list_count"], bad)
    assert e.value.kind == "corruption"


def test_rerank_vs_oracle_and_shard_refusal(port):
    rng = np.random.default_rng(17)
    dims, text = 128, "16x{4,4}"
    s, so = qb.allocate_dims(dims, text), port.spec(dims, text)
    cb = (rng.standard_normal(s.cb_floats) * 2).astype(np.float32)
    n = 50000
    pk = qb.pack_list(s, random_codes(s, n, seed=5))
    queries = (rng.standard_normal((40, dims)) * 2).astype(np.float32)
    want = port.flat_search(so, cb, pk, n, queries, r=100, t=400, family=0x100, threads=8)
    with qb.FlatIndex(s, cb, pk, n) as idx:
        got = idx.search(queries, qb.SearchParams(rerank=True))
        assert np.array_equal(got.ids, want[0]) and bits_equal(got.dists, want[1])
    with qb.FlatIndex(s, cb, pk, n, base_id=1000) as shard:
        with pytest.raises(qb.QadcError) as e:
            shard.search(queries, qb.SearchParams(rerank=True))
        assert e.value.kind == "config"


# ------------------------------------------------ N1: reference containers opened directly --

@pytest.mark.parametrize("stem", ["flat_pq16x4", "flat_irr655", "flat_pq16x4_short"])
def test_open_qflt_written_by_reference(golden, stem):
    """QFLT written by the reference's save_flat_index (io.hpp:276-284): open directly, search, compare."""
    from tests.conftest import GOLDEN
    g = golden(stem + ".npz")
    with qb.open_index(GOLDEN / (stem + ".qflt")) as idx:
        assert isinstance(idx, qb.FlatIndex) and idx.size() == int(g["count"])
        assert np.array_equal(idx.download_codes(0, idx.size()), g["codes"])
        res = idx.search(g["queries"], qb.SearchParams(r=int(g["r"]), t=int(g["t"])))
    assert np.array_equal(res.counts, g["counts"])
    for qi in range(len(g["queries"])):
        c = int(res.counts[qi])
        assert np.array_equal(res.ids[qi, :c], g["ids"][qi, :c]) and bits_equal(res.dists[qi, :c], g["dists"][qi, :c])


@pytest.mark.parametrize("stem", ["ivf_irr655", "ivf_pq16x4"])
def test_open_qivf_written_by_reference(golden, stem):
    from tests.conftest import GOLDEN
    g = golden(stem + ".npz")
    with qb.open_index(GOLDEN / (stem + ".qivf")) as idx:
        assert isinstance(idx, qb.IvfIndex) and idx.cells() == len(g["list_count"]) and idx.size() == int(g["list_count"].sum())
        for pr in g["probe_list"]:
            res = idx.search(g["queries"], qb.SearchParams(probes=int(pr), r=int(g["r"]), t=int(g["t"])))
            assert np.array_equal(res.counts, g[f"counts_p{pr}"])
            for qi in range(len(g["queries"])):
                c = int(res.counts[qi])
                assert np.array_equal(res.ids[qi, :c], g[f"ids_p{pr}"][qi, :c])
                assert bits_equal(res.dists[qi, :c], g[f"dists_p{pr}"][qi, :c])


# ------------------------------------------------------------------ N3: IVF list construction --

@pytest.mark.parametrize("name", ["ivfbuild_pq8x4.npz", "ivfbuild_irr655.npz"])
def test_ivf_build_lists_match_reference_build(golden, name):
    """GPU assignment + residual encode + pack reproduces, byte for byte, the lists the reference's
    IvfIndex::build produced from the same vectors (fixture holds its centroids, codebook, lists and ids)."""
    g = golden(name)
    s = qb.allocate_dims(int(g["dims"]), str(g["spec"]))
    built = qb.build_ivf_lists(s, g["codebook"], g["coarse"], g["vectors"])
    for key in ("packed", "list_byte_off", "list_id_off", "list_count", "ids"):
        assert np.array_equal(built[key], g[key]), key


def test_ivf_build_lists_grouping_and_packing_many_cells():
    """qadc_ivf_build_lists (device histogram + scans + stable grouping + pack kernel) against the host restatement of
    index.hpp:219-227 on the same assignment: more cells than vectors in places (empty lists), ragged tails in every
    block size / word width, ids ascending inside every list, offsets consistent with qadc_packed_bytes."""
    rng = np.random.default_rng(33)
    for dims, text, k, n in [(40, "10x{4,4}", 1000, 2500 + 7), (48, "6x{6,5,5}", 300, 20_011), (32, "4x{8}", 70, 5_000),
                             (64, "8x{8,8}", 17, 33)]:
        s = qb.allocate_dims(dims, text)
        cb = rng.standard_normal(s.cb_floats).astype(np.float32)
        coarse = (rng.standard_normal((k, dims)) * 3).astype(np.float32)
        v = (rng.standard_normal((n, dims)) * 3).astype(np.float32)
        built = qb.build_ivf_lists(s, cb, coarse, v)
        assign, codes = qb.ivf_assign_encode(s, cb, coarse, v)
        assert np.array_equal(built["assign"], assign)
        order = np.argsort(assign, kind="stable").astype(np.uint32)
        counts = np.bincount(assign, minlength=k).astype(np.uint64)
        assert np.array_equal(built["list_count"], counts) and np.array_equal(built["ids"], order)
        id_off = np.concatenate([[0], np.cumsum(counts)[:-1]]).astype(np.uint64)
        assert np.array_equal(built["list_id_off"], id_off)
        b = 0
        for c in range(k):
            assert int(built["list_byte_off"][c]) == b
            i0, cnt = int(id_off[c]), int(counts[c])
            want = qb.pack_list(s, codes[order[i0:i0 + cnt]]) if cnt else np.zeros(0, np.uint8)
            assert np.array_equal(built["packed"][b:b + want.size], want), (text, c)
            b += qb.packed_bytes(s, cnt)
        assert built["packed"].size == b


def test_ivf_assign_encode_vs_oracle_many_cells(port):
    """More cells than one CTA covers (cross-block reduction), duplicated centroids (ties to the lowest cell),
    a ragged vector count, NaN / infinite inputs (never win: cell 0, like the reference's '<' loop)."""
    rng = np.random.default_rng(12)
    dims, text, k = 40, "10x{4,4}", 1000
    s, so = qb.allocate_dims(dims, text), port.spec(dims, text)
    cb = rng.standard_normal(s.cb_floats).astype(np.float32)
    coarse = (rng.standard_normal((k, dims)) * 3).astype(np.float32)
    coarse[700] = coarse[5]
    coarse[999] = coarse[300]
    v = (rng.standard_normal((2500 + 7, dims)) * 3).astype(np.float32)
    v[0], v[1] = coarse[5], coarse[300]
    v[2, 3] = np.nan
    v[3, 0] = np.inf
    a, c = qb.ivf_assign_encode(s, cb, coarse, v)
    a2, c2 = port.ivf_assign_encode(so, cb, coarse, v)
    assert a[0] == 5 and a[1] == 300 and a[2] == 0 and a[3] == 0
    assert np.array_equal(a, a2)
    ok = np.ones(len(v), bool)
    ok[2:4] = False  # the residual of a NaN/inf vector encodes to whatever '<' on NaN picks; compared separately
    assert np.array_equal(c[ok], c2[ok])
    assert np.array_equal(c[~ok], c2[~ok])


def test_ivf_built_on_gpu_then_searched(port):
    """End to end: lists built on the GPU, opened, searched -- equal to the oracle searching the oracle-built lists."""
    rng = np.random.default_rng(13)
    dims, text, k, n = 48, "12x{6,5,5}", 64, 30000
    s, so = qb.allocate_dims(dims, text), port.spec(dims, text)
    centres = rng.standard_normal((k, dims)).astype(np.float32) * 4
    v = (centres[rng.integers(0, k, size=n)] + rng.standard_normal((n, dims))).astype(np.float32)
    cb = (rng.standard_normal(s.cb_floats) * 0.7).astype(np.float32)
    b = qb.build_ivf_lists(s, cb, centres, v)
    a2, c2 = port.ivf_assign_encode(so, cb, centres, v)
    assert np.array_equal(b["assign"], a2)
    queries = (centres[rng.integers(0, k, size=20)] + rng.standard_normal((20, dims))).astype(np.float32)
    want = port.ivf_search(so, cb, centres, b["packed"], b["list_byte_off"], b["list_id_off"], b["list_count"],
                           b["ids"], queries, probes=8, r=50, t=200, threads=4)
    with qb.IvfIndex(s, cb, centres, b["packed"], b["list_byte_off"], b["list_id_off"], b["list_count"],
                     b["ids"]) as idx:
        got = idx.search(queries, qb.SearchParams(probes=8, r=50, t=200))
    assert np.array_equal(got.ids, want[0]) and bits_equal(got.dists, want[1]) and np.array_equal(got.counts, want[2])


# ------------------------------------------------------------------ probe order at scale (tensor-core prefilter) --

def _empty_ivf(s, cb, coarse):
    k = coarse.shape[0]
    z64 = np.zeros(k, np.uint64)
    return qb.IvfIndex(s, cb, coarse, np.zeros(0, np.uint8), z64, z64, z64, np.zeros(0, np.uint32))


@pytest.mark.parametrize("offset,spread", [(0.0, 3.0), (100.0, 1.0), (-7.0, 0.01)])
def test_probe_order_prefilter_is_exact(port, offset, spread):
    """K >= 512 takes the bf16 tensor-core prefilter + exact re-evaluation (ivf_probe_tc.cu): the order must equal
    the reference's probe_order bit for bit -- for centred data, data with a large common offset, and tightly
    packed centroids; with exact ties (duplicated centroids: the lower cell first), for several probe counts,
    and identically with the prefilter switched off."""
    rng = np.random.default_rng(int(abs(offset) * 10 + spread * 100))
    dims, text, k = 40, "10x{4,4}", 2048 + 3
    s = qb.allocate_dims(dims, text)
    cb = rng.standard_normal(s.cb_floats).astype(np.float32)
    coarse = (offset + rng.standard_normal((k, dims)) * spread).astype(np.float32)
    coarse[1500] = coarse[11]
    coarse[2050] = coarse[11]
    coarse[900] = coarse[33]
    queries = (offset + rng.standard_normal((37, dims)) * spread).astype(np.float32)
    queries[0] = coarse[11]
    queries[1] = coarse[33] + np.float32(1e-3)
    with _empty_ivf(s, cb, coarse) as idx:
        for a in (1, 3, 64, 256):
            got = idx.probe_order(queries, a)
            idx.set_option("probe_tc", 0)
            exact = idx.probe_order(queries, a)
            idx.set_option("probe_tc", 1)
            assert np.array_equal(got, exact), a
            for qi in range(len(queries)):
                assert np.array_equal(got[qi], port.probe_order(dims, coarse, queries[qi], a)), (a, qi)
        assert idx.probe_order(queries, 3)[0].tolist() == [11, 1500, 2050]


def test_probe_order_prefilter_bf16_midpoints(port):
    """Adversarial inputs for the prefilter's error bound: low dimension, every coordinate of every
    centroid and query sits just BELOW a bf16 rounding midpoint (1 + (2k+1) 2^-8 - 2^-20) * 2^e, so each input loses
    almost the full unit roundoff 2^-8 in the same direction; the centroid set is symmetric (c and -c) so the mean
    is exactly zero and the bf16 images are the rounded inputs themselves.  Distances to the near centroids differ
    by less than the bf16-induced error, so a too-small eps drops true top-a cells; the order must still be the
    reference's, bit for bit, and equal to the exact kernels'."""
    rng = np.random.default_rng(77)
    dims, text, half = 8, "2x{4,4}", 600
    s = qb.allocate_dims(dims, text)
    cb = rng.standard_normal(s.cb_floats).astype(np.float32)

    def below_midpoint(shape):
        k = rng.integers(0, 64, size=shape)           # which bf16 interval of [1, 2): mantissa 7 bits -> 128 intervals
        e = rng.integers(-1, 2, size=shape)           # exponents -1..1
        sign = rng.choice([-1.0, 1.0], size=shape)
        v = (1.0 + (2 * k + 1) * 2.0 ** -8 - 2.0 ** -20) * 2.0 ** e
        return (sign * v).astype(np.float32)

    pos = below_midpoint((half, dims))
    coarse = np.concatenate([pos, -pos]).astype(np.float32)          # K = 1200, mean exactly 0
    queries = below_midpoint((40, dims))
    queries[:10] = coarse[rng.integers(0, 2 * half, size=10)] * np.float32(1.0 + 2.0 ** -9)
    with _empty_ivf(s, cb, coarse) as idx:
        for a in (1, 5, 64, 256):
            got = idx.probe_order(queries, a)
            idx.set_option("probe_tc", 0)
            exact = idx.probe_order(queries, a)
            idx.set_option("probe_tc", 1)
            assert np.array_equal(got, exact), a
            for qi in range(len(queries)):
                assert np.array_equal(got[qi], port.probe_order(dims, coarse, queries[qi], a)), (a, qi)


def test_probe_order_prefilter_overflow_falls_back(port):
    """3000 identical centroids: every one of them is a candidate, the candidate buffer overflows and the query
    is redone by the exact kernels (ties resolve to the lowest cells)."""
    rng = np.random.default_rng(8)
    dims, text, k = 32, "8x{4,4}", 4096
    s = qb.allocate_dims(dims, text)
    cb = rng.standard_normal(s.cb_floats).astype(np.float32)
    coarse = (rng.standard_normal((k, dims)) * 2).astype(np.float32)
    coarse[500:3500] = coarse[500]
    queries = (rng.standard_normal((9, dims)) * 2).astype(np.float32)
    queries[0] = coarse[500]
    with _empty_ivf(s, cb, coarse) as idx:
        got = idx.probe_order(queries, 32)
    assert got[0].tolist() == list(range(500, 532))
    for qi in range(len(queries)):
        assert np.array_equal(got[qi], port.probe_order(dims, coarse, queries[qi], 32)), qi


@pytest.mark.parametrize("dims,text,k_cells,n,probes,nq", [(96, "12x{6,5,5}", 1024, 400000, 24, 96),
                                                           (128, "16x{4,4}", 600, 200000, 12, 70),
                                                           (64, "8x{8,8}", 512, 120000, 9, 50)])
def test_ivf_search_many_cells_vs_oracle(port, dims, text, k_cells, n, probes, nq):
    """The batch-scale IVF stages -- tensor-core probe prefilter (K >= 512), register-tiled residual tables, fused
    quantize + tile pack, 32/64-row tiles with two tile buffers -- against the oracle end to end, on clustered
    queries (many queries share cells, so tiles are full) with a skewed list-length distribution."""
    rng = np.random.default_rng(k_cells + probes)
    s, so = qb.allocate_dims(dims, text), port.spec(dims, text)
    cb = (rng.standard_normal(s.cb_floats) * 0.8).astype(np.float32)
    coarse = (rng.standard_normal((k_cells, dims)) * 2 + 5.0).astype(np.float32)
    # skewed list sizes: a few long lists, many short ones, two empty cells
    w = rng.pareto(1.5, size=k_cells) + 0.05
    w[[3, k_cells - 1]] = 0
    assign = rng.choice(k_cells, size=n, p=w / w.sum())
    codes = random_codes(s, n, seed=5)
    order = np.argsort(assign, kind="stable")
    counts = np.bincount(assign, minlength=k_cells).astype(np.uint64)
    ioff = np.concatenate([[0], np.cumsum(counts)[:-1]]).astype(np.uint64)
    parts, boff, b = [], [], 0
    for c in range(k_cells):
        boff.append(b)
        if counts[c]:
            parts.append(qb.pack_list(s, codes[order[int(ioff[c]):int(ioff[c] + counts[c])]]))
            b += parts[-1].size
    packed, boff, ids = np.concatenate(parts), np.array(boff, np.uint64), order.astype(np.uint32)
    hot = rng.integers(0, k_cells, size=6)
    queries = (coarse[hot[rng.integers(0, 6, size=nq)]] + rng.standard_normal((nq, dims)) * 0.7).astype(np.float32)
    with qb.IvfIndex(s, cb, coarse, packed, boff, ioff, counts, ids) as idx:
        for pr, r, t in [(probes, 100, 400), (3, 20, 60)]:
            want = port.ivf_search(so, cb, coarse, packed, boff, ioff, counts, ids, queries, probes=pr, r=r, t=t, threads=8)
            got = idx.search(queries, qb.SearchParams(probes=pr, r=r, t=t))
            assert np.array_equal(got.counts, want[2]), (pr, r, t)
            assert np.array_equal(got.ids, want[0]), (pr, r, t)
            assert bits_equal(got.dists, want[1]), (pr, r, t)
            rr = port.ivf_search(so, cb, coarse, packed, boff, ioff, counts, ids, queries, probes=pr, r=r, t=t,
                                 threads=8, family=0x100)
            got_rr = idx.search(queries, qb.SearchParams(probes=pr, r=r, t=t, rerank=True))
            assert np.array_equal(got_rr.ids, rr[0]) and bits_equal(got_rr.dists, rr[1]), ("rerank", pr)


def test_full_size_c2_properties(port):
    """BASELINE configs[1] at full size (12x{6,5,5}, d=96, N=1e7, Q=1e4 -- the default bench workload) through
    size-independent properties: for every query the result is full, sorted by (distance, id) and duplicate free;
    for a sample of queries the quantized tables equal the oracle's, every returned distance is the unquantized
    oracle ADC sum of that code, and no code of a 100k uniform sample beats the R-th result; and two queries are
    compared with the complete oracle search."""
    dims, text, n, nq, r, t = 96, "12x{6,5,5}", 10_000_000, 10_000, 100, 400
    s, so = qb.allocate_dims(dims, text), port.spec(dims, text)
    from paper_1812_09162_b200.synth import train_codebook
    cb = train_codebook(s, gaussian_mixture(20000, dims, seed=14), iters=3)
    codes = random_codes(s, n, seed=16)
    pk = qb.pack_list(s, codes)
    queries = gaussian_mixture(nq, dims, seed=13)
    with qb.FlatIndex(s, cb, pk, n) as idx:
        res = idx.search(queries, qb.SearchParams(r=r, t=t))
        check_q = np.arange(0, nq, 250)
        _, qluts, _ = idx.tables(queries[check_q], qb.SearchParams(r=r, t=t))
    assert np.all(res.counts == r)
    assert np.all(np.diff(res.dists, axis=1) >= 0)
    srt = np.sort(res.ids, axis=1)
    assert np.all(srt[:, 1:] != srt[:, :-1])
    bits = np.array(so.bits_list())
    off = np.concatenate([[0], np.cumsum(1 << bits)[:-1]])
    sample = np.random.default_rng(5).choice(n, size=100_000, replace=False)
    for k, qi in enumerate(check_q):
        lut = port.compute_tables(so, cb, queries[qi])
        pre = port.prefix_float(so, pk, n, lut, t)
        dmin, dmax = port.calibrate(so, lut, pre, r)
        qlut, _, delta, own = port.quantize(so, lut, dmin, dmax, 16)
        assert np.array_equal(qlut, qluts[k]), qi
        q32 = qlut.astype(np.uint32)
        sums = np.minimum(q32[off[None, :] + codes[res.ids[qi]].astype(np.int64)].sum(1), 65535)
        want = (sums.astype(np.float32) * delta + own).astype(np.float32)
        assert bits_equal(res.dists[qi], want), qi
        keys = sums.astype(np.int64) << 32 | res.ids[qi].astype(np.int64)
        assert np.all(np.diff(keys) > 0), qi
        ssum = np.minimum(q32[off[None, :] + codes[sample].astype(np.int64)].sum(1), 65535)
        skeys = ssum.astype(np.int64) << 32 | sample.astype(np.int64)
        assert np.all(skeys[~np.isin(sample, res.ids[qi])] > keys[-1]), qi
    ref = port.flat_search(so, cb, pk, n, queries[:2], r=r, t=t, threads=2)
    assert np.array_equal(res.ids[:2], ref[0]) and bits_equal(res.dists[:2], ref[1])


def test_c5_shape_ivf_sampled_queries_vs_oracle(port):
    """BASELINE configs[4] shape (K=16384 cells, d=128, 12x{6,5,5}, nprobe=64, R=100, t=400) on a smaller database
    (8e6 codes, skewed list lengths) and 2000 queries: the probe order of every sampled query and its complete
    result (ids, distances, counts) equal the oracle's.  This is the path the C5 bench line times: tensor-core probe
    prefilter at the real K, 128k (query, cell) pairs of residual tables, fused quantize + pack, duplicated-line
    32-row tiles, two scan rounds."""
    rng = np.random.default_rng(55)
    dims, text, k_cells, n, nq, probes = 128, "12x{6,5,5}", 16384, 8_000_000, 2000, 64
    s, so = qb.allocate_dims(dims, text), port.spec(dims, text)
    centres = (rng.standard_normal((64, dims)) * 3).astype(np.float32)
    coarse = (centres[rng.integers(0, 64, size=k_cells)] + rng.standard_normal((k_cells, dims))).astype(np.float32)
    cb = (rng.standard_normal(s.cb_floats) * 0.6).astype(np.float32)
    w = rng.pareto(2.0, size=k_cells) + 0.2
    counts = np.floor(w / w.sum() * n).astype(np.uint64)
    counts[:5] = [0, 1, 15, 16, 17]  # empty / tiny lists next to the long ones
    pbytes = np.array([qb.packed_bytes(s, int(c)) for c in counts], dtype=np.uint64)
    boff = np.concatenate([[0], np.cumsum(pbytes)[:-1]]).astype(np.uint64)
    ioff = np.concatenate([[0], np.cumsum(counts)[:-1]]).astype(np.uint64)
    packed = rng.integers(0, 256, size=int(pbytes.sum()), dtype=np.uint8)  # every {6,5,5} bit pattern is a valid code
    ids = rng.permutation(int(counts.sum())).astype(np.uint32)
    queries = (centres[rng.integers(0, 64, size=nq)] + rng.standard_normal((nq, dims)) * 1.2).astype(np.float32)
    with qb.IvfIndex(s, cb, coarse, packed, boff, ioff, counts, ids) as idx:
        got = idx.search(queries, qb.SearchParams(probes=probes, r=100, t=400))
        order = idx.probe_order(queries, probes)
    assert np.all(np.diff(got.dists, axis=1)[got.counts == 100] >= 0)
    sel = np.arange(0, nq, 67)
    for qi in sel:
        assert np.array_equal(order[qi], port.probe_order(dims, coarse, queries[qi], probes)), qi
    want = port.ivf_search(so, cb, coarse, packed, boff, ioff, counts, ids, queries[sel], probes=probes, r=100, t=400,
                           threads=8)
    assert np.array_equal(got.counts[sel], want[2])
    assert np.array_equal(got.ids[sel], want[0])
    assert bits_equal(got.dists[sel], want[1])


def test_concurrent_calls_on_one_handle_serialise():
    """The reference lets any number of threads call search() on one index (the CLI's worker pool,
    pqscan_cli.cpp:141-166).  A GPU handle owns workspaces and a stream, so concurrent calls must serialise inside
    the library: every thread gets exactly the result a lone caller gets."""
    import threading
    rng = np.random.default_rng(21)
    dims, text, n = 96, "12x{6,5,5}", 200_000
    s = qb.allocate_dims(dims, text)
    cb = (rng.standard_normal(s.cb_floats) * 2).astype(np.float32)
    pk = qb.pack_list(s, random_codes(s, n, seed=3))
    batches = [(rng.standard_normal((nq, dims)) * 2).astype(np.float32) for nq in (1, 7, 64, 33, 1, 128, 5, 16)]
    with qb.FlatIndex(s, cb, pk, n) as idx:
        want = [idx.search(q) for q in batches]
        got = [None] * len(batches)
        errors = []

        def work(k):
            try:
                for _ in range(3):
                    got[k] = idx.search(batches[k])
            except Exception as e:  # noqa: BLE001
                errors.append(e)

        threads = [threading.Thread(target=work, args=(k,)) for k in range(len(batches))]
        for th in threads:
            th.start()
        for th in threads:
            th.join()
    assert not errors, errors
    for w, g in zip(want, got):
        assert np.array_equal(w.ids, g.ids) and bits_equal(w.dists, g.dists) and np.array_equal(w.counts, g.counts)


@pytest.mark.parametrize("dims,text,variants", [
    (128, "16x{4,4}", [0, 1, 2, 3, 7, 9, 12, 13, 14]),   # f16x8, f32x2, u16x1, u8x1, f16x4-c4, merged pair tables, tcgen05 one-hot GEMM (dense, 2:4 sparse, sparse on CTA pairs)
    (96, "12x{6,5,5}", [1, 2, 3, 4, 5, 6, 8, 10, 11]),   # f32x2, u16x1, u8x1, f16x4h, -c2, -c4, -c4d, merged quad, 16-row quad
    (64, "12x{6,6,4}", [1, 2, 4, 5, 10]),        # f32x2, u16x1, f16x4h, -c2, merged quad (default)
    (60, "12x{5,5,5}", [1, 2, 4, 5, 10]),        # f32x2, u16x1, f16x4h, -c2, merged quad (default)
    (64, "8x{8,8}", [2, 3, 6]),                  # u16x1, u8x1, f16x4h-c4 (default)
    (64, "8x{8}", [2, 3, 7]),                    # u16x1, u8x1, f16x4-c4
])
def test_every_scan_variant_is_exact(port, dims, text, variants):
    """Each scan variant that can serve a spec (the planner's default and every fallback layout), forced through
    qadc_set_option, returns the oracle's result bit for bit -- flat search with a ragged query count, and the
    variant name reported by the library matches the one requested."""
    rng = np.random.default_rng(len(text) + dims)
    s, so = qb.allocate_dims(dims, text), port.spec(dims, text)
    cb = (rng.standard_normal(s.cb_floats) * 2).astype(np.float32)
    n, nq = 70_001, 77
    pk = qb.pack_list(s, random_codes(s, n, seed=11))
    queries = (rng.standard_normal((nq, dims)) * 2).astype(np.float32)
    want = port.flat_search(so, cb, pk, n, queries, r=100, t=400, threads=8)
    with qb.FlatIndex(s, cb, pk, n) as idx:
        ran = 0
        for v in [-1] + variants:
            idx.set_option("force_variant", v)
            try:
                got = idx.search(queries, qb.SearchParams(r=100, t=400))
            except qb.QadcError as e:  # a layout whose tables do not fit shared memory for this spec
                assert e.kind == "config", (v, e)
                continue
            if v >= 0:
                assert idx.stats().scan_variant == v
            assert np.array_equal(got.ids, want[0]), v
            assert bits_equal(got.dists, want[1]), v
            assert np.array_equal(got.counts, want[2]), v
            ran += 1
        assert ran >= len(variants)  # the default plus all but at most one fallback must run


@pytest.mark.parametrize("variant", [12, 13, 14])
@pytest.mark.parametrize("distinct,r,cand_cap", [(40, 100, 0), (3, 257, 0), (500, 1000, 512)])
def test_tensor_core_search_with_massive_ties(port, variant, distinct, r, cand_cap):
    """Flat search through each tensor-core form over a list made of a handful of DISTINCT codes repeated -- every
    quantized sum ties with thousands of others, so the result is decided by ids alone (heap.hpp:46-47).  Covers the
    threshold rows that exclude ties where ids only grow, the lane-local admission queues (dense admissions, queue-full
    retries) and, with a small candidate buffer, the overflow retry; 700 queries = a ragged last tile and, for the pair
    form, an odd number of 240-query tiles (its second tile of the last job is half padding)."""
    rng = np.random.default_rng(distinct * 7 + r)
    dims, text = 64, "16x{4,4}"
    s, so = qb.allocate_dims(dims, text), port.spec(dims, text)
    cb = (rng.standard_normal(s.cb_floats) * 2).astype(np.float32)
    n, nq = 300_007, 700
    pool = random_codes(s, distinct, seed=distinct)
    codes = pool[rng.integers(0, distinct, size=n)]
    pk = qb.pack_list(s, codes)
    queries = (rng.standard_normal((nq, dims)) * 2).astype(np.float32)
    want = port.flat_search(so, cb, pk, n, queries, r=r, t=max(r, 400), threads=8)
    with qb.FlatIndex(s, cb, pk, n) as idx:
        idx.set_option("force_variant", variant)
        if cand_cap:
            idx.set_option("cand_cap", cand_cap)
        got = idx.search(queries, qb.SearchParams(r=r, t=max(r, 400)))
        assert idx.stats().scan_variant == variant
        if cand_cap:
            assert idx.stats().overflow_retries >= 1
    assert np.array_equal(got.ids, want[0])
    assert bits_equal(got.dists, want[1])
    assert np.array_equal(got.counts, want[2])


@pytest.mark.parametrize("dims,text", [(128, "16x{4,4}"), (96, "12x{6,5,5}"), (64, "12x{6,6,4}"), (60, "12x{5,5,5}"),
                                       (64, "8x{8,8}"), (64, "8x{8}")])
def test_randomised_search_parameters_vs_oracle(port, dims, text):
    """Random (n, nq, r, t) around the edges the planner's default variants see: one query, ragged tiles, r = 1,
    r close to n, t = r and t > n, lists shorter than one stage buffer and longer than several segments."""
    rng = np.random.default_rng(abs(hash(text)) % 9973)
    s, so = qb.allocate_dims(dims, text), port.spec(dims, text)
    cb = (rng.standard_normal(s.cb_floats) * 1.7).astype(np.float32)
    for n, nq, r, t in [(1, 1, 1, 1), (17, 3, 5, 5), (700, 1, 100, 400), (5000, 33, 1, 1), (40000, 16, 250, 250),
                        (300000, 47, 100, 400), (9000, 129, 1000, 5000), (70000, 5, 999, 1000)]:
        pk = qb.pack_list(s, random_codes(s, n, seed=n))
        queries = (rng.standard_normal((nq, dims)) * 1.7).astype(np.float32)
        want = port.flat_search(so, cb, pk, n, queries, r=r, t=t, threads=8)
        with qb.FlatIndex(s, cb, pk, n) as idx:
            got = idx.search(queries, qb.SearchParams(r=r, t=t))
        assert np.array_equal(got.counts, want[2]), (n, nq, r, t)
        for qi in range(nq):
            c = int(want[2][qi])
            assert np.array_equal(got.ids[qi, :c], want[0][qi, :c]), (n, nq, r, t, qi)
            assert bits_equal(got.dists[qi, :c], want[1][qi, :c]), (n, nq, r, t, qi)


@pytest.mark.parametrize("dims,text,variants", [(96, "12x{6,5,5}", [1, 2, 4, 5, 6, 8, 11]), (64, "12x{6,6,4}", [4, 5, 6, 11]),
                                                (60, "12x{5,5,5}", [4, 5, 6, 11]), (64, "8x{8,8}", [2, 6]),
                                                (64, "16x{4,4}", [0, 1, 7])])
def test_every_ivf_tile_layout_is_exact(port, dims, text, variants):
    """The IVF batch path writes its LUT tiles itself (fused quantize + pack): every tile layout it can be asked
    for -- 128 / 64 / 32-row tiles, word-pair and byte-pair interleaved lines, duplicated lines, the fallbacks --
    returns the oracle's result bit for bit."""
    rng = np.random.default_rng(len(text) * 7 + dims)
    s, so = qb.allocate_dims(dims, text), port.spec(dims, text)
    k_cells, n, nq, probes = 40, 60000, 90, 6
    cb = (rng.standard_normal(s.cb_floats) * 1.2).astype(np.float32)
    coarse = (rng.standard_normal((k_cells, dims)) * 3).astype(np.float32)
    packed, boff, ioff, counts, ids = _ivf_lists(rng, s, k_cells, n, empty=(2,))
    hot = rng.integers(0, k_cells, size=4)
    queries = (coarse[hot[rng.integers(0, 4, size=nq)]] + rng.standard_normal((nq, dims))).astype(np.float32)
    want = port.ivf_search(so, cb, coarse, packed, boff, ioff, counts, ids, queries, probes=probes, r=60, t=300, threads=8)
    with qb.IvfIndex(s, cb, coarse, packed, boff, ioff, counts, ids) as idx:
        ran = 0
        for v in [-1] + variants:
            idx.set_option("force_variant", v)
            try:
                got = idx.search(queries, qb.SearchParams(probes=probes, r=60, t=300))
            except qb.QadcError as e:
                assert e.kind == "config", (v, e)
                continue
            assert np.array_equal(got.counts, want[2]), v
            assert np.array_equal(got.ids, want[0]), v
            assert bits_equal(got.dists, want[1]), v
            ran += 1
        assert ran >= 2


@pytest.mark.parametrize("dims,text", [(96, "12x{6,5,5}"), (64, "12x{6,6,4}"), (60, "12x{5,5,5}"), (64, "8x{8,8}"),
                                       (64, "16x{4,4}"), (32, "8x{8}")])
def test_randomised_ivf_parameters_vs_oracle(port, dims, text):
    """Random (cells, n, nq, probes, r, t) for the IVF batch path with the planner's own choices: few and many rows
    per cell (every tile height gets picked somewhere), probes from 1 to all cells, r = 1 .. 300, t = r .. > n,
    empty and one-code lists."""
    rng = np.random.default_rng(abs(hash(text)) % 7919)
    s, so = qb.allocate_dims(dims, text), port.spec(dims, text)
    cb = (rng.standard_normal(s.cb_floats) * 1.3).astype(np.float32)
    for k_cells, n, nq, probes, r, t in [(3, 50, 2, 3, 1, 1), (17, 4000, 40, 4, 10, 10), (64, 50000, 300, 2, 100, 400),
                                         (600, 90000, 25, 37, 300, 300), (9, 30000, 513, 9, 50, 16000),
                                         (200, 2500, 64, 200, 5, 40)]:
        coarse = (rng.standard_normal((k_cells, dims)) * 3).astype(np.float32)
        empty = (1,) if k_cells > 2 else ()
        packed, boff, ioff, counts, ids = _ivf_lists(rng, s, k_cells, n, empty=empty)
        hot = rng.integers(0, k_cells, size=max(2, k_cells // 8))
        queries = (coarse[hot[rng.integers(0, len(hot), size=nq)]] + rng.standard_normal((nq, dims)) * 1.5).astype(np.float32)
        want = port.ivf_search(so, cb, coarse, packed, boff, ioff, counts, ids, queries, probes=probes, r=r, t=t, threads=8)
        with qb.IvfIndex(s, cb, coarse, packed, boff, ioff, counts, ids) as idx:
            got = idx.search(queries, qb.SearchParams(probes=probes, r=r, t=t))
        assert np.array_equal(got.counts, want[2]), (k_cells, n, nq, probes, r, t)
        for qi in range(nq):
            c = int(want[2][qi])
            assert np.array_equal(got.ids[qi, :c], want[0][qi, :c]), (k_cells, n, nq, probes, r, t, qi)
            assert bits_equal(got.dists[qi, :c], want[1][qi, :c]), (k_cells, n, nq, probes, r, t, qi)
