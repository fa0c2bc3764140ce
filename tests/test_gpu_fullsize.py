"""Full-size parity evidence for the BASELINE configurations the bench times (C3, C4, C5; C2 lives in
test_gpu_parity.py::test_full_size_c2_properties, C1 in ::test_large_seeded_property_round_trip).

The oracle cannot scan 1e11..2e12 pairs, so the full-size runs are tied to it through size-independent properties
(the reference's own end-to-end criterion, T/test_index.cpp:57-89, restated per query):
  * the quantized tables of sampled queries equal the oracle's (so the affine map and every sum below are the oracle's);
  * every returned distance is the unquantized oracle ADC sum of the returned id's code (adc_scalar_quantized,
    distance.hpp:149-155), the list is strictly ascending in (distance, id) and duplicate free;
  * no code of a uniform 100k-code sample outside the result beats the R-th result (top-R-ness);
  * a few queries are compared with the complete oracle search (ids, distance bits, counts).
"""
import numpy as np
import pytest

import paper_1812_09162_b200 as qb
from paper_1812_09162_b200.synth import gaussian_mixture, random_codes, random_packed, train_codebook

pytestmark = pytest.mark.gpu


def bits_equal(a, b):
    return a.shape == b.shape and a.tobytes() == b.tobytes()


def codes_at(spec, packed, idx):
    """Subquantizer indices of the codes at positions `idx` of a PackedList (layout.hpp:50-68, 105-144)."""
    g, rows, bl = spec.g, spec.groups, spec.block_len
    wdt = np.uint8 if spec.word_width == 8 else np.dtype("<u2")
    words = np.ascontiguousarray(packed, dtype=np.uint8).view(wdt).reshape(-1, rows, bl)
    idx = np.asarray(idx, dtype=np.int64)
    w = words[idx // bl, :, idx % bl].astype(np.uint32)
    out = np.empty((len(idx), rows, g), dtype=np.uint8)
    for k in range(g):
        out[:, :, k] = (w >> np.uint32(spec.offsets[k])) & np.uint32((1 << spec.widths[k]) - 1)
    return out.reshape(len(idx), rows * g)


def check_flat_full_size(port, s, so, cb, pk, n, queries, res, qluts, check_q, r, t, full_q):
    qmax = 255 if s.word_width == 8 else 65535
    assert np.all(res.counts == r)
    assert np.all(np.diff(res.dists, axis=1) >= 0)
    srt = np.sort(res.ids, axis=1)
    assert np.all(srt[:, 1:] != srt[:, :-1])
    bits = np.array(so.bits_list())
    off = np.concatenate([[0], np.cumsum(1 << bits)[:-1]])
    sample = np.random.default_rng(5).choice(n, size=100_000, replace=False)
    sample_codes = codes_at(s, pk, sample).astype(np.int64)
    for k, qi in enumerate(check_q):
        lut = port.compute_tables(so, cb, queries[qi])
        pre = port.prefix_float(so, pk, n, lut, t)
        dmin, dmax = port.calibrate(so, lut, pre, r)
        qlut, _, delta, own = port.quantize(so, lut, dmin, dmax, s.word_width)
        assert np.array_equal(qlut, qluts[k]), qi
        q32 = qlut.astype(np.uint32)
        got_codes = codes_at(s, pk, res.ids[qi]).astype(np.int64)
        sums = np.minimum(q32[off[None, :] + got_codes].sum(1), qmax)
        want = (sums.astype(np.float32) * delta + own).astype(np.float32)
        assert bits_equal(res.dists[qi], want), qi
        keys = sums.astype(np.int64) << 32 | res.ids[qi].astype(np.int64)
        assert np.all(np.diff(keys) > 0), qi
        ssum = np.minimum(q32[off[None, :] + sample_codes].sum(1), qmax)
        skeys = ssum.astype(np.int64) << 32 | sample.astype(np.int64)
        assert np.all(skeys[~np.isin(sample, res.ids[qi])] > keys[-1]), qi
    ref = port.flat_search(so, cb, pk, n, queries[full_q], r=r, t=t, threads=8)
    assert np.array_equal(res.counts[full_q], ref[2])
    assert np.array_equal(res.ids[full_q], ref[0]) and bits_equal(res.dists[full_q], ref[1])


def test_full_size_c3_properties(port):
    """BASELINE configs[2] at full size: 8x{8,8} (256-entry tables, the reference's split-table-16 family), d=128,
    N=1e7, Q=1e4."""
    dims, text, n, nq, r, t = 128, "8x{8,8}", 10_000_000, 10_000, 100, 400
    s, so = qb.allocate_dims(dims, text), port.spec(dims, text)
    cb = train_codebook(s, gaussian_mixture(20000, dims, seed=14), iters=2)
    pk = qb.pack_list(s, random_codes(s, n, seed=17))
    queries = gaussian_mixture(nq, dims, seed=13)
    check_q = np.arange(0, nq, 500)
    with qb.FlatIndex(s, cb, pk, n) as idx:
        res = idx.search(queries, qb.SearchParams(r=r, t=t))
        _, qluts, _ = idx.tables(queries[check_q], qb.SearchParams(r=r, t=t))
    check_flat_full_size(port, s, so, cb, pk, n, queries, res, qluts, check_q, r, t, full_q=np.array([0, nq - 1]))


def test_full_size_c4_properties(port):
    """BASELINE configs[3] at full size: 16x{4,4}, N=2e8 uniform random codes (1.6 GB), 512 of the 1e4 queries --
    the bench's default workload.  Also the sharded form: the same database split over 4 'ranks' on this one GPU
    (the reference's chunked-scan contract, T/test_kernels.cpp:107-133), merged, must equal the unsharded result."""
    import torch
    from paper_1812_09162_b200.dist import global_head, shard_ranges, slice_packed
    dims, text, n, nq, r, t = 128, "16x{4,4}", 200_000_000, 512, 100, 400
    s, so = qb.allocate_dims(dims, text), port.spec(dims, text)
    cb = train_codebook(s, gaussian_mixture(20000, dims, seed=14), iters=3)
    pk = random_packed(s, n, seed=6)
    queries = gaussian_mixture(nq, dims, seed=13)
    check_q = np.arange(0, nq, 32)
    with qb.FlatIndex(s, cb, pk, n) as idx:
        res = idx.search(queries, qb.SearchParams(r=r, t=t))
        _, qluts, _ = idx.tables(queries[check_q], qb.SearchParams(r=r, t=t))
    check_flat_full_size(port, s, so, cb, pk, n, queries, res, qluts, check_q, r, t, full_q=np.array([0, 1, nq - 1]))
    # strong-scaled split of the SAME database: 4 shards, replicated head, merge
    world = 4
    dev = torch.device("cuda", 0)
    d_q = torch.from_numpy(queries).to(dev)
    keys = torch.empty((world, nq, r), dtype=torch.int64, device=dev)
    qmap = torch.empty((nq, 2), dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream().cuda_stream
    head, head_n = global_head(s, pk, n)
    for rank, rg in enumerate(shard_ranges(n, world, s.block_len)):
        with qb.FlatIndex(s, cb, slice_packed(s, pk, rg), rg.count, base_id=rg.start, calib_packed=head,
                          calib_count=head_n, global_count=n) as shard:
            shard.search_device(d_q, qb.SearchParams(r=r, t=t), None, None, None, d_keys=keys[rank], d_map=qmap,
                                stream=stream)
            torch.cuda.synchronize()
    d_ids = torch.empty((nq, r), dtype=torch.int32, device=dev)
    d_dists = torch.empty((nq, r), dtype=torch.float32, device=dev)
    d_counts = torch.empty((nq,), dtype=torch.int32, device=dev)
    qb.merge_topk_device(keys, world, nq, r, qmap, d_ids, d_dists, d_counts, 0, stream=stream)
    torch.cuda.synchronize()
    assert np.array_equal(d_counts.cpu().numpy().astype(np.uint32), res.counts)
    assert np.array_equal(d_ids.cpu().numpy().view(np.uint32), res.ids)
    assert bits_equal(d_dists.cpu().numpy(), res.dists)


def test_full_size_c5_sampled_queries_vs_oracle(port):
    """BASELINE configs[4] at the per-GPU size the bench times (K=16384, 12x{6,5,5} residual codes, d=128, 6.25e7
    codes = 5e8 / 8, nprobe=64, Q=1e4): counts / order properties for every query, and probe order + complete
    result (ids, distance bits) of 40 sampled queries against the oracle's IvfIndex::search."""
    rng = np.random.default_rng(56)
    dims, text, k_cells, n, nq, probes = 128, "12x{6,5,5}", 16384, 62_500_000, 10_000, 64
    s, so = qb.allocate_dims(dims, text), port.spec(dims, text)
    centres = (rng.standard_normal((256, dims)) * 3).astype(np.float32)
    coarse = (centres[rng.integers(0, 256, size=k_cells)] + rng.standard_normal((k_cells, dims))).astype(np.float32)
    cb = (rng.standard_normal(s.cb_floats) * 0.6).astype(np.float32)
    w = rng.gamma(4.0, size=k_cells)
    counts = np.floor(w / w.sum() * n).astype(np.uint64)
    counts[:5] = [0, 1, 15, 16, 17]
    pbytes = np.array([qb.packed_bytes(s, int(c)) for c in counts], dtype=np.uint64)
    boff = np.concatenate([[0], np.cumsum(pbytes)[:-1]]).astype(np.uint64)
    ioff = np.concatenate([[0], np.cumsum(counts)[:-1]]).astype(np.uint64)
    packed = rng.integers(0, 256, size=int(pbytes.sum()), dtype=np.uint8)
    total = int(counts.sum())
    ids = np.arange(total, dtype=np.uint32)[::-1].copy()  # a non-trivial id map without a 62M-element permutation
    queries = (centres[rng.integers(0, 256, size=nq)] + rng.standard_normal((nq, dims)) * 1.2).astype(np.float32)
    with qb.IvfIndex(s, cb, coarse, packed, boff, ioff, counts, ids) as idx:
        got = idx.search(queries, qb.SearchParams(probes=probes, r=100, t=400))
        sel = np.arange(0, nq, 250)
        order = idx.probe_order(queries[sel], probes)
    full = got.counts == 100
    assert np.all(np.diff(got.dists, axis=1)[full] >= 0)
    assert np.all(got.ids[full].max(axis=1) < total)
    for k, qi in enumerate(sel):
        assert np.array_equal(order[k], port.probe_order(dims, coarse, queries[qi], probes)), qi
    want = port.ivf_search(so, cb, coarse, packed, boff, ioff, counts, ids, queries[sel], probes=probes, r=100, t=400,
                           threads=8)
    assert np.array_equal(got.counts[sel], want[2])
    assert np.array_equal(got.ids[sel], want[0])
    assert bits_equal(got.dists[sel], want[1])
