#!/usr/bin/env python
"""Generate tests/golden/*.npz by running the UNMODIFIED reference (oracle/_ref shim).

Run in the build container (needs /root/reference to have built oracle/_ref):

    python oracle/make_golden.py

Every fixture stores the inputs (spec string, codebook, packed list, queries, ...)
and the reference's outputs (float LUTs, calibration, quantized LUTs, top-R ids
and distances), so that both the plain-C port and the CUDA path can be checked
on machines where the reference tree does not exist.  Inputs are seeded
synthetic data (Gaussian blobs); no benchmark dataset items are involved.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from oracle.pyoracle import Oracle, build  # noqa: E402

GOLD = ROOT / "tests" / "golden"

FAMILIES = [
    # name, dims, spec, n_db
    ("pq16x4", 64, "16x{4,4}", 1500),
    ("irr655", 48, "12x{6,5,5}", 1300),
    ("irr664", 64, "12x{6,6,4}", 1100),
    ("irr555", 60, "12x{5,5,5}", 1000),
    ("split88", 32, "8x{8,8}", 1200),
    ("split8", 32, "8x{8}", 1400),
]


def blobs(rng, n, d, clusters=24, spread=1.0, scale=5.0):
    centers = rng.normal(size=(clusters, d)) * scale
    which = rng.integers(0, clusters, size=n)
    return (centers[which] + rng.normal(size=(n, d)) * spread).astype(np.float32)


def flat_fixture(R: Oracle, name, dims, text, n_db, seed):
    rng = np.random.default_rng(seed)
    s = R.spec(dims, text)
    train = blobs(rng, 3000, dims)
    iters = 6 if s.total_entries > 1000 else 12
    cb = R.train_codebook(s, train, iters=iters, seed=seed)
    db = blobs(rng, n_db, dims)
    codes = R.encode(s, cb, db)
    packed = R.pack_list(s, codes)
    queries = blobs(rng, 6, dims)
    r, t = 100, 400
    ids, dists, counts, qlut, params = R.flat_search(s, cb, packed, n_db, queries, r=r, t=t, family=0, debug=True)
    # the natural vector family must agree with the normative scalar scan
    ids_v, dists_v, counts_v = R.flat_search(s, cb, packed, n_db, queries, r=r, t=t, family=1)
    assert np.array_equal(ids, ids_v) and np.array_equal(dists, dists_v) and np.array_equal(counts, counts_v)
    ids_rr, dists_rr, counts_rr = R.flat_search(s, cb, packed, n_db, queries, r=r, t=t, family=0x100)  # rerank=true
    luts = np.stack([R.compute_tables(s, cb, q) for q in queries])
    prefix = np.stack([R.prefix_float(s, packed, n_db, lut, t) for lut in luts])
    sums = np.stack([R.adc_sums(s, packed, n_db, qlut[i], 0, n_db) for i in range(len(queries))])
    np.savez_compressed(
        GOLD / f"flat_{name}.npz", spec=text, dims=dims, codebook=cb, codes=codes, packed=packed, count=n_db,
        queries=queries, r=r, t=t, ids=ids, dists=dists, counts=counts, qlut=qlut, params=params, luts=luts,
        prefix=prefix, sums=sums, vector_family=R.auto_family(s), ids_rr=ids_rr, dists_rr=dists_rr)
    if name in ("pq16x4", "irr655", "pq16x4_short"):  # container fixtures written by the reference's io.hpp
        R.save_flat(s, cb, packed, n_db, GOLD / f"flat_{name}.qflt")
    print(f"flat_{name}: {text} d={dims} n={n_db} family={R.auto_family(s)}")


def scan_fixture(R: Oracle, seed=77):
    """Randomised QuantizedScanFn cases in the style of selftest.hpp:40-127 (outputs from the reference)."""
    rng = np.random.default_rng(seed)
    cases = {}
    fams = [("{4,4}", [2, 4, 6, 8, 10, 16, 32]), ("{6,6,4}", [3, 6, 12, 24]), ("{6,5,5}", [3, 6, 12, 24]),
            ("{5,5,5}", [3, 6, 12, 24]), ("{8,8}", [2, 4, 8, 16]), ("{8}", [1, 2, 4, 8, 16])]
    idx = 0
    for pat, ms in fams:
        for trial in range(6):
            m = int(ms[rng.integers(len(ms))])
            text = f"{m}x{pat}"
            s = R.spec(16 * m, text)
            qmax = s.q_max
            sat = rng.integers(4) == 0
            if sat:
                qlut = (qmax - rng.integers(0, qmax // 4 + 1, size=s.total_entries)).astype(s.qdtype)
            else:
                qlut = rng.integers(0, qmax + 1, size=s.total_entries).astype(s.qdtype)
            n = int(1 + rng.integers(s.block_len * 3))
            codes = np.stack([rng.integers(0, 1 << b, size=n) for b in s.bits_list()], 1).astype(np.uint8)
            packed = R.pack_list(s, codes)
            cap = int(1 + rng.integers(24))
            init = int(rng.integers(qmax + 2)) if rng.integers(4) == 0 else 0
            base = int(rng.integers(100000))
            ids = rng.integers(0, 1000000, size=n).astype(np.uint32) if rng.integers(2) else None
            pre = [(int(rng.integers(qmax + 1)), 2000000 + i) for i in range(int(rng.integers(4)))]
            od, oi = R.scan_quantized(s, packed, n, qlut, ids=ids, base_id=base, acc_init=init, cap=cap, heap_in=pre,
                                      family=0)
            od2, oi2 = R.scan_quantized(s, packed, n, qlut, ids=ids, base_id=base, acc_init=init, cap=cap,
                                        heap_in=pre, family=1)
            assert np.array_equal(od, od2) and np.array_equal(oi, oi2)
            p = f"c{idx}_"
            cases[p + "spec"] = text
            cases[p + "dims"] = 16 * m
            cases[p + "qlut"] = qlut
            cases[p + "packed"] = packed
            cases[p + "n"] = n
            cases[p + "cap"] = cap
            cases[p + "init"] = init
            cases[p + "base"] = base
            cases[p + "ids"] = ids if ids is not None else np.zeros(0, np.uint32)
            cases[p + "pre"] = np.array(pre, dtype=np.int64).reshape(-1, 2)
            cases[p + "out_d"] = od
            cases[p + "out_i"] = oi
            idx += 1
    cases["n_cases"] = idx
    np.savez_compressed(GOLD / "scan_cases.npz", **cases)
    print(f"scan_cases: {idx} cases")


def ivf_fixture(R: Oracle, name, dims, text, k_cells, n_db, probes, seed):
    rng = np.random.default_rng(seed)
    s = R.spec(dims, text)
    db = blobs(rng, n_db, dims, clusters=40)
    coarse, assign = R.kmeans(db, k_cells, iters=8, seed=seed)
    resid = db - coarse[assign]
    cb = R.train_codebook(s, resid, iters=6, seed=seed + 1)
    codes = R.encode(s, cb, resid)
    # force two empty cells to exercise the empty-list paths
    packed_parts, ids_parts, counts, boff, ioff = [], [], [], [], []
    b = i = 0
    for c in range(k_cells):
        members = np.nonzero(assign == c)[0].astype(np.uint32)
        pk = R.pack_list(s, codes[members]) if len(members) else np.zeros(0, np.uint8)
        boff.append(b)
        ioff.append(i)
        counts.append(len(members))
        packed_parts.append(pk)
        ids_parts.append(members)
        b += len(pk)
        i += len(members)
    packed = np.concatenate(packed_parts)
    ids = np.concatenate(ids_parts)
    queries = blobs(rng, 8, dims, clusters=40)
    out = {}
    for pr in (1, probes, k_cells):
        oi, od, oc = R.ivf_search(s, cb, coarse, packed, boff, ioff, counts, ids, queries, probes=pr, r=50, t=200,
                                  family=0)
        oi2, od2, oc2 = R.ivf_search(s, cb, coarse, packed, boff, ioff, counts, ids, queries, probes=pr, r=50, t=200,
                                     family=1)
        assert np.array_equal(oi, oi2) and np.array_equal(od, od2) and np.array_equal(oc, oc2)
        out[f"ids_p{pr}"], out[f"dists_p{pr}"], out[f"counts_p{pr}"] = oi, od, oc
    oi, od, oc = R.ivf_search(s, cb, coarse, packed, boff, ioff, counts, ids, queries, probes=probes, r=50, t=200,
                              family=0x100)  # rerank=true
    out["ids_rr"], out["dists_rr"] = oi, od
    order = np.stack([R.probe_order(dims, coarse, q, probes) for q in queries])
    np.savez_compressed(
        GOLD / f"ivf_{name}.npz", spec=text, dims=dims, codebook=cb, coarse=coarse, packed=packed,
        list_byte_off=np.array(boff, np.uint64), list_id_off=np.array(ioff, np.uint64),
        list_count=np.array(counts, np.uint64), list_ids=ids, queries=queries, r=50, t=200,
        probe_list=np.array([1, probes, k_cells]), order=order, **out)
    R.save_ivf(s, cb, coarse, packed, boff, ioff, counts, ids, GOLD / f"ivf_{name}.qivf")
    print(f"ivf_{name}: {text} K={k_cells} n={n_db} min/max list {min(counts)}/{max(counts)}")


def ivf_build_fixture(R: Oracle, name, dims, text, k_cells, n_db, seed):
    """IvfIndex::build itself (index.hpp:179-230): its trained centroids/codebook plus the lists it produced, so
    that the assignment + residual-encode + pack stage can be replayed from the same inputs."""
    rng = np.random.default_rng(seed)
    db = blobs(rng, n_db, dims, clusters=30)
    built = R.ivf_build(db, text, k_cells, iters=6, seed=seed)
    np.savez_compressed(GOLD / f"ivfbuild_{name}.npz", spec=text, dims=dims, vectors=db, **built)
    print(f"ivfbuild_{name}: {text} K={k_cells} n={n_db} min/max list "
          f"{int(built['list_count'].min())}/{int(built['list_count'].max())}")


def main():
    build()
    R = Oracle("reference")
    GOLD.mkdir(parents=True, exist_ok=True)
    for i, (name, dims, text, n_db) in enumerate(FAMILIES):
        flat_fixture(R, name, dims, text, n_db, seed=100 + i)
    # short list: fewer codes than R and than t (T/test_index.cpp:24-55 edge cases)
    flat_fixture(R, "pq16x4_short", 64, "16x{4,4}", 37, seed=200)
    flat_fixture(R, "irr655_short", 48, "12x{6,5,5}", 150, seed=201)
    scan_fixture(R)
    ivf_fixture(R, "irr655", 48, "12x{6,5,5}", 24, 4000, 6, seed=300)
    ivf_fixture(R, "pq16x4", 32, "8x{4,4}", 12, 2500, 4, seed=301)
    ivf_build_fixture(R, "pq8x4", 32, "8x{4,4}", 20, 3000, seed=400)
    ivf_build_fixture(R, "irr655", 48, "12x{6,5,5}", 40, 3500, seed=401)


if __name__ == "__main__":
    main()
