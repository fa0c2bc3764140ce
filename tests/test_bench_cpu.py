"""Host logic of bench.py that needs no GPU: the chunk-seeded database generator must give every rank the same ONE
database (strong scaling: any code range can be produced without the other ranks' streams), and both arms must
describe a workload with the same `config` object."""
import importlib.util
import sys
from pathlib import Path

import numpy as np
import pytest

import paper_1812_09162_b200 as qb
from paper_1812_09162_b200.dist import shard_ranges

ROOT = Path(__file__).resolve().parent.parent


@pytest.fixture(scope="module")
def bench():
    spec = importlib.util.spec_from_file_location("bench_under_test", ROOT / "bench.py")
    mod = importlib.util.module_from_spec(spec)
    sys.modules["bench_under_test"] = mod
    spec.loader.exec_module(mod)
    return mod


@pytest.mark.parametrize("text,dims,n", [("16x{4,4}", 128, 10_000), ("12x{6,5,5}", 96, 7_777), ("8x{8}", 64, 4_096)])
def test_chunked_generator_is_shard_invariant(bench, monkeypatch, text, dims, n):
    monkeypatch.setattr(bench, "CHUNK", 2048)
    monkeypatch.setattr(bench, "HEAD_MAX", 512)
    s = qb.allocate_dims(dims, text)
    wl = dict(kind="flat", spec=text, dims=dims, n=n, nq=4, data="random")
    monkeypatch.setattr("paper_1812_09162_b200.synth.train_codebook",
                        lambda spec, x, iters=1, seed=0: np.zeros(spec.cb_floats, np.float32))
    whole = bench.make_flat(qb, s, wl, have_gpu=False)
    assert whole["packed"].size == qb.packed_bytes(s, n) and whole["full"] is whole["packed"]
    codes = qb.unpack_list(s, whole["packed"], n)
    for world in (2, 3, 8):
        parts = []
        for rg in shard_ranges(n, world, s.block_len):
            d = bench.make_flat(qb, s, wl, have_gpu=False, start=rg.start, count=rg.count)
            assert d["packed"].size == qb.packed_bytes(s, rg.count)
            parts.append(qb.unpack_list(s, d["packed"], rg.count))
            assert np.array_equal(d["head"], whole["head"]) and d["head_n"] == min(512, n)
        assert np.array_equal(np.concatenate(parts), codes), world
    d = bench.make_flat(qb, s, wl, have_gpu=False, start=2048, count=1024, whole=True)
    assert np.array_equal(d["full"], whole["packed"])
    assert np.array_equal(qb.unpack_list(s, d["packed"], 1024), codes[2048:3072])


def test_both_arms_describe_the_same_config(bench):
    for name, wl in bench.WORKLOADS.items():
        for world in (1, 2, 8):
            a = bench.describe(name, dict(wl), world, "strong")
            b = bench.describe(name, dict(wl), world, "strong")
            assert a == b and a["database_codes"] == wl["n"] and a["codes_per_gpu"] == -(-wl["n"] // world)
    assert bench.WORKLOADS["c4"]["n"] == 200_000_000 and bench.WORKLOADS["c5"]["n"] == 500_000_000
