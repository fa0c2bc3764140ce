"""Multi-rank host logic on CPU (gloo, world_size 2 and 3): shard partitioning on block boundaries, base ids,
replication of the global calibration head, the all_gather exchange and the merge.  The per-shard searches
are done by the CPU oracle here (the CUDA path is covered by the -m gpu tests); what is under test is that
'shard + global head + gather + merge' reproduces the unsharded search bit-for-bit, as the reference's
chunked-scan contract promises (T/test_kernels.cpp:107-133)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_1812_09162_b200 as qb
from paper_1812_09162_b200.dist import global_head, merge_keys_numpy, shard_ranges, slice_packed
from paper_1812_09162_b200.synth import random_codes


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _oracle_shard_keys(port, so, s, cb, shard_packed, rng_, head, head_n, queries, r, t):
    """What one rank computes: tables calibrated on the GLOBAL head, scan of its own shard with base_id."""
    keys = np.full((len(queries), r), np.iinfo(np.uint64).max, dtype=np.uint64)
    maps = np.zeros((len(queries), 2), np.float32)
    for qi, q in enumerate(queries):
        lut = port.compute_tables(so, cb, q)
        pre = port.prefix_float(so, head, head_n, lut, t)
        dmin, dmax = port.calibrate(so, lut, pre, min(r, len(pre)))
        qlut, _, delta, own = port.quantize(so, lut, dmin, dmax, so.word_width)
        d, i = port.scan_quantized(so, shard_packed, rng_.count, qlut, base_id=rng_.start, cap=r)
        keys[qi, :len(d)] = (d.astype(np.uint64) << np.uint64(32)) | i.astype(np.uint64)
        maps[qi] = (delta, own)
    return keys, maps


def _worker(rank, world, port_no, dims, text, n, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_no)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.pyoracle import Oracle
        port = Oracle("port")
        s, so = qb.allocate_dims(dims, text), port.spec(dims, text)
        rng = np.random.default_rng(1)
        cb = (rng.standard_normal(s.cb_floats) * 2).astype(np.float32)
        packed = qb.pack_list(s, random_codes(s, n, seed=2))
        queries = (rng.standard_normal((12, dims)) * 2).astype(np.float32)
        r, t = 50, 200
        ranges = shard_ranges(n, world, s.block_len)
        assert sum(x.count for x in ranges) == n and all(x.start % s.block_len == 0 for x in ranges)
        mine = ranges[rank]
        head, head_n = global_head(s, packed, n, t_max=512)
        keys, maps = _oracle_shard_keys(port, so, s, cb, slice_packed(s, packed, mine), mine, head, head_n, queries, r, t)
        gathered = [torch.empty_like(torch.from_numpy(keys.view(np.int64))) for _ in range(world)]
        dist.all_gather(gathered, torch.from_numpy(keys.view(np.int64)))
        allk = np.stack([g.numpy().view(np.uint64) for g in gathered])
        merged = merge_keys_numpy(allk, r)
        # every rank must hold the same map (replicated calibration, no communication)
        gm = [torch.empty(len(queries), 2) for _ in range(world)]
        dist.all_gather(gm, torch.from_numpy(maps))
        assert all(torch.equal(gm[0], x) for x in gm)
        want = port.flat_search(so, cb, packed, n, queries, r=r, t=t)
        valid = merged != np.iinfo(np.uint64).max
        ids = (merged & np.uint64(0xFFFFFFFF)).astype(np.uint32)
        dq = (merged >> np.uint64(32)).astype(np.float32)
        dists = (dq * maps[:, :1] + maps[:, 1:2]).astype(np.float32)
        ok = bool(np.array_equal(valid.sum(1), want[2]))
        for qi in range(len(queries)):
            c = int(want[2][qi])
            ok &= bool(np.array_equal(ids[qi, :c], want[0][qi, :c]))
            ok &= dists[qi, :c].tobytes() == want[1][qi, :c].tobytes()
        out_q.put((rank, ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,dims,text,n", [(2, 64, "16x{4,4}", 5000), (3, 48, "12x{6,5,5}", 3333), (2, 32, "8x{8}", 130)])
def test_sharded_search_equals_unsharded(world, dims, text, n):
    from oracle.pyoracle import build
    build()
    ctx = mp.get_context("spawn")
    out_q = ctx.Queue()
    port_no = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port_no, dims, text, n, out_q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=180)
        assert p.exitcode == 0
    results = sorted(out_q.get(timeout=10) for _ in range(world))
    assert results == [(r, True) for r in range(world)]


def test_shard_ranges_properties():
    for total in (0, 1, 15, 16, 17, 1000, 12345):
        for world in (1, 2, 3, 8):
            for bl in (16, 32, 64):
                rs = shard_ranges(total, world, bl)
                assert len(rs) == world and sum(x.count for x in rs) == total
                pos = 0
                for x in rs:
                    assert x.start == pos or x.count == 0
                    assert x.start % bl == 0 or x.count == 0
                    pos = x.start + x.count
