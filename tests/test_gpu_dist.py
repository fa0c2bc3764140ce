"""The multi-rank PRODUCT path with world_size 2 on one GPU: two processes (gloo backend, CUDA tensors) each build
their shard with ShardedFlatIndex.from_global / shard_ivf_lists + ShardedIndex and call search_device -- the shard
search, the all_gather of the per-rank key lists and the CUDA merge kernel, all on ONE explicit non-default stream.
Every rank must end with the unsharded oracle result (ids, distance bits, counts): the reference's chunked-scan
contract (T/test_kernels.cpp:107-133) plus the replicated calibration head (index.hpp:124-129).

The ranks never wait on each other's KERNELS (the collective is a host-side gloo exchange of finished key lists), so
sharing one GPU is safe here; under NCCL on a multi-GPU box the same class runs with one GPU per rank."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_1812_09162_b200 as qb
from paper_1812_09162_b200.synth import random_codes

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _ivf_lists(rng, s, k_cells, n):
    assign = rng.integers(0, k_cells, size=n)
    codes = random_codes(s, n, seed=9)
    packed, ids, boff, ioff, counts = [], [], [], [], []
    b = i = 0
    for c in range(k_cells):
        members = np.nonzero(assign == c)[0].astype(np.uint32)
        pk = qb.pack_list(s, codes[members])
        boff.append(b); ioff.append(i); counts.append(len(members)); packed.append(pk); ids.append(members)
        b += pk.size; i += len(members)
    return (np.concatenate(packed), np.array(boff, np.uint64), np.array(ioff, np.uint64), np.array(counts, np.uint64),
            np.concatenate(ids))


def _worker(rank, world, port_no, kind, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_no)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.pyoracle import Oracle
        from paper_1812_09162_b200.dist import ShardedFlatIndex, ShardedIndex, shard_ivf_lists
        port = Oracle("port")
        torch.cuda.set_device(0)
        dev = torch.device("cuda", 0)
        rng = np.random.default_rng(4)  # same seed on every rank: identical database, queries and codebook
        r, t = 100, 400
        if kind == "flat":
            dims, text, n = 128, "16x{4,4}", 300_000
            s, so = qb.allocate_dims(dims, text), port.spec(dims, text)
            cb = (rng.standard_normal(s.cb_floats) * 2).astype(np.float32)
            packed = qb.pack_list(s, random_codes(s, n, seed=8))
            queries = (rng.standard_normal((48, dims)) * 2).astype(np.float32)
            want = port.flat_search(so, cb, packed, n, queries, r=r, t=t, threads=4)
            sharded = ShardedFlatIndex.from_global(s, cb, packed, n, rank, world, 0, t_max=1024)
            params = qb.SearchParams(r=r, t=t)
            bad = qb.SearchParams(r=r, t=1025)  # beyond the truncated head: refused, never clamped
        else:
            dims, text, k_cells, n = 64, "12x{6,5,5}", 48, 120_000
            s, so = qb.allocate_dims(dims, text), port.spec(dims, text)
            cb = (rng.standard_normal(s.cb_floats) * 1.5).astype(np.float32)
            coarse = (rng.standard_normal((k_cells, dims)) * 3).astype(np.float32)
            packed, boff, ioff, counts, ids = _ivf_lists(rng, s, k_cells, n)
            queries = (rng.standard_normal((40, dims)) * 3).astype(np.float32)
            want = port.ivf_search(so, cb, coarse, packed, boff, ioff, counts, ids, queries, probes=9, r=r, t=t, threads=4)
            kw = shard_ivf_lists(s, packed, boff, ioff, counts, ids, rank, world, t_max=512)
            sharded = ShardedIndex(qb.IvfIndex(s, cb, coarse, kw["packed"], kw["list_byte_off"], kw["list_id_off"],
                                               kw["list_count"], kw["ids"], device=0, calib_packed=kw["calib_packed"],
                                               calib_byte_off=kw["calib_byte_off"], calib_count=kw["calib_count"],
                                               global_list_count=kw["global_list_count"]), 0)
            params = qb.SearchParams(probes=9, r=r, t=t)
            bad = qb.SearchParams(probes=9, r=r, t=513)
        nq = len(queries)
        side = torch.cuda.Stream(device=dev)  # NOT torch's current stream: search, gather and merge must all follow it
        d_q = torch.from_numpy(queries).to(dev)
        d_ids = torch.empty((nq, r), dtype=torch.int32, device=dev)
        d_dists = torch.empty((nq, r), dtype=torch.float32, device=dev)
        d_counts = torch.empty((nq,), dtype=torch.int32, device=dev)
        torch.cuda.synchronize()
        refused = False
        try:
            sharded.search_device(d_q, bad, d_ids, d_dists, d_counts, stream=side.cuda_stream)
        except qb.QadcError as e:
            refused = e.kind == "config"
        for _ in range(2):  # twice: workspaces are reused across calls
            sharded.search_device(d_q, params, d_ids, d_dists, d_counts, stream=side.cuda_stream)
        side.synchronize()
        ids_g = d_ids.cpu().numpy().view(np.uint32)
        dists_g = d_dists.cpu().numpy()
        counts_g = d_counts.cpu().numpy().astype(np.uint32)
        ok = refused and bool(np.array_equal(counts_g, want[2]))
        for qi in range(nq):
            c = int(want[2][qi])
            ok &= bool(np.array_equal(ids_g[qi, :c], want[0][qi, :c]))
            ok &= dists_g[qi, :c].tobytes() == want[1][qi, :c].tobytes()
        sharded.close()
        out_q.put((rank, ok, refused))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind", ["flat", "ivf"])
def test_two_rank_sharded_index_on_one_gpu(kind):
    from oracle.pyoracle import build
    qb.build()
    build()
    world = 2
    ctx = mp.get_context("spawn")
    out_q = ctx.Queue()
    port_no = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port_no, kind, out_q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
        assert p.exitcode == 0
    results = sorted(out_q.get(timeout=10) for _ in range(world))
    assert results == [(r, True, True) for r in range(world)]
