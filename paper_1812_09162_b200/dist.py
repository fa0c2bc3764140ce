"""Multi-GPU flat search: database shards + one exchange step.

One process per GPU (torch.distributed, NCCL over NVLink/NVSwitch for the plumbing).  The code
array is partitioned into contiguous ranges on packed-block boundaries; shard s scans with
``base_id = start_s`` exactly like the reference's chunked-scan contract
(T/test_kernels.cpp:107-133).  The quantization map is calibrated on the first t codes of the
WHOLE list (index.hpp:124-129), so every shard is opened with that global head and derives
bit-identical tables with no communication.  Per query each rank produces its local top-R as
64-bit keys (distance << 32 | id); ONE all_gather of nq*R keys per rank (8 MB at nq=10^4, R=100:
latency-bound on NVSwitch) is followed by a merge kernel.  The final list is the R smallest keys
of the union, which is exact because the reference heap is order-independent (heap.hpp:12-14).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from ._lib import QadcSpec
from .index import FlatIndex, SearchParams, merge_topk_device, packed_bytes


@dataclass
class ShardRange:
    start: int  # first code of the shard (multiple of block_len)
    count: int


def shard_ranges(total: int, world: int, block_len: int) -> list[ShardRange]:
    """Even split of ``total`` codes over ``world`` ranks with every boundary on a packed-block boundary."""
    blocks = (total + block_len - 1) // block_len
    out = []
    for r in range(world):
        b0 = blocks * r // world
        b1 = blocks * (r + 1) // world
        start = min(b0 * block_len, total)
        end = min(b1 * block_len, total)
        out.append(ShardRange(start, end - start))
    return out


def slice_packed(spec: QadcSpec, packed: np.ndarray, rng: ShardRange) -> np.ndarray:
    """Byte range of a block-aligned shard inside a PackedList (blocks are contiguous, layout.hpp:135-144)."""
    bb = spec.groups * spec.block_len * (spec.word_width // 8)
    b0 = rng.start // spec.block_len
    return packed[b0 * bb: b0 * bb + packed_bytes(spec, rng.count)]


T_MAX = 16384  # QADC_MAX_T: the longest calibration prefix the ABI accepts, so a default head never truncates one


def global_head(spec: QadcSpec, packed: np.ndarray, total: int, t_max: int = T_MAX):
    """PackedList prefix holding the first min(total, t_max) codes (rounded up to whole blocks).  A shard opened
    with this head serves every t <= t_max exactly; a larger t is refused (QADC_ERR_CONFIG), never clamped."""
    n = min(total, t_max)
    return packed[: packed_bytes(spec, n)], n


class ShardedIndex:
    """One index shard per rank (flat or IVF) plus the gather + merge exchange (NCCL all_gather of the per-rank
    key lists, then the CUDA merge kernel qadc_merge_topk_device)."""

    def __init__(self, index, device, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.device = device
        self.spec = index.spec
        self.index = index

    def search_device(self, d_queries, params: SearchParams, d_ids, d_dists, d_counts, stream=None):
        """All tensors are torch CUDA tensors on this rank's device; results are replicated on every rank.

        ``stream`` (an int cudaStream_t; default: torch's current stream) carries ALL three steps -- the shard
        search, the all_gather and the merge kernel: the collective is issued under ``torch.cuda.stream`` of the
        same stream, so the exchange is ordered behind the search and in front of the merge by stream order
        alone, whatever the caller's current stream is."""
        import torch
        nq, r = int(d_queries.shape[0]), int(params.r)
        dev = d_queries.device
        ext = torch.cuda.current_stream(dev) if not stream else torch.cuda.ExternalStream(int(stream), device=dev)
        with torch.cuda.stream(ext):
            keys = torch.empty((nq, r), dtype=torch.int64, device=dev)
            qmap = torch.empty((nq, 2), dtype=torch.float32, device=dev)
            self.index.search_device(d_queries, params, None, None, None, d_keys=keys, d_map=qmap,
                                     stream=ext.cuda_stream)
            if self.world == 1:
                gathered = keys.unsqueeze(0)
            else:
                gathered = torch.empty((self.world, nq, r), dtype=torch.int64, device=dev)
                # flat [world * nq, r] view: the layout NCCL and gloo both accept for the tensor form
                self.dist.all_gather_into_tensor(gathered.view(self.world * nq, r), keys, group=self.group)
            merge_topk_device(gathered, self.world, nq, r, qmap, d_ids, d_dists, d_counts, self.device,
                              fma_unquantize=params.fma_unquantize, stream=ext.cuda_stream)
            for t in (keys, qmap, gathered):  # allocated under `ext`, consumed there: nothing to record elsewhere
                t.record_stream(ext)

    def close(self):
        self.index.close()


class ShardedFlatIndex(ShardedIndex):
    """A FlatIndex shard per rank: contiguous block-aligned code range, base_id, replicated global head."""

    def __init__(self, spec: QadcSpec, codebook, shard_packed, shard: ShardRange, head_packed, head_count, device,
                 group=None, global_count: int = 0):
        """``global_count`` = codes of the WHOLE database (0 = unknown: then the head is taken as truncated and a
        search with t > head_count is refused rather than calibrated on fewer codes than the reference uses)."""
        super().__init__(FlatIndex(spec, codebook, shard_packed, shard.count, base_id=shard.start,
                                   calib_packed=head_packed, calib_count=head_count, global_count=global_count,
                                   device=device), device, group)

    @classmethod
    def from_global(cls, spec: QadcSpec, codebook, packed, total: int, rank: int, world: int, device, group=None,
                    t_max: int = T_MAX):
        """Shard `rank` of `world` of one whole PackedList (each rank passes the same `packed`)."""
        rg = shard_ranges(total, world, spec.block_len)[rank]
        head, head_n = global_head(spec, packed, total, t_max)
        return cls(spec, codebook, slice_packed(spec, packed, rg), rg, head, head_n, device, group, global_count=total)


def shard_ivf_lists(spec: QadcSpec, packed, list_byte_off, list_id_off, list_count, ids, rank: int, world: int,
                    t_max: int = T_MAX):
    """IVF sharding: EVERY list is split evenly (on packed-block boundaries) across the ranks --
    ids are explicit, so any split is legal (scan_scalar.hpp:60) -- and the first min(count, t_max) codes of every
    unsharded list are replicated as calibration heads, so probe order, tables, d_min_global, d_max, delta and the
    biases come out identical on every rank.  Returns the keyword arguments for :class:`IvfIndex`."""
    packed = np.ascontiguousarray(packed, dtype=np.uint8)
    ids = np.ascontiguousarray(ids, dtype=np.uint32)
    k = len(list_count)
    s_packed, s_ids, s_boff, s_ioff, s_cnt = [], [], [], [], []
    c_packed, c_boff, c_cnt = [], [], []
    b = i = cb = 0
    for c in range(k):
        n = int(list_count[c])
        lp = packed[int(list_byte_off[c]): int(list_byte_off[c]) + packed_bytes(spec, n)]
        rg = shard_ranges(n, world, spec.block_len)[rank]
        sp = slice_packed(spec, lp, rg)
        s_boff.append(b); s_ioff.append(i); s_cnt.append(rg.count)
        s_packed.append(sp)
        s_ids.append(ids[int(list_id_off[c]) + rg.start: int(list_id_off[c]) + rg.start + rg.count])
        b += sp.size; i += rg.count
        hn = min(n, t_max)
        hp = lp[: packed_bytes(spec, hn)]
        c_boff.append(cb); c_cnt.append(hn); c_packed.append(hp)
        cb += hp.size
    cat = lambda xs, dt: np.concatenate(xs).astype(dt) if xs and sum(x.size for x in xs) else np.zeros(0, dt)  # noqa: E731
    return dict(packed=cat(s_packed, np.uint8), list_byte_off=np.array(s_boff, np.uint64),
                list_id_off=np.array(s_ioff, np.uint64), list_count=np.array(s_cnt, np.uint64),
                ids=cat(s_ids, np.uint32), calib_packed=cat(c_packed, np.uint8),
                calib_byte_off=np.array(c_boff, np.uint64), calib_count=np.array(c_cnt, np.uint64),
                global_list_count=np.ascontiguousarray(list_count, dtype=np.uint64))


def merge_keys_numpy(gathered: np.ndarray, r: int) -> np.ndarray:
    """Reference merge for tests: [world, nq, r] uint64 keys (padding = 2^64-1) -> [nq, r] smallest keys."""
    world, nq, _ = gathered.shape
    allk = np.transpose(gathered, (1, 0, 2)).reshape(nq, -1)
    return np.sort(allk, axis=1)[:, :r]
