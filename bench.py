#!/usr/bin/env python
"""bench.py -- throughput of the Quicker ADC scan path on B200 (metric of BASELINE.json).

    python bench.py --gpus N --steps K --warmup W [--workload c4] [--scaling strong|weak] [--impl reference]

A "step" is one pass of the whole hot path (distance tables -> calibration -> quantization -> scan ->
top-R [-> multi-GPU merge]) over one batch of synthetic queries against the resident database.
``value``   = (query, code) pairs evaluated per second, whole job, inputs already in HBM;
``e2e``     = the same metric through the reference-facing C-ABI call with HOST buffers
              (qadc_search_batch: H2D of the queries and D2H of ids/dists/counts inside the timed region);
``roofline``= algorithmic code bytes (8 B per pair) / CUDA-event time of the scan kernels, against the
              measured HBM copy bandwidth of MEASURED_PEAKS.json;
``cpu_baseline`` = the reference's own CPU search (oracle/_ref when it was built, else the oracle port)
              timed on this box's host cores on a bounded query sample of the same workload;
``parity``  = after (outside) the timed region, a seeded sample of the just-benchmarked queries is searched by the
              reference on the CPU and compared with the GPU result (ids, distance bits, counts); a mismatch
              makes the exit code non-zero.

Workloads (BASELINE.json configs; seeded synthetic inputs with the named shapes stand in for the
SIFT/Deep-like data, see paper_1812_09162_b200/synth.py).  N is the size of the WHOLE database:
  c1  16x{4,4}    d=128  N=1e6   Q=1e3     c3  8x{8,8}   d=128  N=1e7  Q=1e4
  c2  12x{6,5,5}  d=96   N=1e7   Q=1e4     c4  16x{4,4}  d=128  N=2e8  Q=1e4 (uniform random codes)
  c5  IVF K=16384, 12x{6,5,5} residual codes, d=128, N=5e8, nprobe=64, Q=1e4
  c5g the share of c5 one GPU of the 8-GPU box holds (N = 5e8 / 8 = 6.25e7): the single-GPU form of config 5
Default c4: the largest single-GPU configuration and the one BASELINE's 1/2/4/8-GPU clause is written on.
With --gpus N > 1 (torchrun, one rank per GPU) the ONE database of the workload is split evenly over the N ranks on
packed-block boundaries (``"scaling": "strong"``: 2e8 / N codes per GPU for c4; IVF: every list is split N ways, list
heads are replicated), queries are replicated and the per-query top-R lists are merged after one NCCL all_gather.
``--scaling weak`` keeps the workload's N per GPU instead (N times the database).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

WORKLOADS = {
    "c1": dict(kind="flat", spec="16x{4,4}", dims=128, n=1_000_000, nq=1_000, data="encoded"),
    "c2": dict(kind="flat", spec="12x{6,5,5}", dims=96, n=10_000_000, nq=10_000, data="encoded"),
    "c3": dict(kind="flat", spec="8x{8,8}", dims=128, n=10_000_000, nq=10_000, data="encoded"),
    "c4": dict(kind="flat", spec="16x{4,4}", dims=128, n=200_000_000, nq=10_000, data="random"),
    "c5": dict(kind="ivf", spec="12x{6,5,5}", dims=128, n=500_000_000, nq=10_000, data="random", k_cells=16384,
               probes=64),
    # the paper's 128-bit configurations at the C2/C3 size, uniform random codes
    "w44": dict(kind="flat", spec="32x{4,4}", dims=128, n=10_000_000, nq=10_000, data="random"),
    "w655": dict(kind="flat", spec="24x{6,5,5}", dims=96, n=10_000_000, nq=10_000, data="random"),
    "w88": dict(kind="flat", spec="16x{8,8}", dims=128, n=10_000_000, nq=10_000, data="random"),
    "c5g": dict(kind="ivf", spec="12x{6,5,5}", dims=128, n=62_500_000, nq=10_000, data="random", k_cells=16384,
                probes=64),
}
R, T = int(os.environ.get("QADC_BENCH_R", 100)), int(os.environ.get("QADC_BENCH_T", 400))  # BASELINE: R=100, t=400 (env: experiments only)
CHUNK = 1 << 20   # the database is generated in chunks of this many codes, each from its own seed, so that any
                  # rank can produce any code range of the ONE database without the others' random streams
HEAD_MAX = 16384  # replicated calibration head (QADC_MAX_T): serves every t the ABI accepts


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ----------------------------------------------------------------------------- data --

def make_flat(qb, spec, wl, have_gpu, start=0, count=None, whole=False):
    """Codes [start, start + count) of the workload's ONE database as a PackedList (start on a block boundary),
    plus the global calibration head (the database's first codes).  whole=True also returns the complete database
    (rank 0 keeps it for the CPU parity check when the database is sharded)."""
    from paper_1812_09162_b200 import synth
    dims, n = wl["dims"], wl["n"]
    count = n - start if count is None else count
    centres = synth.mixture_centres(dims, seed=1)
    train = synth.gaussian_mixture(100_000, dims, seed=4, centres=centres)
    t0 = time.time()
    cb = synth.train_codebook(spec, train, iters=8, seed=5)
    log(f"[bench] codebook ({spec.cb_floats} floats) trained in {time.time() - t0:.1f}s")
    code_bytes = spec.groups * (spec.word_width // 8)
    assert CHUNK % spec.block_len == 0 and start % spec.block_len == 0

    def encode(vecs):
        if have_gpu:
            return qb.encode(spec, cb, vecs)
        from oracle.pyoracle import Oracle  # reference arm on a box without a GPU: CPU encoder
        o = Oracle("port")
        return o.encode(o.spec(dims, wl["spec"]), cb, vecs)

    def chunk_packed(c):
        """PackedList bytes of chunk c = codes [c * CHUNK, min((c + 1) * CHUNK, n)) -- whole blocks except at the end."""
        cn = min(CHUNK, n - c * CHUNK)
        if wl["data"] == "random":
            return synth.random_packed(spec, cn, seed=6 + 1000 * c)
        return qb.pack_list(spec, encode(synth.gaussian_mixture(cn, dims, seed=2 + 1000 * c, centres=centres)))

    def range_packed(lo, hi):
        parts = []
        for c in range(lo // CHUNK, (max(hi, lo + 1) - 1) // CHUNK + 1):
            pk = chunk_packed(c)
            c0 = c * CHUNK
            a_, b_ = max(lo, c0) - c0, min(hi, c0 + CHUNK) - c0  # block-aligned except possibly b_ == chunk end
            parts.append(pk[a_ * code_bytes: qb.packed_bytes(spec, b_)] if a_ else pk[: qb.packed_bytes(spec, b_)])
        return np.concatenate(parts) if parts else np.zeros(0, np.uint8)

    t0 = time.time()
    full = range_packed(0, n) if whole or (start == 0 and count == n) else None
    if full is not None and start == 0 and count == n:
        packed = full
    elif full is not None:
        packed = full[start * code_bytes: start * code_bytes + qb.packed_bytes(spec, count)]
    else:
        packed = range_packed(start, start + count)
    head_n = min(HEAD_MAX, n)
    head = (full if full is not None else range_packed(0, min(n, CHUNK)))[: qb.packed_bytes(spec, head_n)]
    log(f"[bench] codes [{start}, {start + count}) of {n} ready in {time.time() - t0:.1f}s")
    queries = synth.gaussian_mixture(wl["nq"], dims, seed=3, centres=centres)
    return dict(cb=cb, packed=packed, head=head, head_n=head_n, queries=queries, full=full)


def make_ivf(qb, spec, wl, have_gpu, bcast=None):
    """Config 5 stand-in (the WHOLE index): coarse centroids from Lloyd iterations on mixture samples, list sizes
    from the assignment histogram of a mixture sample scaled to N, uniform random residual codes, ids = positions."""
    from paper_1812_09162_b200 import synth
    import torch
    dims, n, K = wl["dims"], wl["n"], wl["k_cells"]
    dev = torch.device("cuda", torch.cuda.current_device()) if have_gpu else torch.device("cpu")
    centres = synth.mixture_centres(dims, seed=1)
    t0 = time.time()
    sample = torch.from_numpy(synth.gaussian_mixture(max(4 * K, 300_000), dims, seed=7, centres=centres)).to(dev)
    g = torch.Generator(device="cpu").manual_seed(8)
    coarse = sample[torch.randperm(sample.shape[0], generator=g)[:K].to(dev)].clone()

    def assign(x):
        out = torch.empty(x.shape[0], dtype=torch.long, device=dev)
        for i in range(0, x.shape[0], 16384):
            xb = x[i:i + 16384]
            d = (xb * xb).sum(1, keepdim=True) - 2.0 * xb @ coarse.T + (coarse * coarse).sum(1)[None, :]
            out[i:i + 16384] = d.argmin(1)
        return out

    for _ in range(2 if have_gpu else 1):  # Lloyd steps (input preparation, not the timed path)
        a = assign(sample)
        sums = torch.zeros_like(coarse).index_add_(0, a, sample)
        cnt = torch.bincount(a, minlength=K).clamp(min=1).unsqueeze(1)
        coarse = sums / cnt
    a = assign(sample)
    hist = torch.bincount(a, minlength=K).double().cpu().numpy() + 0.25
    resid = (sample - coarse[a])[:100_000].cpu().numpy()
    coarse = coarse.cpu().numpy().astype(np.float32)
    counts = np.floor(hist / hist.sum() * n).astype(np.uint64)
    counts[: int(n - counts.sum())] += 1
    cb = synth.train_codebook(spec, resid, iters=6, seed=5)
    if bcast is not None:  # Lloyd on the GPU uses float atomics: every rank must hold rank 0's index, bit for bit
        coarse, cb, counts = bcast(coarse), bcast(cb), bcast(counts.astype(np.int64)).astype(np.uint64)
    log(f"[bench] coarse quantizer (K={K}) + residual codebook in {time.time() - t0:.1f}s; "
        f"list sizes min/median/max = {counts.min()}/{int(np.median(counts))}/{counts.max()}")
    t0 = time.time()
    pbytes = np.array([qb.packed_bytes(spec, int(c)) for c in counts], dtype=np.uint64)
    boff = np.concatenate([[0], np.cumsum(pbytes)[:-1]]).astype(np.uint64)
    ioff = np.concatenate([[0], np.cumsum(counts)[:-1]]).astype(np.uint64)
    packed = np.random.default_rng(6).integers(0, 256, size=int(pbytes.sum()), dtype=np.uint8)  # same stream on every rank
    ids = np.arange(n, dtype=np.uint32)
    out = dict(cb=cb, coarse=coarse, packed=packed, boff=boff, ioff=ioff, counts=counts, ids=ids)
    out["queries"] = synth.gaussian_mixture(wl["nq"], dims, seed=3, centres=centres)
    log(f"[bench] {n} residual codes in {K} lists ready in {time.time() - t0:.1f}s")
    return out


# --------------------------------------------------------------------------- clocks --

class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.samples = []
        self.stop = False
        self.gpu = gpu_index
        self.th = threading.Thread(target=self.run, daemon=True)

    def run(self):
        try:
            p = subprocess.Popen(["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                                  "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE, text=True)
        except Exception:
            return
        while not self.stop:
            line = p.stdout.readline()
            if not line:
                break
            self.samples.append((time.time(), [x.strip() for x in line.split(",")]))
        p.kill()

    def __enter__(self):
        self.th.start()
        return self

    def __exit__(self, *a):
        self.stop = True
        self.th.join(timeout=2)

    def summary(self, t0, t1):
        rows = [s for (t, s) in self.samples if t0 - 0.15 <= t <= t1 + 0.15] or [s for (_, s) in self.samples[-3:]]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = sorted(int(r[0]) for r in rows if r[0].isdigit())
        reasons = []
        for i, name in enumerate(["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]):
            if any(len(r) > 3 + i and r[3 + i].lower().startswith("active") for r in rows):
                reasons.append(name)
        return {"sm_mhz": sm[len(sm) // 2] if sm else None,
                "sm_max_mhz": int(rows[0][1]) if rows[0][1].isdigit() else None, "reasons": reasons,
                "samples": len(rows)}


# --------------------------------------------------------------------- cpu baseline --

class CpuReference:
    """The reference's CPU search on the host cores: query-parallel pool on all cores
    (tools/pqscan_cli.cpp:141-166), kernel family chosen by the reference (auto)."""

    def __init__(self, wl, data):
        from oracle.pyoracle import Oracle, build
        build()
        self.kind = "reference" if Oracle.available("reference") else "port"
        self.o = Oracle(self.kind)
        self.wl = wl
        self.s = self.o.spec(wl["dims"], wl["spec"])
        self.cores = os.cpu_count() or 1
        self.queries = data["queries"]
        if wl["kind"] == "ivf":
            self.h = self.o.ivf_open(self.s, data["cb"], data["coarse"], data["packed"], data["boff"], data["ioff"],
                                     data["counts"], data["ids"])
        else:
            self.h = self.o.flat_open(self.s, data["cb"], data["full"] if data.get("full") is not None else data["packed"],
                                      wl["n"])
        self.family = self.o.auto_family(self.s) if self.kind == "reference" else "scalar-quantized (C port)"

    def search(self, queries):
        return self.o.search_h(self.h, queries, probes=self.wl.get("probes", 1), r=R, t=T, family=1, threads=self.cores)

    def run(self, nq):
        t0 = time.perf_counter()
        self.search(self.queries[:nq])
        return time.perf_counter() - t0

    def sized_sample(self, budget_s, cap=None):
        probe = min(len(self.queries), self.cores)
        dt = max(self.run(probe), 1e-4)
        nq = int(min(len(self.queries), max(probe, budget_s / dt * probe)))
        return min(nq, cap) if cap else nq

    def pairs_per_query(self, data, nq_sample):
        """flat: every query scans the whole list; IVF: mean total length of the probed lists."""
        if self.wl["kind"] != "ivf":
            return float(self.wl["n"])
        lens = data["counts"].astype(np.float64)
        qs = data["queries"][:min(64, nq_sample)]
        return float(np.mean([lens[self.o.probe_order(self.wl["dims"], data["coarse"], q, self.wl["probes"])].sum()
                              for q in qs]))

    def parity(self, got_ids, got_dists, got_counts, n_sample):
        """Seeded sample of the benchmarked queries: reference result vs the GPU's (ids, distance bits, counts)."""
        nq = len(self.queries)
        sel = np.sort(np.random.default_rng(12345).choice(nq, size=min(n_sample, nq), replace=False))
        ids, dists, counts = self.search(self.queries[sel])
        bad = 0
        for k, qi in enumerate(sel):
            c = int(counts[k])
            ok = int(got_counts[qi]) == c and np.array_equal(got_ids[qi, :c], ids[k, :c]) and \
                got_dists[qi, :c].tobytes() == dists[k, :c].tobytes()
            bad += 0 if ok else 1
        return {"queries": int(len(sel)), "mismatches": int(bad), "oracle": self.kind,
                "compared": "ids, distance bits and counts of a seeded query sample, after the timed region"}

    def close(self):
        self.o.close_h(self.h)


# ------------------------------------------------------------------------------ main --

def describe(name, wl, world, scaling):
    """The `config` object: identical in both arms (ours / reference) for one workload."""
    ivf = wl["kind"] == "ivf"
    per_gpu = wl["n"] if scaling == "weak" else (wl["n"] + world - 1) // world
    return {"workload": f"{name}: " + (f"IVF K={wl['k_cells']} nprobe={wl['probes']} " if ivf else "") +
                        f"{wl['spec']} d={wl['dims']} N={wl['n'] * (world if scaling == 'weak' else 1)} Q={wl['nq']} R={R} t={T}",
            "spec": wl["spec"], "dims": wl["dims"], "database_codes": wl["n"] * (world if scaling == "weak" else 1),
            "codes_per_gpu": per_gpu, "queries": wl["nq"], "r": R, "t": T,
            "database": "gaussian-mixture vectors encoded with k-means codebooks" if wl["data"] == "encoded"
            else "uniform random codes", "sharding": f"db{world}" if world > 1 else "none"}


def run_ours(qb, name, wl, args, rank, local_rank, world, dist):
    """One workload on the GPU path; returns the JSON object (rank 0) or None."""
    import torch
    from paper_1812_09162_b200.dist import ShardedFlatIndex, ShardedIndex, ShardRange, shard_ivf_lists, shard_ranges
    ivf = wl["kind"] == "ivf"
    spec = qb.allocate_dims(wl["dims"], wl["spec"])
    dtype = "u16" if spec.word_width == 16 else "u8"
    dev = torch.device("cuda", local_rank)
    weak = args.scaling == "weak" and world > 1
    want_cpu = rank == 0 and not args.no_cpu_baseline and (world == 1 or not args.no_parity)
    params = qb.SearchParams(probes=wl.get("probes", 1), r=R, t=T)

    def bcast(arr):
        t = torch.from_numpy(np.ascontiguousarray(arr)).to(dev)
        dist.broadcast(t, 0)
        return t.cpu().numpy()

    if ivf:
        data = make_ivf(qb, spec, wl, True, bcast if world > 1 else None)
        t0 = time.time()
        if world > 1 and not weak:
            kw = shard_ivf_lists(spec, data["packed"], data["boff"], data["ioff"], data["counts"], data["ids"], rank,
                                 world, t_max=max(4096, T))
            idx = qb.IvfIndex(spec, data["cb"], data["coarse"], kw["packed"], kw["list_byte_off"], kw["list_id_off"],
                              kw["list_count"], kw["ids"], device=local_rank, calib_packed=kw["calib_packed"],
                              calib_byte_off=kw["calib_byte_off"], calib_count=kw["calib_count"],
                              global_list_count=kw["global_list_count"])
            del kw
        else:
            # weak: every rank holds a whole index of the workload's size (ids offset per rank); its own heads are
            # the calibration heads, so every rank derives the same map only if the codes agree -- they do (same seed)
            ids = data["ids"] + np.uint32(rank * wl["n"]) if weak else data["ids"]
            idx = qb.IvfIndex(spec, data["cb"], data["coarse"], data["packed"], data["boff"], data["ioff"],
                              data["counts"], ids, device=local_rank)
        sharded = ShardedIndex(idx, local_rank) if world > 1 else None
    else:
        if weak:
            data = make_flat(qb, spec, wl, True)
            shard = ShardRange(rank * wl["n"], wl["n"])
            t0 = time.time()
            sharded = ShardedFlatIndex(spec, data["cb"], data["packed"], shard, data["head"], data["head_n"], local_rank,
                                       global_count=wl["n"] * world)
        else:
            rg = shard_ranges(wl["n"], world, spec.block_len)[rank]
            data = make_flat(qb, spec, wl, True, rg.start, rg.count, whole=want_cpu)
            t0 = time.time()
            sharded = ShardedFlatIndex(spec, data["cb"], data["packed"], rg, data["head"], data["head_n"], local_rank,
                                       global_count=wl["n"])
        idx = sharded.index
        if world == 1:
            sharded = None  # one GPU: the plain index, no merge step
    for opt in args.option:
        k, v = opt.split("=")
        idx.set_option(k, int(v))
    log(f"[bench] rank {rank}: index open (upload + re-layout) {time.time() - t0:.1f}s")

    queries = data["queries"]
    nq = wl["nq"]
    d_q = torch.from_numpy(queries).to(dev)
    d_ids = torch.empty((nq, R), dtype=torch.int32, device=dev)
    d_dists = torch.empty((nq, R), dtype=torch.float32, device=dev)
    d_counts = torch.empty((nq,), dtype=torch.int32, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2
    stream = torch.cuda.current_stream().cuda_stream

    def step():
        flush.zero_()  # evict the code array / tables from L2 between steps
        if sharded is not None:
            sharded.search_device(d_q, params, d_ids, d_dists, d_counts, stream=stream)
        else:
            idx.search_device(d_q, params, d_ids, d_dists, d_counts, stream=stream)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    st_acc = {"ms_scan": 0.0, "ms_lut": 0.0, "ms_select": 0.0, "launches": 0, "scan_launches": 0, "pairs": 0,
              "admitted": 0, "retries": 0}
    with ClockSampler(local_rank) as clocks:
        for _ in range(args.warmup):
            step()
        barrier()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        # nvidia-smi needs a few hundred ms to produce its first sample: keep the GPU busy with untimed
        # steps until it has, so that the clock record covers the timed region even for ms-long workloads
        spin_until = time.time() + 3.0
        while len(clocks.samples) < 3 and time.time() < spin_until:
            step()
        barrier()
        w0 = time.time()
        ev0.record()
        for _ in range(args.steps):
            step()
            st = idx.stats()
            st_acc["ms_scan"] += st.ms_scan
            st_acc["ms_lut"] += st.ms_lut
            st_acc["ms_select"] += st.ms_select
            st_acc["launches"] += st.kernel_launches + (1 if sharded is not None else 0)  # + the merge kernel
            st_acc["scan_launches"] += st.scan_launches
            st_acc["pairs"] += st.pairs_scanned
            st_acc["admitted"] += st.candidates
            st_acc["retries"] += st.overflow_retries
            st_acc["variant"] = int(st.scan_variant)  # the timed batch's kernel (later one-query calls may plan another)
        ev1.record()
        barrier()
        w1 = time.time()
        clk = clocks.summary(w0, w1)
    ms = ev0.elapsed_time(ev1)
    pairs_rank = torch.tensor([float(st_acc["pairs"])], dtype=torch.float64, device=dev)
    if world > 1:
        tmax = torch.tensor([ms], device=dev)
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        ms = float(tmax.item())
        dist.all_reduce(pairs_rank, op=dist.ReduceOp.SUM)  # strong scaling: the shards' pairs add up to the database's
    total_pairs = float(pairs_rank.item())
    pairs_per_step = total_pairs / args.steps  # flat: N*Q; IVF: sum over queries of the probed lists' lengths
    value = total_pairs / (ms * 1e-3)
    got = (d_ids.cpu().numpy().view(np.uint32), d_dists.cpu().numpy(), d_counts.cpu().numpy().astype(np.uint32))

    # ---- e2e: the host-buffer C-ABI call (H2D + D2H inside), same metric ----
    h_q = torch.from_numpy(queries).pin_memory()
    if world == 1:
        qn = h_q.numpy()
        idx.search(qn, params)  # warm the host path (its workspace is sized on first use)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            flush.zero_()
            idx.search(qn, params)
        torch.cuda.synchronize()
        e2e_ms = (time.perf_counter() - t0) * 1e3
    else:
        # multi-GPU e2e: pinned host queries -> device, sharded search + merge, results back to pinned host
        h_ids = torch.empty((nq, R), dtype=torch.int32).pin_memory()
        h_dists = torch.empty((nq, R), dtype=torch.float32).pin_memory()
        h_counts = torch.empty((nq,), dtype=torch.int32).pin_memory()
        barrier()
        ev0.record()
        for _ in range(args.steps):
            flush.zero_()
            d_q.copy_(h_q, non_blocking=True)
            sharded.search_device(d_q, params, d_ids, d_dists, d_counts, stream=stream)
            h_ids.copy_(d_ids, non_blocking=True)
            h_dists.copy_(d_dists, non_blocking=True)
            h_counts.copy_(d_counts, non_blocking=True)
        ev1.record()
        barrier()
        e2e_ms = ev0.elapsed_time(ev1)
        tmax = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        e2e_ms = float(tmax.item())
    e2e_value = total_pairs / (e2e_ms * 1e-3)

    # single-query latency through the host-buffer call (the reference's own calling pattern: one search per query)
    lat_ms = None
    if world == 1:
        q1 = np.ascontiguousarray(queries[:1])
        idx.search(q1, params)
        t0 = time.perf_counter()
        for i in range(20):
            idx.search(np.ascontiguousarray(queries[i % nq: i % nq + 1]), params)
        lat_ms = (time.perf_counter() - t0) * 1e3 / 20

    out = None
    if rank == 0:
        peaks_path = ROOT / "MEASURED_PEAKS.json"
        if peaks_path.exists():
            peak, peak_src = float(json.loads(peaks_path.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
        else:
            peak, peak_src = 6650.0, "fallback (B200_PROFILING.md)"
        scan_s = st_acc["ms_scan"] * 1e-3
        achieved = (st_acc["pairs"] * 8.0 / scan_s) / 1e9 if scan_s > 0 else None
        traffic, traffic_src = None, None
        tpath = ROOT / "profiles" / "traffic.json"  # dram__bytes_read+write of the dominant launch, from ncu --set full
        if tpath.exists():
            traffic = json.loads(tpath.read_text()).get(name)
            traffic_src = "profiles/traffic.json (dram__bytes_read.sum + dram__bytes_write.sum of the dominant launch, " \
                          "one ncu --set full capture of this workload; not measured in this run)"
        variant = int(st_acc.get("variant", idx.stats().scan_variant))
        vname = qb.lib().qadc_variant_name(variant).decode()
        roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                    "frac": achieved / peak if achieved else None, "traffic": traffic, "traffic_source": traffic_src,
                    "peak_source": peak_src, "kernel": "scan_kernel (" + vname + ")",
                    "algorithmic_bytes_per_pair": 8,
                    "avg_launch_ms": st_acc["ms_scan"] / max(st_acc["scan_launches"], 1),
                    "stage_ms_per_step": {k: st_acc[k] / args.steps for k in ("ms_lut", "ms_scan", "ms_select")},
                    "admitted_pairs_per_query": st_acc["admitted"] / args.steps / nq,
                    "overflow_retries": st_acc["retries"],
                    "note": "codes are streamed once per query tile and reused from shared memory, so algorithmic bytes "
                            "exceed DRAM traffic; the kernel's real ceiling is on-chip (profiles/)"}
        # the kernel's operative ceiling: table-lookup bytes through the shared-memory pipe (128 B/clk/SM)
        entry_bytes = {1: 4, 3: 1}.get(variant, 2)
        # merged layouts: 16x{4,4} -> one lookup per code byte (pair sums); 12x{6,5,5} -> two lookups per 16-bit word
        lookups = spec.m // 2 if variant == 9 else spec.m * 2 // 3 if variant == 10 else spec.m
        sm_clock = (clk.get("sm_mhz") or 1965) * 1e6
        prop = torch.cuda.get_device_properties(dev)
        smem_peak = 128.0 * prop.multi_processor_count * sm_clock / 1e9
        smem_ach = (st_acc["pairs"] * lookups * entry_bytes / scan_s) / 1e9 if scan_s > 0 else None
        if variant == 12:
            # the tensor-core scan: one-hot int8 contraction, K = 256 table bytes + 32 threshold bytes per (code, query)
            top = (st_acc["pairs"] * 2.0 * 288 / scan_s) / 1e12 if scan_s > 0 else None
            roofline["tensor"] = {"bound": "tensor (tcgen05 kind::i8)", "achieved": top, "peak": 4492.0, "unit": "TOP/s",
                                  "frac": top / 4492.0 if top else None, "ops_per_pair": 576,
                                  "peak_source": "measured on this pool: back-to-back M=128 N=256 K=256 kind::i8 MMAs on all "
                                                 "SMs, tools/umma_probe.cu (nominal dense int8: 4500 TOP/s)"}
        if variant in (13, 14):
            # the 2:4-sparse form: same contraction (576 logical ops per pair), half of the table part's products skipped.
            # Ceiling = the MMA-only rate of the kernel's own instruction sequence (4 sparse K = 64 + 1 dense K = 32,
            # M = 128, N = 240), measured with nothing else running: 731 cycles per tile per SM.
            sm_n = prop.multi_processor_count
            mma_cycles = 731.0 if variant == 13 else 647.0  # (14: the CTA-pair form, tools/umma2_probe.cu)
            peak_pairs = 128.0 * 240.0 * sm_n * sm_clock / mma_cycles
            top = (st_acc["pairs"] * 576.0 / scan_s) / 1e12 if scan_s > 0 else None
            roofline["tensor"] = {"bound": "tensor (tcgen05 kind::i8, 2:4 sparse)", "achieved": top,
                                  "peak": peak_pairs * 576.0 / 1e12, "unit": "TOP/s (dense-equivalent)",
                                  "frac": top / (peak_pairs * 576.0 / 1e12) if top else None, "ops_per_pair": 576,
                                  "peak_source": "measured on this pool: the kernel's MMA sequence back to back on all SMs, "
                                                 f"{mma_cycles:.0f} cycles per 128 x 240 tile per SM (tools/umma_probe.cu, umma2_probe.cu); the dense kind::i8 peak "
                                                 "measured the same way is 4492 TOP/s"}
        if variant < 12:
            roofline["smem"] = {"bound": "shared-memory pipe", "achieved": smem_ach, "peak": smem_peak, "unit": "GB/s",
                                "frac": smem_ach / smem_peak if smem_ach else None,
                                "bytes_per_pair": lookups * entry_bytes,
                                "peak_source": "128 B/clk/SM x SMs x sampled SM clock"}
        cpu_out, parity = None, None
        if want_cpu:
            cpu = CpuReference(wl, data)
            if world == 1:
                nq_s = cpu.sized_sample(12.0)
                dt = cpu.run(nq_s)
                cpu_out = {"value": pairs_per_step / nq * nq_s / dt, "unit": "codes/s", "cores": cpu.cores,
                           "kind": cpu.kind, "sample": f"{nq_s} of {nq} queries, kernel {cpu.family}, {dt:.2f}s"}
            if not args.no_parity:
                parity = cpu.parity(*got, 64 if ivf else 32)
                log(f"[bench] parity {name}: {parity}")
            cpu.close()
        out = {
            "metric": "ADC codes scanned/s", "value": value, "unit": "codes/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "weak" if weak or world == 1 else "strong",
            "vs_baseline": None, "dtype": dtype, "data": "synthetic",
            "config": describe(name, wl, world, "weak" if weak else "strong"),
            "pairs_per_step": pairs_per_step,
            "l2": "flushed between steps (256 MiB write inside the timed region); the code array is also re-streamed "
                  "once per query tile",
            "clocks": clk, "gpu_launches": int(st_acc["launches"]),
            "e2e": {"value": e2e_value, "unit": "codes/s", "h2d_bytes_per_step": int(nq * wl["dims"] * 4),
                    "d2h_bytes_per_step": int(nq * R * 8 + nq * 4), "ms_per_step": e2e_ms / args.steps},
            "roofline": roofline, "cpu_baseline": cpu_out, "parity": parity,
            "single_query_latency_ms": lat_ms,
            "per_gpu_value": value / world,
        }
    idx.close()
    del d_q, d_ids, d_dists, d_counts, flush, data
    torch.cuda.empty_cache()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default=os.environ.get("QADC_WORKLOAD", "c4"), choices=sorted(WORKLOADS))
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="N > 1: split ONE database over the ranks (default) or keep the workload's N per GPU")
    ap.add_argument("--also", default=os.environ.get("QADC_ALSO", "c1,c2,c3,c5g"),
                    help="N = 1: further BASELINE configs measured briefly after the headline one and carried under "
                         "'other_configs' ('' = none)")
    ap.add_argument("--n", type=int, default=0, help="override the database size (debug)")
    ap.add_argument("--nq", type=int, default=0, help="override query count (debug)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--option", action="append", default=[], help="name=value passed to qadc_set_option")
    args = ap.parse_args()
    if args.impl == "ours":
        args.warmup = max(args.warmup, 3)

    wl = dict(WORKLOADS[args.workload])
    if args.n:
        wl["n"] = args.n
    if args.nq:
        wl["nq"] = args.nq
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    ivf = wl["kind"] == "ivf"

    if args.impl == "reference" and rank != 0:
        return 0

    import paper_1812_09162_b200 as qb
    qb.build()
    have_gpu = qb.lib().qadc_device_count() > 0
    spec = qb.allocate_dims(wl["dims"], wl["spec"])
    dtype = "u16" if spec.word_width == 16 else "u8"

    # -------------------------------------------------------------- reference arm --
    if args.impl == "reference":
        # the reference's own CPU path on the WHOLE database of the workload (it has no sharding), all host cores
        scaling = "weak" if args.scaling == "weak" and args.gpus > 1 else "strong"
        data = make_ivf(qb, spec, wl, have_gpu) if ivf else make_flat(qb, spec, wl, have_gpu)
        cpu = CpuReference(wl, data)
        nq_step = cpu.sized_sample(6.0)
        ppq = cpu.pairs_per_query(data, nq_step)
        times = []
        for i in range(args.warmup + args.steps):
            dt = cpu.run(nq_step)
            if i >= args.warmup:
                times.append(dt)
        tot_t = sum(times)
        value = ppq * nq_step * len(times) / tot_t
        print(json.dumps({
            "impl": "reference", "metric": "ADC codes scanned/s", "value": value, "unit": "codes/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * tot_t / max(len(times), 1), "higher_is_better": True,
            "scaling": "weak" if scaling == "weak" or args.gpus == 1 else "strong",
            "vs_baseline": None, "dtype": dtype, "data": "synthetic",
            "config": describe(args.workload, wl, args.gpus, scaling),
            "cpu_baseline": {"value": value, "unit": "codes/s", "cores": cpu.cores, "kind": cpu.kind,
                             "sample": f"each step: {nq_step} of {wl['nq']} queries, kernel {cpu.family}"},
            "e2e": {"value": value, "unit": "codes/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}))
        cpu.close()
        return 0

    # --------------------------------------------------------------------- our arm --
    import torch
    if not have_gpu:
        raise SystemExit("bench.py: no CUDA device; the product has no CPU path (use --impl reference for the CPU arm)")
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    out = run_ours(qb, args.workload, wl, args, rank, local_rank, world, dist)
    rc = 0
    if rank == 0:
        if out["parity"] and out["parity"]["mismatches"]:
            rc = 3
        others = []
        if world == 1 and args.also and not args.n and not args.nq:
            # the other BASELINE configs, briefly (2 steps, no CPU timing; parity still checked): context for the
            # headline line, each a complete line of its own under "other_configs"
            import copy
            a2 = copy.copy(args)
            a2.steps, a2.warmup, a2.no_cpu_baseline = 3, 3, False
            for name in [x for x in args.also.split(",") if x and x != args.workload]:
                try:
                    a2.no_cpu_baseline = False
                    o = run_ours(qb, name, dict(WORKLOADS[name]), a2, 0, local_rank, 1, None)
                    keep = ("value", "unit", "ms_per_step", "steps", "warmup", "dtype", "config", "pairs_per_step",
                            "gpu_launches", "e2e", "parity", "single_query_latency_ms", "cpu_baseline")
                    rec = {k: o[k] for k in keep}
                    rec["roofline"] = {k: o["roofline"][k] for k in ("achieved", "peak", "frac", "kernel", "stage_ms_per_step")}
                    others.append(rec)
                    if o["parity"] and o["parity"]["mismatches"]:
                        rc = 3
                except Exception as e:  # an extra config must never take the headline line down
                    others.append({"config": {"workload": name}, "error": f"{type(e).__name__}: {e}"})
        out["other_configs"] = others
        print(json.dumps(out))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return rc


if __name__ == "__main__":
    sys.exit(main())
