#!/usr/bin/env python
"""bench.py -- throughput of the Quicker ADC scan path on B200 (metric of BASELINE.json).

    python bench.py --gpus N --steps K --warmup W [--workload c2] [--impl reference]

A "step" is one pass of the whole hot path (distance tables -> calibration -> quantization -> scan ->
top-R [-> multi-GPU merge]) over one batch of synthetic queries against the resident database.
``value``   = (query, code) pairs evaluated per second, whole job, inputs already in HBM;
``e2e``     = the same metric through the reference-facing C-ABI call with HOST buffers
              (qadc_search_batch: H2D of the queries and D2H of ids/dists/counts inside the timed region);
``roofline``= algorithmic code bytes (8 B per pair) / CUDA-event time of the scan kernels, against the
              measured HBM copy bandwidth of MEASURED_PEAKS.json;
``cpu_baseline`` = the reference's own CPU search (oracle/_ref when it was built, else the oracle port)
              timed on this box's host cores on a bounded query sample of the same workload.

Workloads (BASELINE.json configs; seeded synthetic inputs with the named shapes stand in for the
SIFT/Deep-like data, see paper_1812_09162_b200/synth.py):
  c1  16x{4,4}    d=128  N=1e6   Q=1e3     c3  8x{8,8}   d=128  N=1e7  Q=1e4
  c2  12x{6,5,5}  d=96   N=1e7   Q=1e4     c4  16x{4,4}  d=128  N=2e8  Q=1e4 (uniform random codes)
Default c2 (configs[1]).  With --gpus N > 1 (torchrun, one rank per GPU) every rank holds one database
shard of the per-GPU size above (weak scaling), queries are replicated and the per-query top-R lists are
merged after one NCCL all_gather.
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
    "c1": dict(spec="16x{4,4}", dims=128, n=1_000_000, nq=1_000, data="encoded"),
    "c2": dict(spec="12x{6,5,5}", dims=96, n=10_000_000, nq=10_000, data="encoded"),
    "c3": dict(spec="8x{8,8}", dims=128, n=10_000_000, nq=10_000, data="encoded"),
    "c4": dict(spec="16x{4,4}", dims=128, n=200_000_000, nq=10_000, data="random"),
}
R, T = 100, 400


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ----------------------------------------------------------------------------- data --

def make_database(qb, spec, wl, rank, have_gpu):
    """Packed shard for this rank (seeded by rank) + the global head (rank 0's first codes)."""
    from paper_1812_09162_b200 import synth
    dims, n = wl["dims"], wl["n"]
    centres = synth.mixture_centres(dims, seed=1)
    train = synth.gaussian_mixture(100_000, dims, seed=4, centres=centres)
    t0 = time.time()
    cb = synth.train_codebook(spec, train, iters=8, seed=5)
    log(f"[bench] codebook ({spec.cb_floats} floats) trained in {time.time() - t0:.1f}s")

    def encode(vecs):
        if have_gpu:
            return qb.encode(spec, cb, vecs)
        from oracle.pyoracle import Oracle  # reference arm on a box without a GPU: CPU encoder
        o = Oracle("port")
        return o.encode(o.spec(dims, wl["spec"]), cb, vecs)

    def shard_codes(r, count, first_only=None):
        if wl["data"] == "random":
            return None
        parts, done, batch = [], 0, 500_000
        b = 0
        while done < count:
            nb = min(batch, count - done)
            vecs = synth.gaussian_mixture(nb, dims, seed=2 + 1000 * r + b, centres=centres)
            parts.append(encode(vecs))
            done += nb
            b += 1
            if first_only and done >= first_only:
                break
        return np.concatenate(parts)

    t0 = time.time()
    if wl["data"] == "random":
        packed = synth.random_packed(spec, n, seed=6 + 1000 * rank)
        # the global head (first codes of rank 0's shard) comes from its own seed so that every rank can
        # regenerate it without rank 0's stream; rank 0 splices it in front of its shard
        head_n = min(4096, n) // spec.block_len * spec.block_len
        head = synth.random_packed(spec, head_n, seed=600)
        if rank == 0:
            packed[: head.size] = head
    else:
        codes = shard_codes(rank, n)
        packed = qb.pack_list(spec, codes)
        head_n = min(4096, n)
        head_codes = codes[:head_n] if rank == 0 else shard_codes(0, head_n, first_only=head_n)[:head_n]
        head = qb.pack_list(spec, head_codes)
    log(f"[bench] rank {rank}: database shard of {n} codes ready in {time.time() - t0:.1f}s")
    queries = synth.gaussian_mixture(wl["nq"], dims, seed=3, centres=centres)
    return cb, packed, head, head_n, queries


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

def cpu_reference_rate(wl, cb, packed, queries, budget_s=12.0, max_queries=None):
    """The reference's CPU search on the host cores (query-parallel pool, all cores), bounded sample."""
    from oracle.pyoracle import Oracle, build
    build()
    kind = "reference" if Oracle.available("reference") else "port"
    o = Oracle(kind)
    s = o.spec(wl["dims"], wl["spec"])
    cores = os.cpu_count() or 1
    fam = 1  # auto: the natural SIMD family when the host supports it
    n = wl["n"]
    probe = min(len(queries), cores)
    t0 = time.perf_counter()
    o.flat_search(s, cb, packed, n, queries[:probe], r=R, t=T, family=fam, threads=cores)
    dt = max(time.perf_counter() - t0, 1e-4)
    nq = int(min(len(queries), max(probe, budget_s / dt * probe)))
    if max_queries:
        nq = min(nq, max_queries)
    t0 = time.perf_counter()
    o.flat_search(s, cb, packed, n, queries[:nq], r=R, t=T, family=fam, threads=cores)
    dt = time.perf_counter() - t0
    family = o.auto_family(s) if kind == "reference" else "scalar-quantized (C port)"
    return {"value": n * nq / dt, "unit": "codes/s", "cores": cores, "kind": kind,
            "sample": f"{nq} of {len(queries)} queries x {n} codes, kernel {family}, {dt:.2f}s"}, nq, dt


# ------------------------------------------------------------------------------ main --

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default=os.environ.get("QADC_WORKLOAD", "c2"), choices=sorted(WORKLOADS))
    ap.add_argument("--n", type=int, default=0, help="override codes per GPU (debug)")
    ap.add_argument("--nq", type=int, default=0, help="override query count (debug)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--option", action="append", default=[], help="name=value passed to qadc_set_option")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup

    wl = dict(WORKLOADS[args.workload])
    if args.n:
        wl["n"] = args.n
    if args.nq:
        wl["nq"] = args.nq
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))

    if args.impl == "reference" and rank != 0:
        return 0

    import paper_1812_09162_b200 as qb
    qb.build()
    have_gpu = qb.lib().qadc_device_count() > 0
    spec = qb.allocate_dims(wl["dims"], wl["spec"])
    config = {"workload": f"{args.workload}: {wl['spec']} d={wl['dims']} N={wl['n']}/GPU Q={wl['nq']} R={R} t={T}",
              "spec": wl["spec"], "dims": wl["dims"], "codes_per_gpu": wl["n"], "queries": wl["nq"], "r": R, "t": T,
              "database": "gaussian-mixture vectors encoded with k-means codebooks" if wl["data"] == "encoded"
              else "uniform random codes", "sharding": f"db{world}" if world > 1 else "none"}

    # -------------------------------------------------------------- reference arm --
    if args.impl == "reference":
        cb, packed, head, head_n, queries = make_database(qb, spec, wl, 0, have_gpu)
        per_step = []
        base = None
        nq_step = None
        for i in range(args.warmup + args.steps):
            base, nq_used, dt = cpu_reference_rate(wl, cb, packed, queries, budget_s=8.0, max_queries=nq_step)
            nq_step = nq_used
            if i >= args.warmup:
                per_step.append((nq_used, dt))
        tot_pairs = sum(n for n, _ in per_step) * wl["n"]
        tot_t = sum(t for _, t in per_step)
        value = tot_pairs / tot_t
        base["value"] = value
        print(json.dumps({
            "impl": "reference", "metric": "ADC codes scanned/s", "value": value, "unit": "codes/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot_t / max(args.steps, 1),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u16" if spec.word_width == 16 else "u8",
            "data": "synthetic", "config": config, "cpu_baseline": base,
            "e2e": {"value": value, "unit": "codes/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}))
        return 0

    # --------------------------------------------------------------------- our arm --
    import torch
    if not have_gpu:
        raise SystemExit("bench.py: no CUDA device; the product has no CPU path (use --impl reference for the CPU arm)")
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    cb, packed, head, head_n, queries = make_database(qb, spec, wl, rank, have_gpu)

    from paper_1812_09162_b200.dist import ShardedFlatIndex, ShardRange
    t0 = time.time()
    sharded = ShardedFlatIndex(spec, cb, packed, ShardRange(rank * wl["n"], wl["n"]), head, head_n, local_rank)
    idx = sharded.index
    for opt in args.option:
        k, v = opt.split("=")
        idx.set_option(k, int(v))
    log(f"[bench] rank {rank}: index open (upload + re-layout) {time.time() - t0:.1f}s")

    nq = wl["nq"]
    params = qb.SearchParams(r=R, t=T)
    d_q = torch.from_numpy(queries).to(dev)
    d_ids = torch.empty((nq, R), dtype=torch.int32, device=dev)
    d_dists = torch.empty((nq, R), dtype=torch.float32, device=dev)
    d_counts = torch.empty((nq,), dtype=torch.int32, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2
    stream = torch.cuda.current_stream().cuda_stream

    def step():
        flush.zero_()  # evict the code array / tables from L2 between steps
        sharded.search_device(d_q, params, d_ids, d_dists, d_counts, stream=stream)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    st_acc = {"ms_scan": 0.0, "ms_lut": 0.0, "ms_select": 0.0, "launches": 0, "scan_launches": 0, "pairs": 0}
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
            st_acc["launches"] += st.kernel_launches + (1 if True else 0)  # + the merge kernel
            st_acc["scan_launches"] += st.scan_launches
            st_acc["pairs"] += st.pairs_scanned
        ev1.record()
        barrier()
        w1 = time.time()
        clk = clocks.summary(w0, w1)
    ms = ev0.elapsed_time(ev1)
    if world > 1:
        tmax = torch.tensor([ms], device=dev)
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        ms = float(tmax.item())
    total_pairs = float(wl["n"]) * nq * world * args.steps
    value = total_pairs / (ms * 1e-3)

    # ---- e2e: the host-buffer C-ABI call (H2D + D2H inside), same metric ----
    h_q = torch.from_numpy(queries).pin_memory()
    e2e_ms = None
    if world == 1:
        qn = h_q.numpy()
        idx.search(qn, params)  # warm the host path (its workspace is sized on first use)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            flush.zero_()
            res = idx.search(qn, params)
        torch.cuda.synchronize()
        e2e_ms = (time.perf_counter() - t0) * 1e3
        e2e_value = float(wl["n"]) * nq * args.steps / (e2e_ms * 1e-3)
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

    if rank == 0:
        peaks_path = ROOT / "MEASURED_PEAKS.json"
        if peaks_path.exists():
            peak, peak_src = float(json.loads(peaks_path.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
        else:
            peak, peak_src = 6650.0, "fallback (B200_PROFILING.md)"
        scan_s = st_acc["ms_scan"] * 1e-3
        achieved = (st_acc["pairs"] * 8.0 / scan_s) / 1e9 if scan_s > 0 else None
        roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                    "frac": achieved / peak if achieved else None, "traffic": None, "peak_source": peak_src,
                    "kernel": "scan_kernel (" + qb.lib().qadc_variant_name(idx.stats().scan_variant).decode() + ")",
                    "algorithmic_bytes_per_pair": 8,
                    "avg_launch_ms": st_acc["ms_scan"] / max(st_acc["scan_launches"], 1),
                    "stage_ms_per_step": {k: st_acc[k] / args.steps for k in ("ms_lut", "ms_scan", "ms_select")},
                    "note": "codes are reused across the query tile from shared memory/L2, so algorithmic bytes exceed DRAM traffic"}
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            cpu, _, _ = cpu_reference_rate(wl, cb, packed, queries)
        out = {
            "metric": "ADC codes scanned/s", "value": value, "unit": "codes/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u16" if spec.word_width == 16 else "u8", "data": "synthetic",
            "config": dict(config, l2="flushed between steps (256 MiB write inside the timed region); the code array "
                                      "is also re-streamed once per query tile"),
            "clocks": clk, "gpu_launches": int(st_acc["launches"]),
            "e2e": {"value": e2e_value, "unit": "codes/s", "h2d_bytes_per_step": int(nq * wl["dims"] * 4),
                    "d2h_bytes_per_step": int(nq * R * 8 + nq * 4), "ms_per_step": e2e_ms / args.steps},
            "roofline": roofline, "cpu_baseline": cpu,
            "per_gpu_value": value / world,
        }
        print(json.dumps(out))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
