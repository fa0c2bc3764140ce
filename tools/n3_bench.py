"""Throughput of the GPU IVF list construction (N3) at C5's shape: K=16384 cells, d=96, 12x{6,5,5}."""
import time
import numpy as np
import paper_1812_09162_b200 as qb

rng = np.random.default_rng(0)
dims, text, k, n = 96, "12x{6,5,5}", 16384, 1 << 19
s = qb.allocate_dims(dims, text)
cb = rng.standard_normal(s.cb_floats).astype(np.float32)
coarse = (rng.standard_normal((k, dims)) * 3).astype(np.float32)
v = (rng.standard_normal((n, dims)) * 3).astype(np.float32)
qb.ivf_assign_encode(s, cb, coarse, v[:4096])
t0 = time.perf_counter()
a, c = qb.ivf_assign_encode(s, cb, coarse, v)
t1 = time.perf_counter()
print(f"assign+encode: {n} vectors x {k} cells d={dims}: {t1 - t0:.3f} s  ({n / (t1 - t0) / 1e6:.2f} M vectors/s, "
      f"{2 * 3 * n * k * dims / (t1 - t0) / 1e12:.2f} fp64 TFLOP/s in the assignment)")
t0 = time.perf_counter()
b = qb.build_ivf_lists(s, cb, coarse, v)
print(f"build_ivf_lists incl. host pack: {time.perf_counter() - t0:.3f} s; cells used {np.count_nonzero(b['list_count'])}")
