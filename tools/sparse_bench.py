"""Sparse (CSR truncated Taylor) mixer timing: the hypercube sum_j X_j as CSR at n qubits."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2110_03963_b200 as Q
n = int(sys.argv[1]) if len(sys.argv) > 1 else 20
N = 1 << n
rows = np.arange(N)
col = np.stack([rows ^ (1 << j) for j in range(n)], axis=1).astype(np.int32).ravel()
row_ptr = (np.arange(N + 1) * n).astype(np.int64)
q = np.random.default_rng(0).standard_normal(N)
with Q.Plan(N, "sparse") as P:
    P.set_qualities(q)
    P.set_sparse_mixer(row_ptr, col)
    P.apply_mixer(0.3)
    P.set_profiling(True); P.reset_kernel_stats()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(5):
        P.apply_mixer(0.7)
    torch.cuda.synchronize(); dt = (time.perf_counter() - t0) / 5
    k = P.kernel_stats("spmv")
    print("n=%d nnz=%d: %.3f ms per mixer, %d SpMV launches per mixer, %.3f ms SpMV time, %.0f GB/s algorithmic"
          % (n, len(col), dt * 1e3, k["launches"] // 5, k["ms"] / 5, k["bytes"] / (k["ms"] * 1e-3) / 1e9))
