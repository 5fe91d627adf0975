"""Precision probe for the complex64 engine step paths (tensor-core vs SIMT).

Network 0-1-2: step 1 is acc[M, K] x S1[K, N] (the probed step), step 2 closes
against S2[M, N].  Prints |err| / sum|terms| so cancellation does not inflate it.
Run under different TNC_KERNELS settings."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2011_02621_b200.engine import ContractionPlan, NetworkSpec, PathExecutor  # noqa: E402


def probe(M, K, N, seed=0, dtype="complex64"):
    rng = np.random.default_rng(seed)
    edges = {(0, 1): K, (0, 2): M, (1, 2): N}
    legs = {0: [(0, 1), (0, 2)], 1: [(0, 1), (1, 2)], 2: [(0, 2), (1, 2)]}
    spec = NetworkSpec([0, 1, 2], edges, legs)
    sites = {}
    for q in range(3):
        dims = spec.site_dims(q)
        sites[q] = (rng.standard_normal((1,) + dims) + 1j * rng.standard_normal((1,) + dims)).astype(np.complex64).astype(np.complex128)
    plan = ContractionPlan(spec, [0, 1, 2])
    ex = PathExecutor(plan, {q: torch.from_numpy(sites[q]) for q in range(3)}, dtype=dtype)
    amp = torch.zeros(1, dtype=ex.tdtype, device="cuda")
    ex.run(None, 1, amp)
    got = complex(amp.cpu().numpy()[0])
    a = np.einsum("km->mk", sites[0][0]) if spec.site_dims(0) == (K, M) else sites[0][0]
    # generic reference by labels
    sub = {(0, 1): "k", (0, 2): "m", (1, 2): "n"}
    ein = ",".join("".join(sub[l] for l in legs[q]) for q in range(3)) + "->"
    ref = np.einsum(ein, *(sites[q][0] for q in range(3)))
    scale = np.einsum(ein, *(np.abs(sites[q][0]) for q in range(3)))
    steps = [(s.M, s.K, s.N) for s in plan.steps]
    return abs(got - ref) / scale, steps


if __name__ == "__main__":
    for M, K, N in [(128, 64, 4), (128, 256, 4), (128, 1024, 4), (128, 4096, 4), (128, 16384, 4),
                    (256, 1024, 64), (256, 4096, 64), (128, 4096, 128)]:
        errs = [probe(M, K, N, seed=s)[0] for s in range(3)]
        print(f"M={M} K={K} N={N} err/scale max={max(errs):.3e} steps={probe(M, K, N)[1]}", flush=True)
