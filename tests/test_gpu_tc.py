"""Tensor-core (tcgen05 3xTF32) contraction path vs the CPU oracle."""

import numpy as np
import pytest

import tn_oracle as O

pytestmark = pytest.mark.gpu


def rel_l2(got, ref):
    return float(np.linalg.norm(np.asarray(got) - ref) / np.linalg.norm(ref))


@pytest.mark.parametrize("r,k,n,B", [(7, 1, 2, 2), (7, 2, 2, 3), (8, 3, 3, 2), (9, 1, 3, 2), (9, 3, 2, 3),
                                     (10, 2, 3, 1), (11, 3, 3, 1), (7, 3, 2, 1), (8, 3, 1, 3), (9, 3, 1, 1)])
def test_tc_pair_matches_oracle(r, k, n, B):
    import torch

    from paper_2011_02621_b200.engine import PairPlan

    rng = np.random.default_rng(1000 + r * 100 + k * 10 + n)
    perm = list(rng.permutation(r + k))
    dims = [2 if x < r else 4 for x in perm]
    size = int(np.prod(dims))
    acc = ((rng.standard_normal((B, size)) + 1j * rng.standard_normal((B, size))) / np.sqrt(2)).astype(np.complex64)
    site = ((rng.standard_normal((2,) + (4,) * (k + n)) + 1j * rng.standard_normal((2,) + (4,) * (k + n))) / 2
            ).astype(np.complex64)
    bits = rng.integers(0, 2, B)
    shared_pos = sorted((i for i, x in enumerate(perm) if x >= r), key=lambda i: perm[i])
    pairs = [(p, j) for j, p in enumerate(shared_pos)]
    plan = PairPlan(dims, [4] * (k + n), pairs, dtype="complex64")
    K, N = 4 ** k, 4 ** n
    if K * N >= 256:
        assert plan.kernel == "tcgen05-3xtf32"
    ta = torch.from_numpy(acc).cuda()
    sb = torch.from_numpy(np.ascontiguousarray(site[bits].reshape(B, -1))).cuda()
    out = torch.empty((B, size // K * N), dtype=torch.complex64, device="cuda")
    plan(ta, sb, out, B, size, K * N, size // K * N)
    torch.cuda.synchronize()
    ref = O.sweep_step(acc.astype(np.complex128), perm, r, k, site.astype(np.complex128), bits)
    err = rel_l2(out.cpu().numpy(), ref)
    assert err <= 2e-6, err


def test_tc_engine_step_contiguous():
    """Engine-layout step (accumulator rows contiguous) through tnc_step."""
    import torch

    from paper_2011_02621_b200 import AmplitudeEngine, pattern_rqc, sycamore53_graph

    graph, pats, _ = sycamore53_graph()
    seq = [pats[ch] for ch in "ABCDCDAB"]
    c = pattern_rqc(graph, seq, 5, seed=4)
    rng = np.random.default_rng(2)
    outs = ["".join(rng.choice(["0", "1"], 53)) for _ in range(6)]
    e128 = AmplitudeEngine(c, dtype="complex128", max_rank=10)
    ref = e128.amplitudes(outs)
    e64 = AmplitudeEngine(c, dtype="complex64", max_rank=10)
    kn = [(sp.K, sp.N, sp.M, sp.c_rows_contig) for sp in e64.plan.steps]
    got = e64.amplitudes(outs)
    assert rel_l2(got, ref) <= 1e-4, (rel_l2(got, ref), kn)
