"""configs[1] at the bench's own sizes: every (r, k, n, B) case of
bench.sweep_cases() (operands up to 2^32 elements, r up to 28) is contracted
at full size through the C ABI (PairPlan + projection gather, the bench's exact
layouts and seeds) and checked on sampled result rows against the oracle's
algebra in complex128: out[b, f, :] = sum_k acc[b, f, k] S[bits[b]][k, :]
(reference tensor.py:100-115 / oracle sweep_step), rel L2 <= 2e-6."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_every_bench_sweep_case_full_size():
    import torch

    import bench
    from paper_2011_02621_b200 import _native
    from paper_2011_02621_b200.engine import PairPlan, project_variants

    _native.require_device()
    dev = torch.device("cuda", 0)
    cases, _ = bench.sweep_cases()
    assert any(r == 28 for r, *_ in cases)
    max_acc = max(B * 2 ** r * 4 ** k for r, k, n, B in cases)
    max_out = max(B * 2 ** r * 4 ** n for r, k, n, B in cases)
    g = torch.Generator(device=dev)
    g.manual_seed(5)
    acc = torch.randn(max_acc, dtype=torch.complex64, device=dev, generator=g)
    out = torch.empty(max_out, dtype=torch.complex64, device=dev)
    rng = np.random.default_rng(9)
    worst = 0.0
    for ci, (r, k, n, B) in enumerate(cases):
        perm, dims, pairs = bench.case_layout(r, k, n, seed=ci)
        K, N = 4 ** k, 4 ** n
        plan = PairPlan(dims, [4] * (k + n), pairs, dtype="complex64")
        variants = torch.randn((2, K * N), dtype=torch.complex64, device=dev, generator=g)
        bits = torch.randint(0, 2, (B,), dtype=torch.int32, device=dev, generator=g)
        site = torch.empty((B, K * N), dtype=torch.complex64, device=dev)
        project_variants(variants, bits, site, K * N)
        a_z, o_z = 2 ** r * K, 2 ** r * N
        out[: B * o_z].fill_(float("nan"))
        plan(acc, site, out, B, a_z, K * N, o_z)
        torch.cuda.synchronize()
        # sampled rows: (b, f) pairs, f = the free-leg digits in acc axis order
        strides = np.cumprod([1] + [int(d) for d in dims[::-1]])[::-1][1:]
        free_pos = [i for i, x in enumerate(perm) if x < r]
        shared_pos = [p for p, _ in sorted(pairs, key=lambda t: t[1])]
        ns = 48
        bs = rng.integers(0, B, ns)
        fs = rng.integers(0, 2 ** r, ns)
        fbits = (fs[:, None] >> np.arange(r - 1, -1, -1)[None, :]) & 1
        base = bs * a_z + (fbits * strides[free_pos][None, :]).sum(1)
        kd = np.stack(np.unravel_index(np.arange(K), (4,) * k), 1)
        koff = (kd * strides[shared_pos][None, :]).sum(1)
        idx = torch.from_numpy((base[:, None] + koff[None, :]).astype(np.int64)).to(dev)
        a_s = acc[idx].cpu().numpy().astype(np.complex128)                       # [ns, K]
        v = variants.cpu().numpy().astype(np.complex128).reshape(2, K, N)
        bh = bits.cpu().numpy()
        ref = np.einsum("sk,skn->sn", a_s, v[bh[bs]])
        oidx = torch.from_numpy((bs * o_z + fs * N)[:, None] + np.arange(N)[None, :]).to(dev)
        got = out[oidx].cpu().numpy().astype(np.complex128)
        err = float(np.linalg.norm(got - ref) / np.linalg.norm(ref))
        worst = max(worst, err)
        assert err <= 2e-6, (r, k, n, B, plan.kernel, err)
    assert worst <= 2e-6
