"""The Tensor / contract_pair API (reference tensor.py:100-115 and its test
strategy, pkg/tests/test_tensor.py::TestContractPair): argument errors are
raised on the host before any device work (CPU tests); the contractions run
through tnc_contract_pair on the GPU and are checked against an explicit
index-loop contraction."""

import itertools
import random

import numpy as np
import pytest

from paper_2011_02621_b200.tensor import Tensor, TensorError, contract_pair


def loop_contract(a, b, pairs):
    """Sum over the paired indices with explicit loops (result axes: free axes
    of a, then free axes of b)."""
    fa = [i for i in range(a.rank) if i not in {p for p, _ in pairs}]
    fb = [j for j in range(b.rank) if j not in {q for _, q in pairs}]
    out_dims = [a.dims[i] for i in fa] + [b.dims[j] for j in fb]
    out = np.zeros(out_dims, dtype=np.complex128)
    shared = [a.dims[p] for p, _ in pairs]
    for idx in itertools.product(*[range(d) for d in out_dims]):
        ia = [0] * a.rank
        ib = [0] * b.rank
        for k, i in enumerate(fa):
            ia[i] = idx[k]
        for k, j in enumerate(fb):
            ib[j] = idx[len(fa) + k]
        total = 0j
        for s in itertools.product(*[range(d) for d in shared]):
            for (p, q), v in zip(pairs, s):
                ia[p] = v
                ib[q] = v
            total += a.data[tuple(ia)] * b.data[tuple(ib)]
        out[idx] = total
    return out


def crandn(rng, *shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


# ---- argument errors (host side, no device needed) ----

def test_extent_mismatch():
    a = Tensor(np.zeros((2, 3)), ("a", "b"))
    b = Tensor(np.zeros(4), ("c",))
    with pytest.raises(TensorError, match="mismatch"):
        contract_pair(a, b, [(1, 0)])


def test_axis_out_of_range():
    a = Tensor(np.zeros(2), ("a",))
    b = Tensor(np.zeros(2), ("b",))
    with pytest.raises(TensorError, match="out of range"):
        contract_pair(a, b, [(3, 0)])


def test_repeated_axis_rejected():
    a = Tensor(np.zeros((2, 2)), ("a", "b"))
    b = Tensor(np.zeros((2, 2)), ("c", "d"))
    with pytest.raises(TensorError, match="repeated"):
        contract_pair(a, b, [(0, 0), (0, 1)])


def test_duplicate_labels_rejected():
    with pytest.raises(TensorError):
        Tensor(np.zeros((2, 2)), ("a", "a"))


# ---- device contractions ----

@pytest.mark.gpu
def test_identity_contraction():
    a = Tensor(np.eye(2), ("r", "c"))
    b = Tensor(np.array([3.0, 4.0]), ("v",))
    out = contract_pair(a, b, [(1, 0)])
    np.testing.assert_allclose(out.data, [3, 4])
    assert out.labels == ("r",)


@pytest.mark.gpu
def test_dot_product_is_rank0():
    a = Tensor(np.array([1.0, 2.0]), ("x",))
    b = Tensor(np.array([3.0, 4.0]), ("y",))
    out = contract_pair(a, b, [(0, 0)])
    assert out.rank == 0
    assert out.scalar() == pytest.approx(11)


@pytest.mark.gpu
def test_outer_product_no_pairs():
    rng = np.random.default_rng(3)
    a = Tensor(crandn(rng, 2, 3), ("a", "b"))
    b = Tensor(crandn(rng, 3), ("c",))
    out = contract_pair(a, b, [])
    assert out.dims == (2, 3, 3)
    np.testing.assert_allclose(out.data, np.multiply.outer(a.data, b.data), atol=1e-12)


@pytest.mark.gpu
def test_against_loop_oracle():
    rng = np.random.default_rng(0)
    a = Tensor(crandn(rng, 2, 4, 2), ("a", "b", "c"))
    b = Tensor(crandn(rng, 2, 2, 3), ("d", "e", "f"))
    out = contract_pair(a, b, [(0, 1)])
    assert out.dims == (4, 2, 2, 3)
    np.testing.assert_allclose(out.data, loop_contract(a, b, [(0, 1)]), atol=1e-12)


@pytest.mark.gpu
def test_loop_oracle_random_shapes():
    """Ragged extents (1..4, not powers of two), 0..min(ra, rb) pairs in random
    axis order: the generic kernel and the tiled kernels."""
    rng = np.random.default_rng(1)
    rnd = random.Random(1)
    for _ in range(25):
        ra, rb = rnd.randint(1, 3), rnd.randint(1, 3)
        da = [rnd.randint(1, 4) for _ in range(ra)]
        db = [rnd.randint(1, 4) for _ in range(rb)]
        npairs = rnd.randint(0, min(ra, rb))
        pairs = list(zip(rnd.sample(range(ra), npairs), rnd.sample(range(rb), npairs)))
        for pa, pb in pairs:
            db[pb] = da[pa]
        a = Tensor(crandn(rng, *da), tuple(f"a{i}" for i in range(ra)))
        b = Tensor(crandn(rng, *db), tuple(f"b{i}" for i in range(rb)))
        out = contract_pair(a, b, pairs)
        np.testing.assert_allclose(out.data, loop_contract(a, b, pairs), atol=1e-12)


@pytest.mark.gpu
@pytest.mark.parametrize("alpha", [0j, 1 + 0j, -3 + 2j, 5 - 5j])
def test_bilinear_in_first_argument(alpha):
    rng = np.random.default_rng(7)
    a = Tensor(crandn(rng, 3, 2), ("a", "b"))
    b = Tensor(crandn(rng, 2, 3), ("c", "d"))
    lhs = contract_pair(Tensor(alpha * a.data, a.labels), b, [(1, 0)])
    rhs = contract_pair(a, b, [(1, 0)])
    np.testing.assert_allclose(lhs.data, alpha * rhs.data, atol=1e-12)


# ---- batched C-ABI edge cases (engine.contract_pair_device) ----

@pytest.mark.gpu
def test_empty_batch_is_noop():
    import torch

    from paper_2011_02621_b200.engine import contract_pair_device

    ta = torch.ones(8, dtype=torch.complex64, device="cuda")
    tb = torch.ones(4, dtype=torch.complex64, device="cuda")
    out = contract_pair_device(ta, [2, 4], tb, [4], [(1, 0)], batch=0)
    torch.cuda.synchronize()
    assert tuple(out.shape) == (0, 2)


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", ["complex64", "complex128"])
def test_broadcast_site_and_conjugate(dtype):
    """z-stride 0 on b (one site block for every batch element), conj_b, and an
    output permutation, against numpy."""
    import torch

    from paper_2011_02621_b200.engine import contract_pair_device

    rng = np.random.default_rng(4)
    B, a_dims, b_dims = 5, [3, 2, 4, 2], [4, 3, 2]
    pairs = [(2, 0), (0, 1)]
    a = crandn(rng, B, *a_dims)
    b = crandn(rng, *b_dims)
    tdt = torch.complex64 if dtype == "complex64" else torch.complex128
    ta = torch.from_numpy(a.reshape(B, -1)).to("cuda", tdt)
    tb = torch.from_numpy(b.reshape(-1)).to("cuda", tdt)
    out = contract_pair_device(ta, a_dims, tb, b_dims, pairs, out_perm=[2, 0, 1], conj_b=True,
                               batch=B, a_zstride=ta.shape[1], b_zstride=0)
    ref = np.stack([np.transpose(np.tensordot(a[z], np.conj(b), axes=([2, 0], [0, 1])), [2, 0, 1]).reshape(-1)
                    for z in range(B)])
    tol = 1e-5 if dtype == "complex64" else 1e-12
    got = out.cpu().numpy().astype(np.complex128)
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) <= tol
