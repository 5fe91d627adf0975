"""CPU oracle for the contraction path -- TEST INFRASTRUCTURE ONLY.

Plain-numpy restatement of the reference's amplitude-evaluation path
(``tnsim``, /root/reference/pkg/src/tnsim).  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline / ``--impl
reference`` legs may import this module, and only as the checker or the timed
CPU reference -- the product (``paper_2011_02621_b200``) never calls it.

Pinning: ``tests/test_host_parity.py`` checks every function here against
golden vectors produced by the reference itself (``tests/golden/make_golden.py``
imports /root/reference and runs its own ``compute_amplitude``,
``contract_pair``, ``slice_network``, ``amplitude_oracle``), so the oracle is
parity-pinned, not free-standing.

Each function names the reference lines it restates.
"""

from __future__ import annotations

from math import prod
from typing import Sequence

import numpy as np


# -- tensor.py:100-115 ------------------------------------------------------
def contract_pair(a: np.ndarray, a_labels: Sequence, b: np.ndarray, b_labels: Sequence):
    """Contract every label shared by a and b; result axes = unpaired a axes then
    unpaired b axes (np.tensordot, as reference tensor.py:112)."""
    shared = sorted(set(a_labels) & set(b_labels), key=str)
    ia = [list(a_labels).index(s) for s in shared]
    ib = [list(b_labels).index(s) for s in shared]
    out = np.tensordot(a, b, axes=(ia, ib))
    labels = [x for x in a_labels if x not in shared] + [x for x in b_labels if x not in shared]
    return out, labels


def contraction_cost(dims_a, dims_b, n_shared_extents) -> int:
    """tensor.py:164-184: prod(free a) * prod(free b) * prod(shared)."""
    return int(prod(dims_a) * prod(dims_b) // max(1, n_shared_extents))


# -- network.py:218-243 -----------------------------------------------------
def slice_values(cut_extents: Sequence[int], slice_index: int) -> list[int]:
    """Mixed-radix decoding, first cut edge most significant (network.py:228-232)."""
    vals = [0] * len(cut_extents)
    rem = slice_index
    for i in range(len(cut_extents) - 1, -1, -1):
        vals[i] = rem % cut_extents[i]
        rem //= cut_extents[i]
    return vals


def slice_tensors(tensors: dict, cut_edges: Sequence, cut_extents: Sequence[int], slice_index: int) -> dict:
    """Restrict both endpoints of every cut edge (np.take, network.py:234-241).
    ``tensors``: node -> (array, labels)."""
    out = dict(tensors)
    for e, v in zip(cut_edges, slice_values(cut_extents, slice_index)):
        for q in e:
            arr, labels = out[q]
            ax = list(labels).index(e)
            out[q] = (np.take(arr, v, axis=ax), [x for x in labels if x != e])
    return out


# -- network.py:246-268 -----------------------------------------------------
def contract_along_path(tensors: dict, path: Sequence[int]):
    """Fold tensors in path order; returns (scalar, peak_rank, multiplies)."""
    acc, labels = tensors[path[0]]
    peak = sum(1 for d in acc.shape if d > 1)
    mult = 0
    for q in path[1:]:
        t, tl = tensors[q]
        shared = set(labels) & set(tl)
        k = prod(acc.shape[labels.index(s)] for s in shared) if shared else 1
        mult += prod(acc.shape) * prod(t.shape) // k
        acc, labels = contract_pair(acc, labels, t, tl)
        peak = max(peak, sum(1 for d in acc.shape if d > 1))
    return complex(acc.reshape(())), peak, mult


# -- network.py:334-339 -----------------------------------------------------
def sliced_amplitude(tensors: dict, path, cut_edges=(), cut_extents=()):
    """Sum over all slices of the contracted slice scalars."""
    count = prod(cut_extents) if cut_extents else 1
    total = 0j
    for s in range(count):
        total += contract_along_path(slice_tensors(tensors, cut_edges, cut_extents, s), path)[0]
    return total


# -- network.py:95-126 -----------------------------------------------------
def overlap_tensors(phi: dict, psi: dict, node_edges: dict, bonds_phi: dict, bonds_psi: dict) -> dict:
    """C_q = sum_s A_q[s] conj(B_q[s]); parallel bonds merged phi-major.
    phi/psi: node -> (array with axis 0 physical, labels with 'p' first)."""
    out = {}
    for q, edges in node_edges.items():
        a, la = phi[q]
        b, lb = psi[q]
        t = np.tensordot(a, b.conj(), axes=([0], [0]))
        deg = len(edges)
        perm = []
        for e in edges:
            perm += [la.index(e) - 1, deg + lb.index(e) - 1]
        t = t.transpose(perm).reshape(tuple(bonds_phi[e] * bonds_psi[e] for e in edges))
        out[q] = (t, list(edges))
    return out


def projected_amplitudes(variants: dict, node_edges: dict, path, bits: np.ndarray,
                         cut_edges=(), cut_extents=()) -> np.ndarray:
    """Amplitude per bitstring with product-state bras: C_q = V_q[bit_q]
    (network.py:109-122 with psi = |bits>), then the sliced path contraction.
    ``variants``: node -> array [2, dims in node_edges order]."""
    out = np.empty(bits.shape[0], dtype=np.complex128)
    for i, row in enumerate(bits):
        tensors = {q: (variants[q][int(row[q])], list(node_edges[q])) for q in node_edges}
        out[i] = sliced_amplitude(tensors, path, cut_edges, cut_extents)
    return out


# -- oracle.py:68-96 (brute-force state vector) -----------------------------
def statevector(n: int, in_bits: str, ops) -> np.ndarray:
    """Evolve |in_bits> (qubit 0 = least significant bit) through ``ops``:
    ('1', q, 2x2) or ('2', k, l, 4x4 over (s_k s_l), s_k major)."""
    psi = np.zeros(1 << n, dtype=np.complex128)
    psi[sum(1 << q for q, c in enumerate(in_bits) if c == "1")] = 1.0
    t = psi.reshape((2,) * n)          # axis i <-> qubit n-1-i
    for op in ops:
        if op[0] == "1":
            _, q, u = op
            ax = n - 1 - q
            t = np.moveaxis(np.tensordot(u, t, axes=([1], [ax])), 0, ax)
        else:
            _, k, l, m = op
            ak, al = n - 1 - k, n - 1 - l
            g = np.asarray(m).reshape(2, 2, 2, 2)
            t = np.tensordot(g, t, axes=([2, 3], [ak, al]))
            t = np.moveaxis(t, [0, 1], [ak, al])
    return t.reshape(-1)


def circuit_ops(circuit) -> list:
    """Gate sequence of a circuit object (single-qubit layers per moment,
    cycles, trailing), matching oracle.py:77-89."""
    ops = []
    by_m: dict = {}
    for sg in circuit.single_qubit:
        by_m.setdefault(sg.moment, []).append(sg)
    for m in range(circuit.depth + 1):
        for sg in by_m.get(m, []):
            ops.append(("1", sg.qubit, sg.matrix))
        if m == circuit.depth:
            break
        for g in circuit.cycles[m]:
            ops.append(("2", g.pair[0], g.pair[1], g.matrix))
    for q in sorted(circuit.trailing):
        ops.append(("1", q, circuit.trailing[q]))
    return ops


def statevector_amplitudes(circuit, in_bits: str, out_bits: Sequence[str]) -> np.ndarray:
    n = circuit.num_qubits
    psi = statevector(n, in_bits, circuit_ops(circuit))
    idx = [sum(1 << q for q, c in enumerate(b) if c == "1") for b in out_bits]
    return psi[idx]


# -- pairwise-step sweep (BASELINE configs[1]) --------------------------------
def sweep_step(acc: np.ndarray, acc_perm: Sequence[int], r: int, k: int, site: np.ndarray,
               bits: np.ndarray) -> np.ndarray:
    """One projected Contract step of the sweep: acc[b] has r dim-2 free legs
    and k dim-4 shared legs stored in the axis order ``acc_perm`` (a permutation
    of free legs 0..r-1 then shared r..r+k-1); site[v] is [4]*k + [4]*n.
    Returns out[b] with axes (free legs in stored order, new legs)."""
    B = acc.shape[0]
    out = []
    free_pos = [i for i, a in enumerate(acc_perm) if a < r]
    shared_pos = sorted((i for i, a in enumerate(acc_perm) if a >= r), key=lambda i: acc_perm[i])
    for b in range(B):
        a = acc[b].reshape([2 if x < r else 4 for x in acc_perm])
        s = site[int(bits[b])]
        res = np.tensordot(a, s, axes=(shared_pos, list(range(k))))
        out.append(res.reshape(-1))
    return np.stack(out)


# -- CPU reference timing on the bench's networks ----------------------------
def reference_step_layouts(node_edges: dict, edges: dict, path: Sequence[int], cut_edges=()):
    """Per path step, the operand layouts the reference's contract_along_path
    (network.py:246-266) hands to np.tensordot for one slice: accumulator
    labels in tensordot output order (free a axes, then free b axes,
    tensor.py:100-115), the site's labels in node order, cut edges removed
    (np.take in slice_network).  Returns [(acc_labels, site_labels, shared)]."""
    cut = set(tuple(e) for e in cut_edges)
    lab = {q: [e for e in node_edges[q] if tuple(e) not in cut] for q in node_edges}
    acc = list(lab[path[0]])
    out = []
    for q in path[1:]:
        t = lab[q]
        shared = sorted(set(acc) & set(t))
        out.append((list(acc), list(t), shared))
        acc = [x for x in acc if x not in shared] + [x for x in t if x not in shared]
    return out


def time_sampled_path(layouts, edges: dict, dtype=np.complex64, work_cap: float = 2e8, seed: int = 0):
    """CPU time of one slice contracted the reference's way (np.tensordot on
    the reference layouts), estimated step by step: each step runs on a
    sub-block of its accumulator (outermost free legs fixed until at most
    ``work_cap`` complex multiplies remain -- a row subset of the step's GEMM)
    and its time is scaled by the row ratio.  Returns (seconds per slice,
    seconds measured, multiplies run)."""
    import time

    total = spent = 0.0
    done = 0
    for acc_l, site_l, shared in layouts:
        dims = [int(edges[e]) for e in acc_l]
        tdims = [int(edges[e]) for e in site_l]
        free_idx = [i for i, e in enumerate(acc_l) if e not in shared]
        full_rows = prod(dims[i] for i in free_idx) if free_idx else 1
        kn = prod(tdims) if tdims else 1          # K * N of the step
        rows_cap = max(1, int(work_cap // kn))
        sdims = list(dims)
        rows = full_rows
        for i in free_idx:                       # fix outermost free legs first
            if rows <= rows_cap:
                break
            rows //= sdims[i]
            sdims[i] = 1
            if rows < rows_cap:                  # keep part of this leg
                keep = min(dims[i], max(1, rows_cap // rows))
                sdims[i] = keep
                rows *= keep
        # operand values do not change a dense tensordot's time: cheap fills
        a = np.full(sdims, 0.5 - 0.25j, dtype=dtype)
        b = np.full(tdims, 0.25 + 0.5j, dtype=dtype)
        ia = [acc_l.index(s) for s in shared]
        ib = [site_l.index(s) for s in shared]
        t0 = time.perf_counter()
        np.tensordot(a, b, axes=(ia, ib))
        dt = time.perf_counter() - t0
        spent += dt
        done += rows * kn
        total += dt * full_rows / rows
    return total, spent, done
