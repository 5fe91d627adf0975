"""Multi-rank sharding (CPU, gloo, world size 2): every (bitstring, slice) item
is contracted by exactly one rank and one all-reduce reproduces the
single-process amplitudes (the reference's slice sum)."""

import os
import socket

import numpy as np
import pytest

from paper_2011_02621_b200.distributed import rank_chunks, shard_items


@pytest.mark.parametrize("B,S,W", [(1, 1, 2), (1, 7, 2), (5, 1, 2), (3, 5, 2), (4, 6, 8), (7, 3, 4), (2, 16, 8)])
def test_chunks_partition_items(B, S, W):
    seen = np.zeros((B, S), dtype=int)
    for r in range(W):
        i0, i1 = shard_items(B, S, r, W)
        n = 0
        for ch in rank_chunks(B, S, r, W):
            seen[ch.b0:ch.b0 + ch.nb, ch.s0:ch.s1] += 1
            n += ch.nb * (ch.s1 - ch.s0)
        assert n == i1 - i0
    assert (seen == 1).all()


class _InterpExecutor:
    """Executor stand-in: the numpy descriptor interpreter (test infra)."""

    def __init__(self, plan, sites):
        self.plan = plan
        self.sites = sites

    def run(self, sel, nb, amp, slices=None, b_offset=0, accumulate=True):
        from plan_interp import run_plan

        sub = None if sel is None else {q: v[b_offset:b_offset + nb] for q, v in sel.items()}
        vals = run_plan(self.plan, self.sites, sub, nb, slices)
        import torch

        amp[b_offset:b_offset + nb] += torch.from_numpy(vals)


def _worker(rank, world, port, payload, out_q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2011_02621_b200.distributed import sharded_amplitudes

        plan, sites, sel, B = payload
        ex = _InterpExecutor(plan, sites)
        amp = torch.zeros(B, dtype=torch.complex128)
        sharded_amplitudes(ex, sel, B, amp)
        out_q.put((rank, amp.numpy().copy()))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_gloo_two_ranks_match_single_process(golden_amplitudes):
    import torch.multiprocessing as mp

    from paper_2011_02621_b200 import fuse_single_qubit_gates, parse_circuit
    from paper_2011_02621_b200.engine import ContractionPlan, NetworkSpec
    from paper_2011_02621_b200.tns import evolve, init_state
    from plan_interp import run_plan

    case = golden_amplitudes[0]                      # 3x3, 8 cycles, projected
    c = parse_circuit(case["circuit"])
    fused = fuse_single_qubit_gates(c)
    n = c.num_qubits
    phi = evolve(init_state(c.graph, case["in_bits"]), fused)
    ne = {q: c.graph.node_edges(q) for q in range(n)}
    sites = {}
    for q in range(n):
        a = phi.tensors[q]
        v = np.transpose(a.data, [0] + [a.axis(e) for e in ne[q]])
        if q in fused.trailing:
            v = np.tensordot(fused.trailing[q], v, axes=([1], [0]))
        sites[q] = v
    cuts = [(1, 4), (4, 5)]                           # 2 cut edges -> several slices
    spec = NetworkSpec(list(range(n)), dict(phi.bond_dims), ne)
    from paper_2011_02621_b200.pathfind import NetworkShape, find_optimal_path

    est = dict(phi.bond_dims)
    for e in cuts:
        est[e] = 1
    path, _ = find_optimal_path(NetworkShape(tuple(range(n)), est), 4)
    plan = ContractionPlan(spec, path, cuts)
    assert plan.slice_count > 1
    B = 3
    outs = [r["out"] for r in case["results"]][:B]
    bits = np.array([[int(ch) for ch in b] for b in outs], dtype=np.int32)
    sel = {q: bits[:, q] for q in range(n)}
    full = run_plan(plan, sites, sel, B)
    ref = np.array([complex(*r["statevector"]) for r in case["results"]][:B])
    np.testing.assert_allclose(full, ref, atol=1e-12)

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, (plan, sites, sel, B), q)) for r in range(2)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=180) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(2):
        np.testing.assert_allclose(results[r], full, atol=1e-12)


def test_bench_self_launch_two_ranks():
    """bench.py --gpus 2 outside torchrun re-launches itself with two ranks
    (gloo on CPU in --dry-run): the JSON line reports n_gpus 2 and both ranks'
    slice ranges were summed by the all-reduce."""
    import json
    import subprocess
    import sys

    from conftest import ROOT

    proc = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--dry-run", "--steps", "3"],
                          capture_output=True, text=True, timeout=300, cwd=str(ROOT))
    assert proc.returncode == 0, proc.stderr[-2000:]
    line = json.loads([ln for ln in proc.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["dry_run"]
    assert line["slices_covered"] == 6
    assert line["slice_index_sum"] == sum(range(6))
