"""Whole sliced amplitudes of a square-lattice or 53-qubit Sycamore circuit on
the GPU, checked against the dense state vector (oracle) when the lattice has
<= 24 qubits.

    python tools/full_amplitude.py --rows 5 --cols 4 --depth 16 --split 8 --cuts 4-8,11-15 \
        [--nbits 1] [--chunk 512] [--dtype complex64] [--json out.json]
    python tools/full_amplitude.py --net syc53 --depth 12 --split 6 --cap 12 --cuts 9-14,2-8 --chunk 16

All slices of the cut plan are contracted in chunks of ``--chunk`` slices
(accumulated on the device); the JSON is rewritten after every chunk, so an
interrupted run still leaves its partial sums and timing.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def main():
    import torch

    import tn_oracle as O  # checker only
    from paper_2011_02621_b200 import generate_lattice, pattern_rqc, square_patterns, sycamore53_graph
    from paper_2011_02621_b200.network import TwoSidedEngine

    ap = argparse.ArgumentParser()
    ap.add_argument("--net", default="square", choices=["square", "syc53"])
    ap.add_argument("--rows", type=int, default=5)
    ap.add_argument("--cols", type=int, default=4)
    ap.add_argument("--depth", type=int, default=16)
    ap.add_argument("--split", type=int, default=8)
    ap.add_argument("--cap", type=int, default=6)
    ap.add_argument("--cuts", default="")
    ap.add_argument("--nbits", type=int, default=1)
    ap.add_argument("--chunk", type=int, default=512)
    ap.add_argument("--dtype", default="complex64")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--z", type=int, default=0, help="batch elements (bitstring x slice) per device pass (0: auto)")
    ap.add_argument("--json", default=None)
    ap.add_argument("--slice-lo", type=int, default=0, help="first slice of this run (a run cut off by a time "
                    "limit is continued from its JSON's slices_done; the partial sums add)")
    ap.add_argument("--slice-hi", type=int, default=-1)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    if args.net == "syc53":
        graph, pats, _ = sycamore53_graph()
        circ = pattern_rqc(graph, [pats[c] for c in "ABCDCDAB"], args.depth, seed=args.seed)
        n = 53
    else:
        n = args.rows * args.cols
        graph = generate_lattice("square", args.rows, args.cols)
        circ = pattern_rqc(graph, square_patterns(args.rows, args.cols), args.depth, seed=args.seed)
    cuts = [tuple(int(x) for x in c.split("-")) for c in args.cuts.split(",")] if args.cuts else None
    t0 = time.perf_counter()
    eng = TwoSidedEngine(circ, split_cycle=args.split, cuts=cuts, max_rank=args.cap, dtype=args.dtype, device=dev,
                         max_batch_elems=args.z or None)
    rng = np.random.default_rng(1000 + args.depth)
    outs = ["".join(rng.choice(["0", "1"], n)) for _ in range(args.nbits)]
    ex = eng.prepare(outs)
    S = eng.plan.slice_count
    doc = {"args": vars(args), "bitstrings": outs, "slices": S, "multiplies_per_amplitude": eng.plan.multiplies,
           "max_elems": eng.plan.max_elems, "path": list(eng.path), "setup_s": time.perf_counter() - t0,
           "slices_done": 0, "gpu_s": 0.0}
    ref = None
    if n <= 24:
        ref = O.statevector_amplitudes(circ, "0" * n, outs)
        doc["statevector"] = [[float(a.real), float(a.imag)] for a in ref]
    tdt = torch.complex64 if args.dtype == "complex64" else torch.complex128
    amp = torch.zeros(args.nbits, dtype=tdt, device=dev)
    s_hi = S if args.slice_hi < 0 else min(S, args.slice_hi)
    doc["slice_range"] = [args.slice_lo, s_hi]
    for lo in range(args.slice_lo, s_hi, args.chunk):
        hi = min(s_hi, lo + args.chunk)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        eng.run(ex, args.nbits, amp, slices=range(lo, hi), accumulate=True)
        torch.cuda.synchronize()
        doc["gpu_s"] += time.perf_counter() - t1
        doc["slices_done"] = hi
        a = amp.cpu().numpy().astype(np.complex128)
        doc["partial_sum"] = [[float(x.real), float(x.imag)] for x in a]
        doc["est_total_s"] = doc["gpu_s"] * S / (hi - args.slice_lo)
        if args.json:
            with open(args.json, "w") as f:
                json.dump(doc, f, indent=1)
        print(f"slices {hi}/{S}  {doc['gpu_s']:.1f} s  est total {doc['est_total_s']:.0f} s", flush=True)
    got = amp.cpu().numpy().astype(np.complex128)
    doc["amplitude"] = [[float(x.real), float(x.imag)] for x in got]
    doc["amplitudes_per_s"] = args.nbits / doc["gpu_s"] * (s_hi - args.slice_lo) / S
    if ref is not None and args.slice_lo == 0 and s_hi == S:
        doc["rel_l2_vs_statevector"] = float(np.linalg.norm(got - ref) / np.linalg.norm(ref))
        print("rel L2 vs state vector:", doc["rel_l2_vs_statevector"])
    if args.json:
        with open(args.json, "w") as f:
            json.dump(doc, f, indent=1)
    print(json.dumps({k: v for k, v in doc.items() if k not in ("path",)}))


if __name__ == "__main__":
    main()
