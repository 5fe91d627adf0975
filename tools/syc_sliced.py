"""Sliced 53-qubit Sycamore amplitudes (projected engine with cut edges).

Usage: python tools/syc_sliced.py [--check DEPTH] [--time DEPTH] [--reps R]

--check D: amplitudes of 2 bitstrings at depth D unsliced vs sliced with the
           cut set below (slice sum on the device); prints the relative error.
--time D:  one bitstring at depth D, all slices per pass, R timed passes.

Cut set: greedy over edges of bond dim <= 16 minimising the largest
intermediate, then total multiplies (depth 10: (9,14) dim 16 and (2,9) dim 4
-> 64 slices, largest intermediate 2^31 elements, 1.9e14 complex multiplies
per amplitude; unsliced depth 10 needs 2^35-element intermediates)."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2011_02621_b200 import AmplitudeEngine, pattern_rqc, sycamore53_graph  # noqa: E402

CUTS = [(9, 14), (2, 9)]


def engine(depth, cuts):
    graph, pats, _ = sycamore53_graph()
    circ = pattern_rqc(graph, [pats[c] for c in "ABCDCDAB"], depth, seed=0)
    return AmplitudeEngine(circ, dtype="complex64", max_rank=12, cuts=cuts,
                           max_batch_elems=int(os.environ.get("SYC_Z", "1")))


def main():
    args = sys.argv[1:]
    reps = int(args[args.index("--reps") + 1]) if "--reps" in args else 2
    rng = np.random.default_rng(5)
    res = {}
    if "--check" in args:
        d = int(args[args.index("--check") + 1])
        bits = rng.integers(0, 2, (2, 53)).astype(np.int32)
        outs = ["".join(map(str, r)) for r in bits]
        e0 = engine(d, None)
        ref = e0.amplitudes(outs, graph=False)
        del e0
        torch.cuda.empty_cache()
        e1 = engine(d, CUTS)
        got = e1.amplitudes(outs, graph=False)
        err = float(np.linalg.norm(got - ref) / np.linalg.norm(ref))
        res["check"] = {"depth": d, "slices": e1.plan.slice_count, "rel_l2": err,
                        "unsliced": [complex(x) for x in ref], "sliced": [complex(x) for x in got]}
        print(f"depth {d}: unsliced vs {e1.plan.slice_count}-slice rel L2 {err:.2e}", flush=True)
        del e1
        torch.cuda.empty_cache()
    if "--time" in args:
        d = int(args[args.index("--time") + 1])
        t0 = time.perf_counter()
        eng = engine(d, CUTS)
        setup = time.perf_counter() - t0
        plan = eng.plan
        bits = rng.integers(0, 2, (1, 53)).astype(np.int32)
        sel = eng.selectors(bits)
        amp = torch.zeros(1, dtype=torch.complex64, device="cuda")
        eng.amplitudes_device(sel, 1, amp)          # warm-up
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record()
        for _ in range(reps):
            amp.zero_()
            eng.amplitudes_device(sel, 1, amp)
        ev[1].record()
        torch.cuda.synchronize()
        t = ev[0].elapsed_time(ev[1]) * 1e-3 / reps
        res["time"] = {"depth": d, "slices": plan.slice_count, "s_per_amplitude": t, "amplitudes_per_s": 1.0 / t,
                       "multiplies_per_amplitude": plan.multiplies, "max_elems": plan.max_elems,
                       "tflops_complex64_work": 8 * plan.multiplies / t / 1e12, "host_setup_s": setup,
                       "amplitude": complex(amp.cpu().numpy()[0])}
        print(json.dumps(res["time"], default=str), flush=True)
    if "--json" in args:
        json.dump(res, open(args[args.index("--json") + 1], "w"), indent=1, default=str)


if __name__ == "__main__":
    main()
