"""Per-step GPU timing of one amplitude network (two-sided or projected).

    python tools/net_probe.py --net syc53 --depth 12 --split 6 --cuts 45-49,38-45 \
        [--slices 2] [--batch 1] [--dtype complex64] [--full] [--json out.json]

Builds the engine (host: evolution, path search, plan), runs ``--slices``
slices of ``--batch`` bitstrings once untimed, then re-launches every path
step of the last chunk alone between CUDA events and prints (M, K, N, ms,
complex-work TF/s, path roofline share).  ``--full`` additionally times all
slices of one amplitude batch end to end.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def build(args, dev):
    from paper_2011_02621_b200 import (AmplitudeEngine, generate_lattice, pattern_rqc, square_patterns,
                                       sycamore53_graph)
    from paper_2011_02621_b200.network import TwoSidedEngine

    if args.net == "syc53":
        graph, pats, _ = sycamore53_graph()
        circ = pattern_rqc(graph, [pats[c] for c in "ABCDCDAB"], args.depth, seed=args.seed)
    else:
        graph = generate_lattice("square", args.rows, args.cols)
        circ = pattern_rqc(graph, square_patterns(args.rows, args.cols), args.depth, seed=args.seed)
    cuts = None
    if args.cuts:
        cuts = [tuple(int(x) for x in c.split("-")) for c in args.cuts.split(",")]
    if args.split >= args.depth:
        return AmplitudeEngine(circ, dtype=args.dtype, max_rank=args.cap, cuts=cuts, device=dev,
                               max_batch_elems=args.z or None), circ
    return TwoSidedEngine(circ, split_cycle=args.split, dtype=args.dtype, max_rank=args.cap, cuts=cuts,
                          device=dev, max_batch_elems=args.z or None), circ


def main():
    import torch

    from paper_2011_02621_b200 import _native as NV

    ap = argparse.ArgumentParser()
    ap.add_argument("--net", default="syc53", choices=["syc53", "square"])
    ap.add_argument("--rows", type=int, default=5)
    ap.add_argument("--cols", type=int, default=4)
    ap.add_argument("--depth", type=int, default=12)
    ap.add_argument("--split", type=int, default=6)
    ap.add_argument("--cap", type=int, default=12)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--cuts", default="")
    ap.add_argument("--dtype", default="complex64")
    ap.add_argument("--slices", type=int, default=1)
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--z", type=int, default=0, help="max batch elements per device pass (0: auto)")
    ap.add_argument("--full", action="store_true")
    ap.add_argument("--json", default=None)
    ap.add_argument("--ncu-step", type=int, default=-1,
                    help="after the timing, relaunch this step alone between cudaProfilerStart/Stop "
                         "(ncu --profile-from-start off captures just it)")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    t0 = time.perf_counter()
    eng, circ = build(args, dev)
    setup = time.perf_counter() - t0
    plan = eng.plan
    n = circ.num_qubits
    rng = np.random.default_rng(7)
    outs = ["".join(rng.choice(["0", "1"], n)) for _ in range(args.batch)]
    B = args.batch
    S = min(args.slices, plan.slice_count)
    sl = range(0, S)
    if hasattr(eng, "prepare"):
        t1 = time.perf_counter()
        ex = eng.prepare(outs)
        torch.cuda.synchronize()
        prep = time.perf_counter() - t1
        sel = ex._tw_sel
    else:
        ex = eng.executor
        bits = np.array([[int(c) for c in o] for o in outs], dtype=np.int32)
        sel = eng.selectors(bits)
        prep = 0.0
    amp = torch.zeros(B, dtype=ex.tdtype, device=dev)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    ex.run(sel, B, amp, slices=sl)
    torch.cuda.synchronize()
    first = time.perf_counter() - t1
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    amp.zero_()
    ev0.record()
    ex.run(sel, B, amp, slices=sl)
    ev1.record()
    torch.cuda.synchronize()
    t_pass = ev0.elapsed_time(ev1) * 1e-3
    # per-step re-launch (descriptors of the last chunk)
    L = NV.lib()
    stream = torch.cuda.current_stream(dev)
    sptr = C.c_void_p(stream.cuda_stream)
    z = ex._steps[0].Z
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(len(plan.steps) + 1)]
    evs[0].record(stream)
    for i in range(len(plan.steps)):
        NV.check(L.tnc_step(C.byref(ex._steps[i]), sptr), "tnc_step")
        evs[i + 1].record(stream)
    torch.cuda.synchronize()
    if args.ncu_step >= 0:
        torch.cuda.profiler.start()
        NV.check(L.tnc_step(C.byref(ex._steps[args.ncu_step]), sptr), "tnc_step")
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
    peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                        "MEASURED_PEAKS.json")))
    hbm, bf16 = peaks["hbm_gbs"], peaks["bf16_tflops"]
    item = 8 if args.dtype == "complex64" else 16
    rows = []
    tot = roof = 0.0
    for i, sp in enumerate(plan.steps):
        ts = evs[i].elapsed_time(evs[i + 1]) * 1e-3
        fl = 8.0 * sp.M * sp.K * sp.N * z
        by = (sp.M * sp.K + sp.M * sp.N) * item * z
        r = max(by / (hbm * 1e9), fl / (bf16 * 1e12))
        tot += ts
        roof += r
        rows.append({"step": i, "node": sp.node, "M": sp.M, "K": sp.K, "N": sp.N, "ms": ts * 1e3,
                     "tflops": fl / ts / 1e12 if ts else 0, "GBps": by / ts / 1e9 if ts else 0,
                     "roof_frac": r / ts if ts else 0})
    rows_sorted = sorted(rows, key=lambda r: -r["ms"])
    for r in rows_sorted[:20]:
        print("step %2d node %2d M 2^%-4.1f K %6d N %6d  %9.3f ms  %7.1f TF/s  %7.0f GB/s  frac %.2f" % (
            r["step"], r["node"], math.log2(r["M"]), r["K"], r["N"], r["ms"], r["tflops"], r["GBps"], r["roof_frac"]))
    res = {"net": vars(args), "setup_s": setup, "prepare_s": prep, "first_pass_s": first,
           "slices_total": plan.slice_count, "slices_run": S, "batch": B, "z_per_chunk": z,
           "pass_s": t_pass, "multiplies_per_amplitude": plan.multiplies, "max_elems": plan.max_elems,
           "steps_sum_s": tot, "path_roofline_frac": roof / tot if tot else None,
           "tflops_work_pass": 8.0 * plan.multiplies_per_slice * S * B / t_pass / 1e12,
           "est_s_per_amplitude": t_pass / (S * B) * plan.slice_count,
           "amplitude_partial": [complex(x) for x in amp.cpu().numpy()], "steps": rows}
    print(json.dumps({k: v for k, v in res.items() if k not in ("steps", "amplitude_partial")}, default=str))
    if args.full:
        amp.zero_()
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        ex.run(sel, B, amp)
        torch.cuda.synchronize()
        tf = time.perf_counter() - t1
        res["full_s"] = tf
        res["amplitudes"] = [complex(x) for x in amp.cpu().numpy()]
        print(json.dumps({"full_s": tf, "amplitudes_per_s": B / tf, "amplitudes": [str(a) for a in res["amplitudes"]]}))
    if args.json:
        with open(args.json, "w") as f:
            json.dump(res, f, indent=1, default=str)


if __name__ == "__main__":
    main()
