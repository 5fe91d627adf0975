"""Per-step timing of the projected 53-qubit Sycamore path (complex64).

Usage: python tools/syc_probe.py DEPTH [B] [--json out]
Builds AmplitudeEngine (host: evolution, path search, plan), then times the
whole path per chunk and every tnc_step individually with CUDA events, and
prints per-step M, K, N, layout, us, GB/s, TF/s and the roofline share."""
import ctypes as C
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2011_02621_b200 import AmplitudeEngine, _native as NV, pattern_rqc, sycamore53_graph  # noqa: E402


def main():
    depth = int(sys.argv[1])
    B = int(sys.argv[2]) if len(sys.argv) > 2 and not sys.argv[2].startswith("-") else 4
    out_json = sys.argv[sys.argv.index("--json") + 1] if "--json" in sys.argv else None
    peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))
    hbm = float(peaks.get("hbm_gbs") or peaks.get("hbm_copy_gbs") or 6553)
    tf = float(peaks.get("bf16_tflops") or 1648)
    graph, pats, _ = sycamore53_graph()
    circ = pattern_rqc(graph, [pats[c] for c in "ABCDCDAB"], depth, seed=0)
    t0 = time.perf_counter()
    dtype = "complex128" if "--c128" in sys.argv else "complex64"
    eng = AmplitudeEngine(circ, dtype=dtype, max_rank=12)
    t_setup = time.perf_counter() - t0
    plan, ex = eng.plan, eng.executor
    print(f"depth {depth}: setup {t_setup:.1f}s steps {len(plan.steps)} max_elems 2^{np.log2(plan.max_elems):.1f} "
          f"mult {plan.multiplies:.3e} slices {plan.slice_count} max_z {ex.max_z}", flush=True)
    rng = np.random.default_rng(0)
    bits = rng.integers(0, 2, (B, 53)).astype(np.int32)
    sel = eng.selectors(bits)
    amp = torch.zeros(B, dtype=getattr(torch, dtype), device="cuda")
    for _ in range(2):
        eng.amplitudes_device(sel, B, amp)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 3
    e0.record()
    for _ in range(reps):
        eng.amplitudes_device(sel, B, amp)
    e1.record()
    torch.cuda.synchronize()
    t_amp = e0.elapsed_time(e1) / reps * 1e-3
    print(f"B={B}: {t_amp * 1e3:.2f} ms per batch, {B / t_amp:.2f} amplitudes/s", flush=True)
    if "--only" in sys.argv:               # one step inside an NVTX range (for ncu --nvtx-include probe/)
        i = int(sys.argv[sys.argv.index("--only") + 1])
        L = NV.lib()
        sptr = C.c_void_p(torch.cuda.current_stream().cuda_stream)
        ex.run(sel, ex.chunks(B, range(plan.slice_count))[0][1], amp)
        for k in range(i):
            NV.check(L.tnc_step(C.byref(ex._steps[k]), sptr), "tnc_step")
        torch.cuda.synchronize()
        torch.cuda.nvtx.range_push("probe")
        NV.check(L.tnc_step(C.byref(ex._steps[i]), sptr), "tnc_step")
        torch.cuda.nvtx.range_pop()
        torch.cuda.synchronize()
        sp = plan.steps[i]
        print(f"ran step {i}: M={sp.M} K={sp.K} N={sp.N} contig={int(sp.c_rows_contig)}")
        return
    # per-step timing (one chunk of the batch)
    L = NV.lib()
    st = torch.cuda.current_stream()
    sptr = C.c_void_p(st.cuda_stream)
    b0, nb, s0, ns = ex.chunks(B, range(plan.slice_count))[0]
    z = nb * ns
    ex.run(sel, nb, amp)        # binds descriptors for this chunk
    pd = ex._pd
    traffic = plan.step_traffic(16 if dtype == "complex128" else 8)
    rows = []
    passes = int(sys.argv[sys.argv.index("--passes") + 1]) if "--passes" in sys.argv else 3
    best = [float("inf")] * len(plan.steps)
    for _ in range(passes):                  # per-step minimum over passes (clock noise)
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(len(plan.steps) + 1)]
        evs[0].record()
        for i in range(len(plan.steps)):
            NV.check(L.tnc_step(C.byref(ex._steps[i]), sptr), "tnc_step")
            evs[i + 1].record()
        torch.cuda.synchronize()
        for i in range(len(plan.steps)):
            best[i] = min(best[i], evs[i].elapsed_time(evs[i + 1]) * 1e-3)
    tot_t = tot_roof = 0.0
    for i, sp in enumerate(plan.steps):
        t = best[i]
        by, fl = traffic[i]
        by *= z
        fl *= z
        roof = max(by / (hbm * 1e9), fl / (tf * 1e12))
        tot_t += t
        tot_roof += roof
        rows.append({"i": i, "M": sp.M, "K": sp.K, "N": sp.N, "contig": bool(sp.c_rows_contig), "us": t * 1e6,
                     "GBps": by / t / 1e9, "TFs": fl / t / 1e12, "roof_us": roof * 1e6})
    rows.sort(key=lambda r: -r["us"])
    for r in (rows if "--all" in sys.argv else rows[:25]):
        print(f"step {r['i']:3d} M={r['M']:>10d} K={r['K']:>5d} N={r['N']:>5d} contig={int(r['contig'])} "
              f"{r['us']:10.1f} us {r['GBps']:8.1f} GB/s {r['TFs']:7.2f} TF/s roof {r['roof_us']:9.1f} us")
    print(f"z={z}: sum step time {tot_t * 1e3:.2f} ms, roofline {tot_roof * 1e3:.2f} ms, frac {tot_roof / tot_t:.3f}")
    if out_json:
        json.dump({"depth": depth, "B": B, "z": z, "setup_s": t_setup, "ms_per_batch": t_amp * 1e3,
                   "steps": rows, "sum_ms": tot_t * 1e3, "roof_ms": tot_roof * 1e3}, open(out_json, "w"), indent=1)


if __name__ == "__main__":
    main()
