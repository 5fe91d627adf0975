#!/usr/bin/env python
"""Benchmark of the contraction hot path (one JSON line on rank 0).

Workloads (``--workload``):

* ``sweep`` (default; BASELINE.json configs[1]) -- isolated pairwise
  contraction sweep in complex64: the accumulator C has r free legs of dim 2
  (r = 16..28) and k shared legs of dim 4 (k = 1..3) in a seeded random leg
  order; it is contracted with the bitstring-projected site tensor (k shared +
  n = 1..3 new dim-4 legs) over a bitstring batch B in {1, 16, 256}; cases are
  kept while every operand fits 2^29 elements.  One *step* = one pass over
  all cases; each case = projection gather + fused permute/contract kernel.
  Unit: bitstring-steps/s (one bitstring's accumulator advanced by one
  Contract step).  The 53-qubit / 12-cycle headline network is not runnable by
  this algorithm on any GPU count (peak intermediate 2^41 elements unsliced,
  see DESIGN.md), so the tier rule's "largest single-GPU configuration"
  applies.
* ``cfg0`` (configs[0]) -- full amplitudes: 3x3 lattice, 8 cycles, 64
  bitstrings, complex128, projected engine.  Unit: amplitudes/s.
* ``syc53`` -- full amplitudes of the configs[4] circuit family (53-qubit
  Sycamore lattice, ABCDCDAB, fSim(pi/2, pi/6)) at the deepest depth whose
  unsliced projected network fits one B200 (8 cycles: 6.4e11 complex
  multiplies and 2^29-element intermediates per amplitude), complex64,
  bitstring batches of the executor's chunk size.  Unit: amplitudes/s.

Timing: W warm-up steps, then K steps; every case (a timed iteration) is
bracketed by CUDA events on the launching stream and preceded by an untimed
L2 flush (256 MiB memset, then a 256 MiB read so the flush's dirty lines are
written back before the timed kernel), so no case reads L2-resident data; barrier +
synchronize around the timed region; max over ranks.  ``--impl reference``
times the CPU oracle port of the reference algorithm (numpy tensordot, as
tnsim.tensor.contract_pair) on a bounded sample and scales to the same unit.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from math import prod
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "amplitudes/sec (53q, depth 12) at 1/2/4/8 GPUs; contraction % of roofline"
SWEEP_LIMIT = 1 << 29          # elements per operand (complex64: 4 GiB)


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), float(d["bf16_tflops"]), "measured"
    return 6650.0, 1590.0, "fallback"


def sweep_cases(limit=SWEEP_LIMIT):
    cases = []
    for r in (16, 20, 24, 28):
        for k in (1, 2, 3):
            for n in (1, 2, 3):
                for B in (1, 16, 256):
                    if B * (2 ** r) * (4 ** max(k, n)) <= limit:
                        cases.append((r, k, n, B))
    return cases


def case_layout(r, k, n, seed):
    rng = np.random.default_rng(seed)
    perm = [int(x) for x in rng.permutation(r + k)]
    dims = [2 if x < r else 4 for x in perm]
    shared_pos = sorted((i for i, x in enumerate(perm) if x >= r), key=lambda i: perm[i])
    pairs = [(p, j) for j, p in enumerate(shared_pos)]
    return perm, dims, pairs


def case_traffic(r, k, n, B, itemsize=8):
    acc = B * 2 ** r * 4 ** k
    out = B * 2 ** r * 4 ** n
    site = B * 4 ** (k + n)
    return (acc + out + 2 * site) * itemsize, 8 * B * 2 ** r * 4 ** k * 4 ** n


# ---------------------------------------------------------------------------
# clocks sampled during the timed region
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t0 = time.time()
            while not self.lines and time.time() - t0 < 5.0 and self.proc.poll() is None:
                time.sleep(0.02)
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(nm)
        loaded = [x for x in sm if x > 0.5 * mx] if mx else sm
        med = float(np.median(loaded)) if loaded else None
        out = {"sm_mhz": med, "sm_max_mhz": mx or None, "reasons": sorted(reasons), "samples": len(sm)}
        if not sm and self.lines:
            out["raw"] = self.lines[:2]
        return out


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def run_sweep(args, rank, world, dev):
    import torch

    from paper_2011_02621_b200.engine import PairPlan, project_variants

    hbm, bf16, peak_src = peaks()
    cases = sweep_cases(args.limit)
    torch.manual_seed(1234 + rank)
    max_acc = max(B * 2 ** r * 4 ** k for r, k, n, B in cases)
    max_out = max(B * 2 ** r * 4 ** n for r, k, n, B in cases)
    acc = torch.randn(max_acc, dtype=torch.complex64, device=dev)
    out = torch.empty(max_out, dtype=torch.complex64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    flush_f = flush.view(torch.float32)
    flush_sink = torch.empty((), dtype=torch.float32, device=dev)
    l2_mode = os.environ.get("BENCH_L2_FLUSH", "write+read")
    plans, inputs = [], []
    gen = torch.Generator(device=dev)
    gen.manual_seed(99 + rank)
    for ci, (r, k, n, B) in enumerate(cases):
        perm, dims, pairs = case_layout(r, k, n, seed=ci)
        plan = PairPlan(dims, [4] * (k + n), pairs, dtype="complex64")
        variants = torch.randn((2, 4 ** (k + n)), dtype=torch.complex64, device=dev, generator=gen)
        bits = torch.randint(0, 2, (B,), dtype=torch.int32, device=dev, generator=gen)
        site = torch.empty((B, 4 ** (k + n)), dtype=torch.complex64, device=dev)
        plans.append(plan)
        inputs.append((variants, bits, site))
    stream = torch.cuda.current_stream(dev)

    def one_step(record):
        tot_case, tot_kern = 0.0, 0.0
        per = []
        for ci, (r, k, n, B) in enumerate(cases):
            variants, bits, site = inputs[ci]
            KN = 4 ** (k + n)
            # untimed L2 flush: write a buffer larger than L2, then read it back,
            # so the flush's own dirty lines are written back before the timed
            # kernel instead of during it
            flush.zero_()
            if l2_mode == "write+read":
                torch.sum(flush_f, dim=0, out=flush_sink)
            e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            e0.record(stream)
            project_variants(variants, bits, site, KN, stream)
            e1.record(stream)
            plans[ci](acc, site, out, B, 2 ** r * 4 ** k, KN, 2 ** r * 4 ** n, stream)
            e2.record(stream)
            per.append((e0, e1, e2))
        torch.cuda.synchronize(dev)
        rows = []
        for (r, k, n, B), (e0, e1, e2) in zip(cases, per):
            tc = e0.elapsed_time(e2) * 1e-3
            tk = e1.elapsed_time(e2) * 1e-3
            tot_case += tc
            tot_kern += tk
            rows.append((r, k, n, B, tc, tk))
        return tot_case, tot_kern, rows

    for _ in range(args.warmup):
        one_step(False)
    barrier(world)
    torch.cuda.synchronize(dev)
    with ClockSampler(dev.index) as clk:
        t_case = t_kern = 0.0
        acc_rows = {}
        for _ in range(args.steps):
            tc, tk, rows = one_step(True)
            t_case += tc
            t_kern += tk
            for r, k, n, B, a, b in rows:
                acc_rows.setdefault((r, k, n, B), [0.0, 0.0])
                acc_rows[(r, k, n, B)][0] += a
                acc_rows[(r, k, n, B)][1] += b
    torch.cuda.synchronize(dev)
    barrier(world)
    t_case_max = allreduce_max(t_case, world, dev)
    units_per_step = sum(B for _, _, _, B in cases)
    value = world * units_per_step * args.steps / t_case_max
    # roofline of the dominant kernel (the fused permute+contract launch)
    bytes_tot = sum(case_traffic(*c)[0] for c in cases) * args.steps
    flops_tot = sum(case_traffic(*c)[1] for c in cases) * args.steps
    roof_t = sum(max(case_traffic(*c)[0] / (hbm * 1e9), case_traffic(*c)[1] / (bf16 * 1e12)) for c in cases) * args.steps
    achieved = bytes_tot / t_kern / 1e9
    detail = []
    for c, (a, b) in acc_rows.items():
        by, fl = case_traffic(*c)
        detail.append({"r": c[0], "k": c[1], "n": c[2], "B": c[3], "kernel_us": 1e6 * b / args.steps,
                       "GBps": by / (b / args.steps) / 1e9, "TFLOPs": fl / (b / args.steps) / 1e12})
    res = {
        "value": value, "unit": "bitstring-steps/s", "ms_per_step": 1e3 * t_case_max / args.steps,
        "gpu_launches": 2 * len(cases) * args.steps,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                     "frac": (roof_t / t_kern), "traffic": None,
                     "peak_source": f"{peak_src} hbm_gbs / bf16_tflops (MEASURED_PEAKS.json)",
                     "kernel": "all contraction launches of the sweep: tnc::k_tc_c64 (tcgen05 3xTF32, K >= 8, K*N >= 256) "
                               "and tnc::k_pair_pipe* (TMA-fed fused permute+contract SIMT); projections excluded",
                     "algorithmic": "per case (acc + out + 2*projected site) * 8 B; flops 8*B*2^r*4^k*4^n",
                     "kernel_share_of_step": t_kern / t_case, "tflops_achieved": flops_tot / t_kern / 1e12,
                     "traffic_ncu": ncu_traffic_check()},
        "config": {"workload": "configs[1] pairwise-contraction sweep", "dtype": "complex64",
                   "cases": len(cases), "r": [16, 20, 24, 28], "k": [1, 2, 3], "n": [1, 2, 3],
                   "batch": [1, 16, 256], "operand_limit_elems": args.limit,
                   "leg_order": "seeded random permutation per case",
                   "l2": ("256 MiB memset + 256 MiB read (write-back of the flush drained) before every case, untimed"
                          if l2_mode == "write+read" else "256 MiB memset flush before every case (untimed)")},
        "clocks": clk.summary(),
        "dtype": "complex64",
        "detail": detail,
    }
    if args.e2e:
        res["e2e"] = sweep_e2e(args, cases, plans, inputs, dev, world)
    return res


def sweep_e2e(args, cases, plans, inputs, dev, world):
    """Same sweep through the public API with host buffers: per case the
    accumulator and projection bits go H2D from pinned memory, gather +
    contract run, the result comes back D2H; all inside the timed region.
    The cases are pipelined over three streams (H2D copies, compute, D2H
    copies) with BENCH_E2E_SLOTS (6) device slots per buffer, so later cases'
    uploads and earlier cases' downloads overlap case i's kernels (PCIe is
    full duplex)."""
    import torch

    from paper_2011_02621_b200.engine import project_variants

    max_acc = max(B * 2 ** r * 4 ** k for r, k, n, B in cases)
    max_out = max(B * 2 ** r * 4 ** n for r, k, n, B in cases)
    h_acc = torch.randn(max_acc, dtype=torch.complex64).pin_memory()
    ns = int(os.environ.get("BENCH_E2E_SLOTS", "6"))
    h_out = [torch.empty(max_out, dtype=torch.complex64).pin_memory() for _ in range(ns)]
    d_acc = [torch.empty(max_acc, dtype=torch.complex64, device=dev) for _ in range(ns)]
    d_out = [torch.empty(max_out, dtype=torch.complex64, device=dev) for _ in range(ns)]
    h_bits = [inputs[i][1].cpu().pin_memory() for i in range(len(cases))]
    stream = torch.cuda.current_stream(dev)
    s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    h2d = d2h = 0
    for r, k, n, B in cases:
        h2d += B * 2 ** r * 4 ** k * 8 + B * 4
        d2h += B * 2 ** r * 4 ** n * 8

    def step():
        nc = len(cases)
        ev_in = [torch.cuda.Event() for _ in range(nc)]
        ev_comp = [torch.cuda.Event() for _ in range(nc)]
        ev_out = [torch.cuda.Event() for _ in range(nc)]
        s_in.wait_stream(stream)
        for ci, (r, k, n, B) in enumerate(cases):
            variants, bits, site = inputs[ci]
            na, no = B * 2 ** r * 4 ** k, B * 2 ** r * 4 ** n
            slot = ci % ns
            with torch.cuda.stream(s_in):
                if ci >= ns:
                    s_in.wait_event(ev_comp[ci - ns])       # slot's accumulator consumed
                d_acc[slot][:na].copy_(h_acc[:na], non_blocking=True)
                bits.copy_(h_bits[ci], non_blocking=True)
                ev_in[ci].record(s_in)
            stream.wait_event(ev_in[ci])
            if ci >= ns:
                stream.wait_event(ev_out[ci - ns])          # slot's result downloaded
            project_variants(variants, bits, site, 4 ** (k + n), stream)
            plans[ci](d_acc[slot], site, d_out[slot], B, 2 ** r * 4 ** k, 4 ** (k + n), 2 ** r * 4 ** n, stream)
            ev_comp[ci].record(stream)
            with torch.cuda.stream(s_out):
                s_out.wait_event(ev_comp[ci])
                h_out[slot][:no].copy_(d_out[slot][:no], non_blocking=True)
                ev_out[ci].record(s_out)
        stream.wait_stream(s_out)
        stream.wait_stream(s_in)
        torch.cuda.synchronize(dev)

    step()
    barrier(world)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    steps = max(1, min(args.steps, 3))
    e0.record(stream)
    for _ in range(steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize(dev)
    t = allreduce_max(e0.elapsed_time(e1) * 1e-3, world, dev)
    units = sum(B for *_, B in cases) * steps * world
    return {"value": units / t, "unit": "bitstring-steps/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "steps": steps, "path": "PairPlan + project_variants on host-resident pinned buffers, H2D / compute / "
                                    "D2H on three streams, %d device slots" % ns}


SYC_DEPTH = 8
SYC_MAX_RANK = 12


def syc_engine(dev, depth=SYC_DEPTH):
    from paper_2011_02621_b200 import AmplitudeEngine, pattern_rqc, sycamore53_graph

    graph, pats, _ = sycamore53_graph()
    circ = pattern_rqc(graph, [pats[c] for c in "ABCDCDAB"], depth, seed=0)
    return AmplitudeEngine(circ, dtype="complex64", max_rank=SYC_MAX_RANK, device=dev)


def run_syc53(args, rank, world, dev, depth=SYC_DEPTH):
    """Amplitudes of the 53-qubit Sycamore circuit (projected engine): each
    step evaluates one batch of B bitstrings per GPU (B = the executor's chunk,
    all resident in HBM).  With N ranks the step is one global batch of N*B
    bitstrings through ``distributed.sharded_amplitudes``: every rank contracts
    its shard, one NCCL all-reduce sums and gathers the amplitudes (weak
    scaling: B per rank)."""
    import ctypes as C

    import torch

    from paper_2011_02621_b200 import _native as NV

    hbm, bf16, peak_src = peaks()
    t0 = time.perf_counter()
    eng = syc_engine(dev, depth)
    setup_s = time.perf_counter() - t0
    ex, plan = eng.executor, eng.plan
    B = ex.max_z
    from paper_2011_02621_b200.distributed import sharded_amplitudes

    Bg = B * world                              # the global batch (same bitstrings on every rank)
    rng = np.random.default_rng(100)
    gbits = rng.integers(0, 2, (Bg, 53)).astype(np.int32)
    gsel = eng.selectors(gbits)
    gamp = torch.zeros(Bg, dtype=torch.complex64, device=dev)

    def one_pass():
        if world > 1:
            sharded_amplitudes(ex, gsel, Bg, gamp)
        else:
            eng.amplitudes_device(gsel, B, gamp)

    bits = gbits[rank * B:(rank + 1) * B]
    sel = eng.selectors(bits)
    amp = torch.zeros(B, dtype=torch.complex64, device=dev)
    stream = torch.cuda.current_stream(dev)
    for _ in range(args.warmup):
        one_pass()
    barrier(world)
    torch.cuda.synchronize(dev)
    # each step's working set (2 x B x 4 GiB ping-pong buffers) is far larger than L2
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with ClockSampler(dev.index) as clk:
        for e0, e1 in evs:
            e0.record(stream)
            one_pass()
            e1.record(stream)
        torch.cuda.synchronize(dev)
    t = sum(e0.elapsed_time(e1) for e0, e1 in evs) * 1e-3
    barrier(world)
    t_max = allreduce_max(t, world, dev)
    value = world * B * args.steps / t_max
    # per-step kernel times (untimed pass, one chunk): dominant kernel + path roofline
    L = NV.lib()
    sptr = C.c_void_p(stream.cuda_stream)
    ex.run(sel, B, amp)
    traffic = plan.step_traffic(8)
    sev = [torch.cuda.Event(enable_timing=True) for _ in range(len(plan.steps) + 1)]
    sev[0].record(stream)
    for i in range(len(plan.steps)):
        NV.check(L.tnc_step(C.byref(ex._steps[i]), sptr), "tnc_step")
        sev[i + 1].record(stream)
    torch.cuda.synchronize(dev)
    tot_t = tot_roof = tot_roof3 = gemm_t = gemm_fl = 0.0
    for i, sp in enumerate(plan.steps):
        ts = sev[i].elapsed_time(sev[i + 1]) * 1e-3
        by, fl = traffic[i][0] * B, traffic[i][1] * B
        tot_t += ts
        tot_roof += max(by / (hbm * 1e9), fl / (bf16 * 1e12))
        # the fp16-split GEMM issues 3 products per real product: its own tensor ceiling is bf16/3
        split = sp.K * sp.N >= 256 and sp.K % 16 == 0
        tot_roof3 += max(by / (hbm * 1e9), (3 * fl if split else fl) / (bf16 * 1e12))
        if sp.K * sp.N >= 256 and sp.K % 8 == 0:      # tensor-core steps
            gemm_t += ts
            gemm_fl += fl
    achieved = gemm_fl / gemm_t / 1e12 if gemm_t else 0.0
    launches = ex.launches_per_chunk() + sum(1 for sp in plan.steps if sp.K * sp.N >= 256 and sp.K % 8 == 0)
    res = {
        "value": value, "unit": "amplitudes/s", "ms_per_step": 1e3 * t_max / args.steps,
        "gpu_launches": launches * args.steps,
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": bf16, "unit": "TFLOP/s",
                     "frac": achieved / bf16, "traffic": None,
                     "peak_source": f"{peak_src} bf16_tflops (MEASURED_PEAKS.json); the kernel issues fp16 MMAs "
                                    "(3 split products per real product, so 3x the algorithmic flops on the pipe)",
                     "kernel": "tnc::k_tc_gemm<16,F16> (tcgen05 kind::f16 fp16-split complex GEMM steps)",
                     "algorithmic": "8*M*K*N flops per step per bitstring",
                     "kernel_share_of_step": gemm_t / tot_t if tot_t else None,
                     "path_roofline_frac": tot_roof / tot_t if tot_t else None,
                     "path_roofline": "sum over steps of max(bytes/HBM, flops/bf16 peak) / sum of step times",
                     "path_roofline_frac_split": tot_roof3 / tot_t if tot_t else None,
                     "path_roofline_split": "same with 3x flops on the fp16-split GEMM steps (the complex64 "
                                            "accuracy bound needs 3 fp16 products per real product)"},
        "config": {"workload": "configs[4] circuit family: 53-qubit Sycamore, ABCDCDAB, "
                               f"{depth} cycles (unsliced projected network on one GPU)",
                   "dtype": "complex64", "bitstrings_per_step": B, "max_rank": SYC_MAX_RANK,
                   "sharding": ("one global batch of N*B bitstrings: per-rank shard (distributed.rank_chunks) + "
                                "one NCCL all_reduce(sum) of the amplitude vector, timed" if world > 1
                                else "single GPU"),
                   "multiplies_per_amplitude": plan.multiplies, "max_elems": plan.max_elems,
                   "path_steps": len(plan.steps), "host_setup_s": setup_s,
                   "l2": "inputs larger than L2 (2 x B x 4 GiB ping-pong buffers)"},
        "clocks": clk.summary(), "dtype": "complex64",
    }
    if args.e2e:
        outs = ["".join(map(str, row)) for row in bits]
        for _ in range(2):                       # first call eager, second captures the path's CUDA graph
            eng.amplitudes(outs)
        torch.cuda.synchronize(dev)
        barrier(world)
        steps = max(1, min(args.steps, 3))
        t0 = time.perf_counter()
        for _ in range(steps):
            eng.amplitudes(outs)
        te = allreduce_max(time.perf_counter() - t0, world, dev)
        res["e2e"] = {"value": world * B * steps / te, "unit": "amplitudes/s", "h2d_bytes_per_step": B * 53 * 4,
                      "d2h_bytes_per_step": B * 8, "steps": steps,
                      "path": "AmplitudeEngine.amplitudes(list of bitstring strings) -> host complex array"}
    res["_plan_steps"] = [(sp.M, sp.K, sp.N) for sp in plan.steps]
    return res


SYC_SLICED_DEPTH = SYC_DEPTH + 2
# cut edges for the sliced depth-10 network (tools/syc_sliced.py: greedy over
# bond dims <= 16, minimising the largest intermediate, then the multiplies)
SYC_SLICED_CUTS = [(9, 14), (2, 9)]


# ncu --set full captures committed under profiles/ (one launch each) and the
# sweep case each was taken on: DRAM bytes per launch vs the algorithmic bytes
NCU_TRAFFIC_PROFILE = "profiles/r01h_ncu_full_summary.json"
NCU_TRAFFIC_CASES = [(16, 2, 2, 256), (24, 1, 2, 1)]


def _ncu_bytes(v: str) -> float:
    num, unit = v.split()
    return float(num) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[unit]


def ncu_traffic_check():
    """Per captured launch: dram read+write bytes (ncu) vs algorithmic bytes."""
    try:
        caps = json.loads((ROOT / NCU_TRAFFIC_PROFILE).read_text())
    except (OSError, ValueError):
        return None
    out = []
    for cap, case in zip(caps, NCU_TRAFFIC_CASES):
        k = cap[0]
        dram = _ncu_bytes(k["dram__bytes_read.sum"]) + _ncu_bytes(k["dram__bytes_write.sum"])
        alg = case_traffic(*case)[0]
        out.append({"kernel": k["kernel"].split("(")[0], "case": "r%d/k%d/n%d/B%d" % case, "dram_bytes": dram,
                    "algorithmic_bytes": alg, "ratio": dram / alg, "source": NCU_TRAFFIC_PROFILE})
    return out


def run_syc53_sliced(args, rank, world, dev, depth=SYC_SLICED_DEPTH):
    """One amplitude of the 53-qubit Sycamore circuit at ``depth`` cycles
    through the reference's slicing scheme (network.py:385-455: cut edges fixed
    per slice, slices summed): unsliced, the network needs 2^35-element
    intermediates; with the two cut edges it runs as 64 slices of at most 2^31
    elements, one slice per device pass, summed on the device.  With N ranks
    the 64 slices are split over the ranks (distributed.sharded_amplitudes)
    and one NCCL all-reduce sums them (strong scaling: one amplitude)."""
    import torch

    from paper_2011_02621_b200 import AmplitudeEngine, pattern_rqc, sycamore53_graph
    from paper_2011_02621_b200.distributed import sharded_amplitudes

    t0 = time.perf_counter()
    graph, pats, _ = sycamore53_graph()
    circ = pattern_rqc(graph, [pats[c] for c in "ABCDCDAB"], depth, seed=0)
    eng = AmplitudeEngine(circ, dtype="complex64", max_rank=SYC_MAX_RANK, cuts=SYC_SLICED_CUTS,
                          max_batch_elems=1, device=dev)
    setup_s = time.perf_counter() - t0
    ex, plan = eng.executor, eng.plan
    rng = np.random.default_rng(100)
    bits = rng.integers(0, 2, (1, 53)).astype(np.int32)
    sel = eng.selectors(bits)
    amp = torch.zeros(1, dtype=torch.complex64, device=dev)

    def one_pass():
        amp.zero_()
        if world > 1:
            sharded_amplitudes(ex, sel, 1, amp)
        else:
            eng.amplitudes_device(sel, 1, amp)

    stream = torch.cuda.current_stream(dev)
    for _ in range(args.warmup):
        one_pass()
    barrier(world)
    torch.cuda.synchronize(dev)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with ClockSampler(dev.index) as clk:
        for e0, e1 in evs:
            e0.record(stream)
            one_pass()
            e1.record(stream)
        torch.cuda.synchronize(dev)
    t = sum(e0.elapsed_time(e1) for e0, e1 in evs) * 1e-3
    barrier(world)
    t_max = allreduce_max(t, world, dev)
    res = {
        "value": args.steps / t_max, "unit": "amplitudes/s", "ms_per_step": 1e3 * t_max / args.steps,
        "scaling": "strong", "tflops_complex64_work": 8 * plan.multiplies * args.steps / t_max / 1e12,
        "config": {"workload": f"configs[4] circuit family: 53-qubit Sycamore, ABCDCDAB, {depth} cycles, "
                               f"sliced over cut edges {SYC_SLICED_CUTS} ({plan.slice_count} slices)",
                   "dtype": "complex64", "bitstrings_per_step": 1, "slices": plan.slice_count,
                   "multiplies_per_amplitude": plan.multiplies, "max_elems": plan.max_elems,
                   "path_steps": len(plan.steps), "host_setup_s": setup_s,
                   "sharding": ("slices split over ranks + one NCCL all_reduce(sum)" if world > 1
                                else "single GPU, one slice per device pass, device slice sum"),
                   "l2": "inputs larger than L2 (2 x 16 GiB ping-pong buffers)"},
        "clocks": clk.summary(), "dtype": "complex64", "steps": args.steps, "warmup": args.warmup,
    }
    if args.e2e and world == 1:
        outs = ["".join(map(str, row)) for row in bits]
        t0 = time.perf_counter()
        eng.amplitudes(outs, graph=False)
        te = time.perf_counter() - t0
        res["e2e"] = {"value": 1.0 / te, "unit": "amplitudes/s", "h2d_bytes_per_step": 53 * 4,
                      "d2h_bytes_per_step": 8, "steps": 1,
                      "path": "AmplitudeEngine.amplitudes(list of bitstring strings, graph=False) -> host complex array"}
    res["_plan_steps"] = [(sp.M, sp.K, sp.N) for sp in plan.steps]
    res["_slices"] = plan.slice_count
    return res


def syc_plan_shapes_host(depth=SYC_DEPTH):
    """(M, K, N) of every path step, computed on the host only (circuit, TNS
    evolution, path search, plan) -- for the CPU reference arm."""
    from paper_2011_02621_b200 import pattern_rqc, sycamore53_graph
    from paper_2011_02621_b200 import network as NW
    from paper_2011_02621_b200.circuit import fuse_single_qubit_gates
    from paper_2011_02621_b200.engine import ContractionPlan, NetworkSpec
    from paper_2011_02621_b200.tns import evolve, init_state

    graph, pats, _ = sycamore53_graph()
    circ = pattern_rqc(graph, [pats[c] for c in "ABCDCDAB"], depth, seed=0)
    fused = fuse_single_qubit_gates(circ)
    phi = evolve(init_state(fused.graph, "0" * 53), fused, range(fused.depth), "forward", 1e-12)
    edges = {e: phi.bond_dims[e] for e in fused.graph.edges}
    path, _ = NW._path_for(NW._ShapeNet(range(53), edges), NW.CutPlan((), ()), SYC_MAX_RANK)
    legs = {q: fused.graph.node_edges(q) for q in range(53)}
    plan = ContractionPlan(NetworkSpec(list(range(53)), edges, legs), path)
    return [(sp.M, sp.K, sp.N) for sp in plan.steps]


def cpu_syc_rate(step_shapes, budget_s: float = 20.0):
    """CPU time per amplitude for the syc53 path, estimated from the oracle's
    contraction primitive (numpy tensordot, as tnsim.tensor.contract_pair) on
    row samples of every distinct step shape (M_s = min(M, 2^14) rows of
    [M, K] x [K, N], complex64), scaled by M / M_s."""
    rng = np.random.default_rng(0)
    shapes = sorted(set((K, N) for _, K, N in step_shapes), key=lambda x: -x[0] * x[1])
    per_row = {}
    t_start = time.perf_counter()
    for K, N in shapes:
        ms = 1 << 14
        a = (rng.standard_normal((ms, K)) + 1j * rng.standard_normal((ms, K))).astype(np.complex64)
        b = (rng.standard_normal((K, N)) + 1j * rng.standard_normal((K, N))).astype(np.complex64)
        reps, t0 = 0, time.perf_counter()
        while True:
            np.tensordot(a, b, axes=([1], [0]))
            reps += 1
            if time.perf_counter() - t0 > min(1.0, budget_s / len(shapes)) or reps >= 20:
                break
        per_row[(K, N)] = (time.perf_counter() - t0) / reps / ms
        if time.perf_counter() - t_start > budget_s:
            break
    worst = max(per_row.values())
    t_amp = sum(M * per_row.get((K, N), worst) for M, K, N in step_shapes)
    return 1.0 / t_amp, time.perf_counter() - t_start


def run_cfg0(args, rank, world, dev):
    import torch

    from paper_2011_02621_b200 import AmplitudeEngine, generate_lattice, pattern_rqc, square_patterns

    g = generate_lattice("square", 3, 3)
    circ = pattern_rqc(g, square_patterns(3, 3), 8, seed=0)
    eng = AmplitudeEngine(circ, "0" * 9, dtype="complex128", device=dev)
    rng = np.random.default_rng(rank)
    B = 64
    bits = rng.integers(0, 2, (B, 9)).astype(np.int32)
    sel = eng.selectors(bits)
    amp = torch.zeros(B, dtype=torch.complex128, device=dev)
    stream = torch.cuda.current_stream(dev)
    for _ in range(args.warmup):
        eng.amplitudes_device(sel, B, amp, graph=True)
    barrier(world)
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev.index) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            eng.amplitudes_device(sel, B, amp, graph=True)
        e1.record(stream)
        torch.cuda.synchronize(dev)
    t = allreduce_max(e0.elapsed_time(e1) * 1e-3, world, dev)
    # e2e: host bitstrings in, host amplitudes out, through the public API
    outs = ["".join(map(str, row)) for row in bits]
    for _ in range(2):                           # eager, then graph capture (untimed)
        eng.amplitudes(outs)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        eng.amplitudes(outs)
    te = allreduce_max(time.perf_counter() - t0, world, dev)
    hbm, _, src = peaks()
    return {"value": world * B * args.steps / t, "unit": "amplitudes/s", "ms_per_step": 1e3 * t / args.steps,
            "gpu_launches": eng.executor.launches_per_chunk() * args.steps,
            "roofline": {"bound": "latency", "achieved": None, "peak": hbm, "unit": "GB/s", "frac": None,
                         "traffic": None, "note": "9-qubit network: launch-bound; every pass replays one "
                                                  "CUDA graph of the whole path (projection, steps, slice sum)"},
            "config": {"workload": "configs[0] 3x3 square, 8 cycles, 64 bitstrings", "dtype": "complex128",
                       "l2": "inputs L2-resident (tiny network)"},
            "clocks": clk.summary(), "dtype": "complex128",
            "e2e": {"value": world * B * args.steps / te, "unit": "amplitudes/s", "h2d_bytes_per_step": B * 9 * 4,
                    "d2h_bytes_per_step": B * 16}}


# ---------------------------------------------------------------------------
# CPU reference arm (oracle port of tnsim's numpy tensordot path)
# ---------------------------------------------------------------------------
def cpu_sweep_rates(budget_s: float = 20.0):
    """Per-(k, n) CPU throughput (bytes/s of algorithmic traffic) of the
    oracle port, measured on r = 16..20, B = 1 cases within ``budget_s``."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import tn_oracle as O

    try:
        from threadpoolctl import threadpool_info

        threads = max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:
        threads = os.cpu_count() or 1
    rng = np.random.default_rng(0)
    rates = {}
    t_start = time.perf_counter()
    per_class = budget_s / 9
    for k in (1, 2, 3):
        for n in (1, 2, 3):
            r = 18
            perm, dims, pairs = case_layout(r, k, n, seed=k * 10 + n)
            acc = (rng.standard_normal((1, 2 ** r * 4 ** k)) + 1j * rng.standard_normal((1, 2 ** r * 4 ** k))).astype(np.complex64)
            site = (rng.standard_normal((2,) + (4,) * (k + n)) + 1j * rng.standard_normal((2,) + (4,) * (k + n))).astype(np.complex64)
            bits = np.zeros(1, dtype=np.int64)
            reps, t0 = 0, time.perf_counter()
            while True:
                O.sweep_step(acc, perm, r, k, site, bits)
                reps += 1
                el = time.perf_counter() - t0
                if el > per_class or reps >= 50:
                    break
            by, _ = case_traffic(r, k, n, 1)
            rates[(k, n)] = by * reps / el
    return rates, threads, time.perf_counter() - t_start


def _cpu_threads():
    try:
        from threadpoolctl import threadpool_info

        return max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:
        return os.cpu_count() or 1


def cpu_value_for(cases, rates):
    t = sum(case_traffic(*c)[0] / rates[(c[1], c[2])] for c in cases)
    return sum(c[3] for c in cases) / t


def run_reference(args):
    rates, threads, spent = cpu_sweep_rates(args.cpu_budget)
    cases = sweep_cases(args.limit)
    v = cpu_value_for(cases, rates)
    return v, threads, spent


# ---------------------------------------------------------------------------
def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def allreduce_max(x, world, dev):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="sweep", choices=["sweep", "cfg0", "syc53"])
    ap.add_argument("--limit", type=int, default=SWEEP_LIMIT)
    ap.add_argument("--no-e2e", dest="e2e", action="store_false")
    ap.add_argument("--no-cpu", dest="cpu", action="store_false")
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--no-syc", dest="syc", action="store_false",
                    help="sweep workload: skip the nested 53-qubit amplitude measurement")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    base = {"metric": METRIC, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "data": "synthetic (seeded)"}

    if args.impl == "reference" and args.workload == "syc53":
        if rank != 0:
            return
        shapes = syc_plan_shapes_host()
        v, spent = cpu_syc_rate(shapes, args.cpu_budget)
        line = dict(base, impl="reference", value=v, unit="amplitudes/s", n_gpus=world, dtype="complex64",
                    ms_per_step=1e3 / v,
                    config={"workload": "configs[4] circuit family: 53-qubit Sycamore, ABCDCDAB, "
                                        f"{SYC_DEPTH} cycles", "dtype": "complex64"},
                    cpu_baseline={"value": v, "unit": "amplitudes/s", "cores": _cpu_threads(), "kind": "port",
                                  "sample": f"numpy tensordot on 2^14-row samples of every distinct step shape, "
                                            f"{spent:.1f}s; scaled by rows"},
                    e2e={"value": v, "unit": "amplitudes/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0})
        print(json.dumps(line))
        return
    if args.impl == "reference":
        if rank != 0:
            return
        v, threads, spent = run_reference(args)
        line = dict(base, impl="reference", value=v, unit="bitstring-steps/s", n_gpus=world, dtype="complex64",
                    ms_per_step=1e3 * sum(c[3] for c in sweep_cases(args.limit)) / v,
                    config={"workload": "configs[1] pairwise-contraction sweep", "dtype": "complex64"},
                    cpu_baseline={"value": v, "unit": "bitstring-steps/s", "cores": threads, "kind": "port",
                                  "sample": f"oracle sweep_step (numpy tensordot) at r=18, B=1 for every (k,n); "
                                            f"{spent:.1f}s of CPU; scaled per case by algorithmic bytes"},
                    e2e={"value": v, "unit": "bitstring-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0})
        print(json.dumps(line))
        return

    import torch

    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    from paper_2011_02621_b200 import _native

    _native.require_device()
    runner = {"sweep": run_sweep, "cfg0": run_cfg0, "syc53": run_syc53}[args.workload]
    res = runner(args, rank, world, dev)
    plan_steps = res.pop("_plan_steps", None)
    syc = syc9 = syc10 = None
    if args.workload == "sweep" and args.syc:
        # the headline circuit family, measured beside the sweep: amplitudes/s of
        # the 53-qubit Sycamore network at the deepest depth one GPU holds
        sargs = argparse.Namespace(**vars(args))
        sargs.steps, sargs.warmup = max(3, min(args.steps, 5)), max(3, args.warmup)
        syc = run_syc53(sargs, rank, world, dev)
        syc_steps = syc.pop("_plan_steps", None)
        if rank == 0 and args.cpu and world == 1 and syc_steps:
            cv, spent = cpu_syc_rate(syc_steps, min(args.cpu_budget, 10.0))
            syc["cpu_baseline"] = {"value": cv, "unit": "amplitudes/s", "cores": _cpu_threads(), "kind": "port",
                                   "sample": f"numpy tensordot on 2^14-row samples of every distinct step shape, "
                                             f"{spent:.1f}s; scaled by rows (permutation cost not included)"}
        syc["steps"], syc["warmup"] = sargs.steps, sargs.warmup
        # one cycle deeper: 6.7e12 multiplies and 2^31-element intermediates per
        # amplitude (one amplitude per device pass), tensor-bound GEMM steps
        import gc

        gc.collect()
        torch.cuda.empty_cache()                 # the depth-8 engine's buffers go back first
        sargs9 = argparse.Namespace(**vars(sargs))
        sargs9.steps = 3
        syc9 = run_syc53(sargs9, rank, world, dev, depth=SYC_DEPTH + 1)
        syc9_steps = syc9.pop("_plan_steps", None)
        if rank == 0 and args.cpu and world == 1 and syc9_steps:
            cv, spent = cpu_syc_rate(syc9_steps, min(args.cpu_budget, 10.0))
            syc9["cpu_baseline"] = {"value": cv, "unit": "amplitudes/s", "cores": _cpu_threads(), "kind": "port",
                                    "sample": f"numpy tensordot on 2^14-row samples of every distinct step shape, "
                                              f"{spent:.1f}s; scaled by rows (permutation cost not included)"}
        syc9["steps"], syc9["warmup"] = sargs9.steps, sargs9.warmup
        # two cycles deeper, sliced (64 slices, 1.9e14 multiplies per amplitude)
        gc.collect()
        torch.cuda.empty_cache()
        sargs10 = argparse.Namespace(**vars(sargs))
        sargs10.steps, sargs10.warmup = 2, 1
        syc10 = run_syc53_sliced(sargs10, rank, world, dev)
        s10_steps, s10_slices = syc10.pop("_plan_steps", None), syc10.pop("_slices", 1)
        if rank == 0 and args.cpu and world == 1 and s10_steps:
            cv, spent = cpu_syc_rate(s10_steps, min(args.cpu_budget, 8.0))
            syc10["cpu_baseline"] = {"value": cv / s10_slices, "unit": "amplitudes/s", "cores": _cpu_threads(),
                                     "kind": "port",
                                     "sample": f"numpy tensordot on 2^14-row samples of every distinct step shape, "
                                               f"{spent:.1f}s; scaled by rows and by the {s10_slices} slices"}
    if rank == 0:
        if args.cpu and world == 1:
            if args.workload == "sweep":
                rates, threads, spent = cpu_sweep_rates(args.cpu_budget)
                cv = cpu_value_for(sweep_cases(args.limit), rates)
                res["cpu_baseline"] = {"value": cv, "unit": "bitstring-steps/s", "cores": threads, "kind": "port",
                                       "sample": f"oracle sweep_step (numpy) r=18, B=1 per (k,n), {spent:.1f}s; "
                                                 "scaled per case by algorithmic bytes"}
            elif args.workload == "syc53" and plan_steps:
                cv, spent = cpu_syc_rate(plan_steps, args.cpu_budget)
                res["cpu_baseline"] = {"value": cv, "unit": "amplitudes/s", "cores": _cpu_threads(), "kind": "port",
                                       "sample": f"numpy tensordot (the oracle/reference contraction primitive) on "
                                                 f"2^14-row samples of every distinct step shape, {spent:.1f}s; "
                                                 "scaled by rows (permutation cost not included: favours the CPU)"}
        detail = res.pop("detail", None)
        line = dict(base, **res)
        if syc is not None:
            line["amplitudes_53q"] = syc
            line["amplitudes_53q_depth9"] = syc9
            line["amplitudes_53q_depth10_sliced"] = syc10
        print(json.dumps(line))
        if detail is not None:
            (ROOT / "gpurun_out").mkdir(exist_ok=True)
            (ROOT / "gpurun_out" / "bench_detail.json").write_text(json.dumps(detail, indent=1))
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
