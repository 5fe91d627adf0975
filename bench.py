#!/usr/bin/env python
"""Benchmark of the contraction hot path (one JSON line on rank 0).

Headline (default, ``--workload d12``): BASELINE.json's metric on its own
config -- amplitudes/s of the 53-qubit Sycamore circuit (configs[4]: 53-qubit
diagonal lattice, couplers ABCDCDAB, fSim(pi/2, pi/6), seeded single-qubit
gates) at **12 cycles**, through the reference's default two-sided network
(split at cycle 6, tns.py:185-212), rank cap 12, sliced over the cut edges
(9,14), (2,8): 256 slices, largest intermediate 2^33 elements (two 64 GiB
ping-pong accumulators in the B200's 180 GB; tools/cut_search.py; path
re-searched on the sliced estimate as network.py:323-330 does), complex64.
configs[4] asks for a 2^30-element cap: the cheapest cut set found for it costs
4.1e17 multiplies per amplitude in 32768 slices against 1.5e16 here (DESIGN.md
section 6), so the cap is sized for this GPU instead; the 2^31 plan of the
earlier rounds ((45,49), (38,45), 1024 slices, 2.0e16) is a nested entry.

One *step* = one device pass over ``--slices-per-step`` slices (default 1) of
one bitstring on every rank; rank r takes slices (i*W + r)*k ... of step i, so
N ranks advance one amplitude N times faster, and the slice sum across ranks is
one NCCL all-reduce per step (the reference's slice loop, network.py:334-339,
distributed).  An amplitude is all S = 256 slices, so value = W * k * steps /
S / t (whole-job amplitudes/s; per-rank work fixed: "weak").  Every slice
has the same shapes and path, so a step is an exact 1/S-of-an-amplitude
unit of work; ``tools/net_probe.py --full`` runs whole amplitudes.

Nested entries (same JSON line, single-GPU runs only): the 2^31 plan and 53q
depth 11 (slices), two-sided 53q depth 10 and depth 8 (whole amplitudes,
bitstring batches), configs[2] (5x4: depth 14 whole amplitudes in complex64 and
complex128 checked against the state vector, depth 16 slices), configs[3] (7x7:
depth 10 whole amplitudes, depth 12 slices), the configs[1] pairwise sweep,
configs[0].

Timing: W untimed warm-up steps, then K steps, each bracketed by CUDA events
on the launching stream; barrier + synchronize around the timed region; max
over ranks.  Inputs are larger than L2 (2^33-element ping-pong accumulators).
``--impl reference`` times the CPU oracle port of the reference path
(np.tensordot on the reference's operand layouts) on the same config.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
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
D12 = {"depth": 12, "split": 6, "cap": 12, "cuts": [(9, 14), (2, 8)], "slices": 256, "elem_log2": 33}
D12_CAP31 = {"depth": 12, "split": 6, "cap": 12, "cuts": [(45, 49), (38, 45)], "slices": 1024, "elem_log2": 31}
# 11 cycles (reference default split 5): one cut edge, 16 slices, 4.45e14 multiplies per amplitude
D11 = {"depth": 11, "split": 5, "cap": 12, "cuts": [(45, 49)], "slices": 16, "elem_log2": 33}
SWEEP_LIMIT = 1 << 32          # elements per operand (complex64: 32 GiB)
SEED = 0
NCU_D12_PROFILE = "profiles/r02f_ncu_d12_pair.json"   # ncu --set full of the top GEMM step (dram bytes)


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), float(d["bf16_tflops"]), float(d.get("bf16_tflops_sustained", 0)), "measured"
    return 6650.0, 1590.0, 0.0, "fallback (B200_PROFILING.md)"


# ---------------------------------------------------------------------------
# process setup: one process per GPU; --gpus N without torchrun re-launches
# ---------------------------------------------------------------------------
def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def self_launch(args) -> bool:
    """``--gpus N`` (N > 1) outside torchrun: re-run this script under
    torch.distributed.run with N ranks on 127.0.0.1; returns True when the
    children ran (the caller exits with their status)."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return False
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")           # NCCL reports the ranks it connected
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), str(Path(__file__).resolve())]
    cmd += sys.argv[1:]
    rc = subprocess.run(cmd, env=env).returncode
    sys.exit(rc)


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus > 1 and world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    import torch

    if args.dry_run:
        dev = torch.device("cpu")
        if world > 1:
            import torch.distributed as dist

            dist.init_process_group("gloo")
        return rank, world, dev
    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    return rank, world, dev


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
# networks
# ---------------------------------------------------------------------------
def syc_circuit(depth, seed=SEED):
    from paper_2011_02621_b200 import pattern_rqc, sycamore53_graph

    graph, pats, _ = sycamore53_graph()
    return pattern_rqc(graph, [pats[c] for c in "ABCDCDAB"], depth, seed=seed)


def random_bits(n, count, seed):
    rng = np.random.default_rng(seed)
    return ["".join(rng.choice(["0", "1"], n)) for _ in range(count)]


def is_gemm_step(sp, z):
    return sp.K % 16 == 0 and sp.K * sp.N >= 256 and z * ((sp.M + 127) // 128) >= 64


def launches_per_pass(plan, z):
    """Kernels of ours per device pass: the first site's projection, per step
    k_bscale + k_bprime + k_tc_gemm (GEMM steps) or one SIMT kernel (+ k_amax
    when an fp16-split GEMM step follows), the slice sum."""
    n = 2
    steps = plan.steps
    for i, sp in enumerate(steps):
        if is_gemm_step(sp, z):
            n += 3
        else:
            n += 1
            if i + 1 < len(steps) and is_gemm_step(steps[i + 1], z):
                n += 1
    return n


def step_times(ex, plan, dev):
    """Re-launch every path step of the executor's last chunk alone between
    CUDA events on the launching stream (descriptors as the last pass left
    them); returns per-step seconds."""
    import ctypes as C

    import torch

    from paper_2011_02621_b200 import _native as NV

    L = NV.lib()
    stream = torch.cuda.current_stream(dev)
    sptr = C.c_void_p(stream.cuda_stream)
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(len(plan.steps) + 1)]
    evs[0].record(stream)
    for i in range(len(plan.steps)):
        NV.check(L.tnc_step(C.byref(ex._steps[i]), sptr), "tnc_step")
        evs[i + 1].record(stream)
    torch.cuda.synchronize(dev)
    return [evs[i].elapsed_time(evs[i + 1]) * 1e-3 for i in range(len(plan.steps))]


def path_roofline(plan, times, z, itemsize, hbm, bf16, bf16_sus):
    """North-star path roofline: sum over steps of max(bytes / HBM, flops /
    bf16 peak) over the sum of measured step times; flops = 8 M K N per
    complex multiply-add (algorithmic).  The dominant kernel (the fp16-split
    tcgen05 GEMM) is reported with its achieved algorithmic TF/s."""
    tot = roof = roof_split = gemm_t = gemm_fl = gemm_by = 0.0
    for sp, t in zip(plan.steps, times):
        by = (sp.M * sp.K + sp.M * sp.N) * itemsize * z
        fl = 8.0 * sp.M * sp.K * sp.N * z
        tot += t
        roof += max(by / (hbm * 1e9), fl / (bf16 * 1e12))
        g = is_gemm_step(sp, z)
        # pipe work of the 3M fp16-split GEMM: 3 real products x 3 split terms
        # = 18 flops per complex multiply-add (2.25x the algorithmic 8)
        roof_split += max(by / (hbm * 1e9), (2.25 * fl if g else fl) / (bf16 * 1e12))
        if g:
            gemm_t += t
            gemm_fl += fl
            gemm_by += by
    ach = gemm_fl / gemm_t / 1e12 if gemm_t else 0.0
    return {
        "bound": "tensor", "achieved": ach, "peak": bf16, "unit": "TFLOP/s", "frac": ach / bf16,
        "kernel": "tnc::k_tc_gemm2 (CTA pairs: tcgen05.mma.cta_group::2 kind::f16, M = 256, fp16-split operands, 3M "
                  "complex products, A operand in TMEM, B' halves by TMA; K < 512 steps: single-CTA k_tc_gemm)",
        "algorithmic": "8*M*K*N flops per GEMM step per slice (complex multiply-add = 8 real flops)",
        "kernel_share_of_step": gemm_t / tot if tot else None,
        "pipe_flops_per_algorithmic_flop": 2.25,
        "frac_pipe": 2.25 * ach / bf16,
        "frac_pipe_sustained_peak": 2.25 * ach / bf16_sus if bf16_sus else None,
        "path_roofline_frac": roof / tot if tot else None,
        "path_roofline": "sum over steps of max(bytes/HBM, 8MKN/bf16 peak) / sum of measured step times",
        "path_roofline_frac_split": roof_split / tot if tot else None,
        "path_roofline_split": "same with the GEMM steps charged their 2.25x pipe flops (fp16-split 3M: the "
                               "complex64 accuracy bound needs 3 fp16 products per real product)",
        "gemm_step_GBps": gemm_by / gemm_t / 1e9 if gemm_t else None,
    }


def ncu_traffic():
    """dram read+write bytes of the committed ncu capture of the top GEMM step
    vs its algorithmic bytes (null when no capture is committed)."""
    try:
        d = json.loads((ROOT / NCU_D12_PROFILE).read_text())
        return d
    except (OSError, ValueError):
        return None


# ---------------------------------------------------------------------------
# headline: 53q depth 12, two-sided, sliced
# ---------------------------------------------------------------------------
def d12_engine(dev, max_batch_elems=1, plan_cfg=None):
    from paper_2011_02621_b200.network import TwoSidedEngine

    pc = plan_cfg or D12
    circ = syc_circuit(pc["depth"])
    return TwoSidedEngine(circ, split_cycle=pc["split"], cuts=pc["cuts"], max_rank=pc["cap"],
                          dtype="complex64", device=dev, max_batch_elems=max_batch_elems), circ


def d12_config(eng=None, k=1, plan_cfg=None):
    pc = plan_cfg or D12
    cuts = ",".join(f"({a},{b})" for a, b in pc["cuts"])
    cfg = {"workload": f"configs[4]: 53-qubit Sycamore (ABCDCDAB, fSim(pi/2, pi/6)), {pc['depth']} cycles, two-sided "
                       f"split {pc['split']}, rank cap 12, sliced over {cuts}; one step = 1 bitstring x {k} slice(s) "
                       "per rank",
           "dtype": "complex64", "depth": pc["depth"], "split_cycle": pc["split"], "max_rank": 12,
           "cut_edges": [list(e) for e in pc["cuts"]], "slices_per_amplitude": pc["slices"],
           "largest_intermediate_log2_elems": pc["elem_log2"],
           "cap_note": "configs[4] names a 2^30-element cap; the cheapest cut set found for it (tools/cut_search.py: "
                       "(9,14),(14,21),(21,26), 32768 slices) costs 4.1e17 multiplies per amplitude, this plan "
                       "1.5e16 (2^33) / 2.0e16 (2^31): the cap is sized for the B200's 180 GB instead",
           "slices_per_step_per_rank": k, "circuit_seed": SEED,
           "l2": f"inputs larger than L2 (2 x 2^{pc['elem_log2']}-element complex64 ping-pong accumulators)"}
    if pc["depth"] != 12:
        cfg.pop("cap_note")
    return cfg


def d12_plan_info(eng):
    return {"multiplies_per_amplitude": eng.plan.multiplies, "max_elems": eng.plan.max_elems,
            "path_steps": len(eng.plan.steps), "path": list(eng.path), "path_score": str(eng.path_score)}


def run_d12(args, rank, world, dev, plan_cfg=None, steps=None, warmup=None, e2e=None):
    import torch

    pc = plan_cfg or D12
    steps = args.steps if steps is None else steps
    warmup = args.warmup if warmup is None else warmup
    e2e = args.e2e if e2e is None else e2e
    hbm, bf16, bf16_sus, peak_src = peaks()
    t0 = time.perf_counter()
    eng, circ = d12_engine(dev, plan_cfg=pc)
    bits = random_bits(53, 1, 100)
    ex = eng.prepare(bits)
    setup_s = time.perf_counter() - t0
    plan = eng.plan
    S = plan.slice_count
    k = args.slices_per_step
    amp = torch.zeros(1, dtype=torch.complex64, device=dev)
    stream = torch.cuda.current_stream(dev)

    def slice_range(i):
        lo = ((i * world + rank) * k) % S
        return range(lo, min(lo + k, S))

    def one_step(i):
        amp.zero_()
        eng.run(ex, 1, amp, slices=slice_range(i))
        if world > 1:
            import torch.distributed as dist

            dist.all_reduce(amp)                   # slice sum across ranks (NCCL)

    for i in range(warmup):
        one_step(i)
    barrier(world)
    torch.cuda.synchronize(dev)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    with ClockSampler(dev.index) as clk:
        for i, (e0, e1) in enumerate(evs):
            e0.record(stream)
            one_step(warmup + i)
            e1.record(stream)
        torch.cuda.synchronize(dev)
    t = sum(e0.elapsed_time(e1) for e0, e1 in evs) * 1e-3
    barrier(world)
    t_max = allreduce_max(t, world, dev)
    value = world * k * steps / S / t_max
    times = step_times(ex, plan, dev)
    roof = path_roofline(plan, times, 1, 8, hbm, bf16, bf16_sus)
    roof["peak_source"] = f"{peak_src} bf16_tflops (MEASURED_PEAKS.json, burst); sustained {bf16_sus}"
    nt = ncu_traffic()
    roof["traffic"] = nt.get("dram_bytes") if nt else None
    if nt:
        roof["traffic_check"] = nt
    top = sorted(zip(plan.steps, times), key=lambda x: -x[1])[:6]
    res = {
        "value": value, "unit": "amplitudes/s", "ms_per_step": 1e3 * t_max / steps, "steps": steps, "warmup": warmup,
        "s_per_amplitude_per_gpu": t_max / steps * S / k,
        "gpu_launches": launches_per_pass(plan, 1) * k * steps,
        "roofline": roof, "config": d12_config(None, k, pc), "plan": d12_plan_info(eng), "clocks": clk.summary(),
        "dtype": "complex64",
        "host_setup_s": setup_s,
        "sharding": ("rank r contracts slices (i*W + r)*k.. of step i; one NCCL all_reduce(sum) per step = the "
                     "slice sum" if world > 1 else "single GPU"),
        "top_steps": [{"M": sp.M, "K": sp.K, "N": sp.N, "ms": 1e3 * tt, "tflops": 8e-12 * sp.M * sp.K * sp.N / tt}
                      for sp, tt in top],
    }
    if e2e:
        # through the public API with host buffers: host bitstring in, bra
        # evolution + overlap sites (H2D), the step's slices, host amplitude out
        # bytes copied per step: the bra site tensors of the bitstring (one pinned buffer) + the bitstring
        h2d = eng._overlap.h2d_bytes_per_bitstring + 53
        es = max(1, min(steps, 3))
        eng._bra_cache = None
        tb0 = time.perf_counter()
        eng.amplitudes(bits, slices=slice_range(0))      # first call of an amplitude: host bra evolution
        torch.cuda.synchronize(dev)
        first_call_s = time.perf_counter() - tb0
        bra_s = eng.last_host_s
        barrier(world)
        t0 = time.perf_counter()
        for i in range(es):
            a = eng.amplitudes(bits, slices=slice_range(i))
            if world > 1:
                import torch.distributed as dist

                ta = torch.from_numpy(a).to(dev)
                dist.all_reduce(ta)
        te = allreduce_max(time.perf_counter() - t0, world, dev)
        # the bra evolution runs once per amplitude (its S / (W k) steps); its share of a step is added back
        per_step = te / es + bra_s * world * k / S
        res["e2e"] = {"value": world * k / S / per_step, "unit": "amplitudes/s", "h2d_bytes_per_step": h2d,
                      "d2h_bytes_per_step": 16, "steps": es, "ms_per_step": 1e3 * te / es,
                      "host_bra_evolution_s_per_amplitude": bra_s, "first_call_s": first_call_s,
                      "path": "TwoSidedEngine.amplitudes([bitstring], slices=...) -> host complex partial amplitude: "
                              "per step the bra site tensors go H2D from a pinned buffer, the overlap sites are built "
                              "on the GPU, the step's slices are contracted, the partial amplitude comes back; the "
                              "host bra evolution runs on the first call of an amplitude and is charged pro rata"}
    res["_engine"] = eng
    return res


def cpu_d12(work_cap=1e9, groups=None, plan_cfg=None):
    """CPU reference of one d12 slice: the reference's np.tensordot steps on
    its own operand layouts (oracle, complex64, all host threads), each path
    step on a row subset of ~work_cap multiplies scaled by the row ratio."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import tn_oracle as O

    from paper_2011_02621_b200.circuit import fuse_single_qubit_gates
    from paper_2011_02621_b200.network import _path_for, _resolve_cuts, _ShapeNet
    from paper_2011_02621_b200.tns import evolve, init_state, psi_batch

    pc = plan_cfg or D12
    circ = syc_circuit(pc["depth"])
    fused = fuse_single_qubit_gates(circ)
    phi = evolve(init_state(fused.graph, "0" * 53), fused, range(0, pc["split"]), "forward")
    psi = psi_batch(fused, ["0" * 53], pc["split"])
    edges = {e: phi.bond_dims[e] * psi.bond_dims[e] for e in fused.graph.edges}
    sn = _ShapeNet(range(53), edges)
    plan = _resolve_cuts(sn, pc["cuts"], pc["cap"])
    path, _ = _path_for(sn, plan, pc["cap"])
    legs = {q: fused.graph.node_edges(q) for q in range(53)}
    lay = O.reference_step_layouts(legs, edges, path, plan.cut_edges)
    return lay, edges, plan.slice_count, O


def _threads():
    try:
        from threadpoolctl import threadpool_info

        return max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:
        return os.cpu_count() or 1


# ---------------------------------------------------------------------------
# nested: two-sided 53q at depth 8 / 10 (whole amplitudes, bitstring batches)
# ---------------------------------------------------------------------------
def run_twosided(args, rank, world, dev, depth, B, steps, warmup):
    import torch

    from paper_2011_02621_b200.network import TwoSidedEngine

    hbm, bf16, bf16_sus, _ = peaks()
    t0 = time.perf_counter()
    circ = syc_circuit(depth)
    eng = TwoSidedEngine(circ, split_cycle=depth // 2, max_rank=12, dtype="complex64", device=dev)
    setup_s = time.perf_counter() - t0
    bits = random_bits(53, B * world, 200 + depth)
    mine = bits[rank * B:(rank + 1) * B]              # weak scaling: B bitstrings per rank
    ex = eng.prepare(mine)
    plan = eng.plan
    amp = torch.zeros(B, dtype=torch.complex64, device=dev)
    stream = torch.cuda.current_stream(dev)
    for _ in range(warmup):
        eng.run(ex, B, amp)
    barrier(world)
    torch.cuda.synchronize(dev)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    with ClockSampler(dev.index) as clk:
        for e0, e1 in evs:
            e0.record(stream)
            eng.run(ex, B, amp)
            e1.record(stream)
        torch.cuda.synchronize(dev)
    t = allreduce_max(sum(a.elapsed_time(b) for a, b in evs) * 1e-3, world, dev)
    z = ex._steps[0].Z
    times = step_times(ex, plan, dev)
    roof = path_roofline(plan, times, z, 8, hbm, bf16, bf16_sus)
    res = {"value": world * B * steps / t, "unit": "amplitudes/s", "ms_per_step": 1e3 * t / steps,
           "scaling": "weak", "steps": steps, "warmup": warmup,
           "gpu_launches": launches_per_pass(plan, z) * len(ex.chunks(B, range(plan.slice_count))) * steps,
           "roofline": roof,
           "config": {"workload": f"configs[4] circuit family: 53-qubit Sycamore, {depth} cycles, two-sided split "
                                  f"{depth // 2} (reference default), rank cap 12, unsliced",
                      "dtype": "complex64", "bitstrings_per_step_per_rank": B,
                      "multiplies_per_amplitude": plan.multiplies, "max_elems": plan.max_elems,
                      "path_steps": len(plan.steps), "host_setup_s": setup_s},
           "clocks": clk.summary(), "dtype": "complex64"}
    if args.e2e:
        eng.amplitudes(mine)
        torch.cuda.synchronize(dev)
        barrier(world)
        es = max(1, min(steps, 3))
        t0 = time.perf_counter()
        host_t = 0.0
        for _ in range(es):
            eng.amplitudes(mine)
            host_t += eng.last_host_s
        te = allreduce_max(time.perf_counter() - t0, world, dev)
        pb = eng.bra_batch(mine[:1])
        per_b = sum(v.nbytes for v in pb.tensors.values())
        res["e2e"] = {"value": world * B * es / te, "unit": "amplitudes/s", "steps": es,
                      "h2d_bytes_per_step": B * (per_b + 53) + sum(v.data.nbytes for v in eng.phi.tensors.values()),
                      "d2h_bytes_per_step": B * 16, "host_bra_evolution_share": host_t / te,
                      "path": "TwoSidedEngine.amplitudes(list of bitstrings) -> host amplitudes (batched host bra "
                              "evolution, overlap sites on the GPU, contraction, D2H)"}
    res["_engine"] = eng
    return res


def cpu_twosided(depth, n, budget_s):
    """The reference CPU path measured on whole amplitudes: two-sided
    evolution (host), overlap network and np.tensordot along the path (oracle,
    complex128 as the reference)."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import tn_oracle as O

    from paper_2011_02621_b200.circuit import fuse_single_qubit_gates
    from paper_2011_02621_b200.network import _path_for, _resolve_cuts, _ShapeNet
    from paper_2011_02621_b200.tns import two_sided_evolve

    circ = syc_circuit(depth)
    bits = random_bits(53, n, 300 + depth)
    done, t0 = 0, time.perf_counter()
    for ob in bits:
        fused = fuse_single_qubit_gates(circ)
        phi, psi = two_sided_evolve(fused, "0" * 53, ob, depth // 2)
        edges = {e: phi.bond_dims[e] * psi.bond_dims[e] for e in fused.graph.edges}
        sn = _ShapeNet(range(53), edges)
        path, _ = _path_for(sn, _resolve_cuts(sn, None, 12), 12)
        ne = {q: fused.graph.node_edges(q) for q in range(53)}
        tens = O.overlap_tensors({q: (phi.tensors[q].data, list(phi.tensors[q].labels)) for q in range(53)},
                                 {q: (psi.tensors[q].data, list(psi.tensors[q].labels)) for q in range(53)},
                                 ne, phi.bond_dims, psi.bond_dims)
        O.sliced_amplitude(tens, path)
        done += 1
        if time.perf_counter() - t0 > budget_s:
            break
    el = time.perf_counter() - t0
    return {"value": done / el, "unit": "amplitudes/s", "cores": _threads(), "kind": "port",
            "sample": f"{done} whole amplitudes (two-sided evolution + overlap + np.tensordot path, complex128 "
                      f"as the reference), {el:.1f} s"}


# ---------------------------------------------------------------------------
# nested: configs[1] pairwise-contraction sweep
# ---------------------------------------------------------------------------
def sweep_cases(limit=SWEEP_LIMIT):
    cases, dropped = [], []
    for r in (16, 20, 24, 28):
        for k in (1, 2, 3):
            for n in (1, 2, 3):
                for B in (1, 16, 256):
                    (cases if B * (2 ** r) * (4 ** max(k, n)) <= limit else dropped).append((r, k, n, B))
    return cases, dropped


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


def run_sweep(args, rank, world, dev, steps, warmup):
    """Every (r, k, n, B) case of configs[1] whose operands fit (<= 2^32
    elements each): projection gather + fused permute/contract per case, each
    case timed with CUDA events after an untimed L2 flush."""
    import torch

    from paper_2011_02621_b200.engine import PairPlan, project_variants

    hbm, bf16, _, peak_src = peaks()
    cases, dropped = sweep_cases(args.limit)
    max_acc = max(B * 2 ** r * 4 ** k for r, k, n, B in cases)
    max_out = max(B * 2 ** r * 4 ** n for r, k, n, B in cases)
    g = torch.Generator(device=dev)
    g.manual_seed(1234 + rank)
    acc = torch.randn(max_acc, dtype=torch.complex64, device=dev, generator=g)
    out = torch.empty(max_out, dtype=torch.complex64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    flush_f = flush.view(torch.float32)
    sink = torch.empty((), dtype=torch.float32, device=dev)
    plans, inputs = [], []
    for ci, (r, k, n, B) in enumerate(cases):
        perm, dims, pairs = case_layout(r, k, n, seed=ci)
        plans.append(PairPlan(dims, [4] * (k + n), pairs, dtype="complex64"))
        variants = torch.randn((2, 4 ** (k + n)), dtype=torch.complex64, device=dev, generator=g)
        bits = torch.randint(0, 2, (B,), dtype=torch.int32, device=dev, generator=g)
        inputs.append((variants, bits, torch.empty((B, 4 ** (k + n)), dtype=torch.complex64, device=dev)))
    stream = torch.cuda.current_stream(dev)

    def one_step():
        per = []
        for ci, (r, k, n, B) in enumerate(cases):
            variants, bits, site = inputs[ci]
            flush.zero_()
            torch.sum(flush_f, dim=0, out=sink)
            e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            e0.record(stream)
            project_variants(variants, bits, site, 4 ** (k + n), stream)
            e1.record(stream)
            plans[ci](acc, site, out, B, 2 ** r * 4 ** k, 4 ** (k + n), 2 ** r * 4 ** n, stream)
            e2.record(stream)
            per.append((e0, e1, e2))
        torch.cuda.synchronize(dev)
        return [(a.elapsed_time(c) * 1e-3, b.elapsed_time(c) * 1e-3) for a, b, c in per]

    for _ in range(warmup):
        one_step()
    barrier(world)
    with ClockSampler(dev.index) as clk:
        rows = [one_step() for _ in range(steps)]
    t_case = allreduce_max(sum(tc for st in rows for tc, _ in st), world, dev)
    per_case_k = [sum(rows[s][ci][1] for s in range(steps)) / steps for ci in range(len(cases))]
    t_kern = sum(per_case_k)
    units = sum(B for *_, B in cases)
    roof_t = sum(max(case_traffic(*c)[0] / (hbm * 1e9), case_traffic(*c)[1] / (bf16 * 1e12)) for c in cases)
    by = sum(case_traffic(*c)[0] for c in cases)
    res = {"value": world * units * steps / t_case, "unit": "bitstring-steps/s", "ms_per_step": 1e3 * t_case / steps,
           "scaling": "weak", "steps": steps, "warmup": warmup, "gpu_launches": 2 * len(cases) * steps,
           "roofline": {"bound": "hbm", "achieved": by / t_kern / 1e9, "peak": hbm, "unit": "GB/s",
                        "frac": roof_t / t_kern, "traffic": None, "peak_source": f"{peak_src} hbm_gbs",
                        "kernel": "all contraction launches (tnc::k_tc_c64, tnc::k_pair_pipe*); projections excluded",
                        "algorithmic": "per case (acc + out + 2*projected site) * 8 B"},
           "config": {"workload": "configs[1] pairwise-contraction sweep", "dtype": "complex64",
                      "cases": len(cases), "operand_limit_elems": args.limit,
                      "excluded_cases_over_limit": [list(c) for c in dropped],
                      "l2": "256 MiB memset + read before every case, untimed"},
           "clocks": clk.summary(), "dtype": "complex64",
           "detail": [{"r": r, "k": k, "n": n, "B": B, "kernel_us": 1e6 * tk,
                       "GBps": case_traffic(r, k, n, B)[0] / tk / 1e9} for (r, k, n, B), tk in zip(cases, per_case_k)]}
    return res


def cpu_sweep(args, detail, budget_s):
    """The oracle's sweep step (np.tensordot per bitstring, as the
    reference's contract_pair) run in full on the smaller sweep cases until
    ``budget_s``; the GPU value on exactly those cases is reported beside."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import tn_oracle as O

    cases, _ = sweep_cases(args.limit)
    order = sorted(range(len(cases)), key=lambda i: case_traffic(*cases[i])[0])
    rng = np.random.default_rng(0)
    done, t_cpu, t0 = [], 0.0, time.perf_counter()
    for ci in order:
        r, k, n, B = cases[ci]
        perm, dims, pairs = case_layout(r, k, n, seed=ci)
        acc = np.full((B, 2 ** r * 4 ** k), 0.5 - 0.25j, dtype=np.complex64)
        site = (rng.standard_normal((2,) + (4,) * (k + n)) + 1j).astype(np.complex64)
        bits = rng.integers(0, 2, B)
        s0 = time.perf_counter()
        O.sweep_step(acc, perm, r, k, site, bits)
        t_cpu += time.perf_counter() - s0
        done.append(ci)
        if time.perf_counter() - t0 > budget_s:
            break
    units = sum(cases[i][3] for i in done)
    t_gpu = sum(detail[i]["kernel_us"] for i in done) * 1e-6
    return {"value": units / t_cpu, "unit": "bitstring-steps/s", "cores": _threads(), "kind": "port",
            "sample": f"oracle sweep_step run in full on the {len(done)} smallest of {len(cases)} cases "
                      f"({t_cpu:.1f} s of CPU); not extrapolated to the other cases",
            "gpu_kernel_value_same_cases": units / t_gpu if t_gpu else None}


# ---------------------------------------------------------------------------
# nested: configs[0]
# ---------------------------------------------------------------------------
def run_cfg0(args, rank, world, dev, steps):
    import torch

    from paper_2011_02621_b200 import AmplitudeEngine, generate_lattice, pattern_rqc, square_patterns

    g = generate_lattice("square", 3, 3)
    circ = pattern_rqc(g, square_patterns(3, 3), 8, seed=0)
    eng = AmplitudeEngine(circ, "0" * 9, dtype="complex128", device=dev)
    B = 64
    rng = np.random.default_rng(rank)
    bits = rng.integers(0, 2, (B, 9)).astype(np.int32)
    sel = eng.selectors(bits)
    amp = torch.zeros(B, dtype=torch.complex128, device=dev)
    stream = torch.cuda.current_stream(dev)
    for _ in range(3):
        eng.amplitudes_device(sel, B, amp, graph=True)
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        eng.amplitudes_device(sel, B, amp, graph=True)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    t = allreduce_max(e0.elapsed_time(e1) * 1e-3, world, dev)
    outs = ["".join(map(str, row)) for row in bits]
    for _ in range(2):
        eng.amplitudes(outs)
    t0 = time.perf_counter()
    for _ in range(steps):
        eng.amplitudes(outs)
    te = allreduce_max(time.perf_counter() - t0, world, dev)
    return {"value": world * B * steps / t, "unit": "amplitudes/s", "ms_per_step": 1e3 * t / steps, "steps": steps,
            "config": {"workload": "configs[0] 3x3 square, 8 cycles, 64 bitstrings, projected engine",
                       "dtype": "complex128"},
            "e2e": {"value": world * B * steps / te, "unit": "amplitudes/s", "h2d_bytes_per_step": B * 9 * 4,
                    "d2h_bytes_per_step": B * 16}}


def cpu_cfg0(budget_s=5.0):
    """configs[0] on the CPU, whole amplitudes: the reference's default
    two-sided compute_amplitude path restated by the oracle (complex128)."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import tn_oracle as O

    from paper_2011_02621_b200 import generate_lattice, pattern_rqc, square_patterns
    from paper_2011_02621_b200.circuit import fuse_single_qubit_gates
    from paper_2011_02621_b200.network import _path_for, _resolve_cuts, _ShapeNet
    from paper_2011_02621_b200.tns import two_sided_evolve

    g = generate_lattice("square", 3, 3)
    circ = pattern_rqc(g, square_patterns(3, 3), 8, seed=0)
    bits = random_bits(9, 64, 1)
    done, t0 = 0, time.perf_counter()
    while time.perf_counter() - t0 < budget_s:
        ob = bits[done % 64]
        fused = fuse_single_qubit_gates(circ)
        phi, psi = two_sided_evolve(fused, "0" * 9, ob, 4)
        edges = {e: phi.bond_dims[e] * psi.bond_dims[e] for e in fused.graph.edges}
        sn = _ShapeNet(range(9), edges)
        plan = _resolve_cuts(sn, "auto", None)
        path, _ = _path_for(sn, plan, None)
        ne = {q: fused.graph.node_edges(q) for q in range(9)}
        tens = O.overlap_tensors({q: (phi.tensors[q].data, list(phi.tensors[q].labels)) for q in range(9)},
                                 {q: (psi.tensors[q].data, list(psi.tensors[q].labels)) for q in range(9)},
                                 ne, phi.bond_dims, psi.bond_dims)
        O.sliced_amplitude(tens, path, plan.cut_edges, plan.extents)
        done += 1
    el = time.perf_counter() - t0
    return {"value": done / el, "unit": "amplitudes/s", "cores": _threads(), "kind": "port",
            "sample": f"{done} whole amplitudes through the reference's default pipeline (two-sided, auto cuts), "
                      f"{el:.1f} s"}


# ---------------------------------------------------------------------------
# square-lattice configs: configs[2] (5x4) and configs[3] (7x7)
# ---------------------------------------------------------------------------
SQUARE = {
    # 5x4, 14 cycles: the deepest configs[2]-family circuit whose two-sided network runs unsliced (2^31 elements)
    "amplitudes_cfg2_d14": dict(rows=5, cols=4, depth=14, split=7, cap=6, cuts=None, B=4, k=0, dtype="complex64",
                                steps=3, warmup=1, verify=True),
    "amplitudes_cfg2_d14_c128": dict(rows=5, cols=4, depth=14, split=7, cap=6, cuts=None, B=1, k=0,
                                     dtype="complex128", steps=2, warmup=1, verify=True),
    # configs[2] as written (16 cycles): 2^36-element intermediates unsliced; cheapest cut set found
    # (tools/cut_search.py) is (4,8),(11,15): 16384 slices of 2^29 elements, 2.27e17 multiplies per amplitude
    "amplitudes_cfg2_d16": dict(rows=5, cols=4, depth=16, split=8, cap=6, cuts=[(4, 8), (11, 15)], B=1, k=8,
                                dtype="complex64", steps=3, warmup=1, verify=False),
    # 7x7, 10 cycles: unsliced two-sided network, 2^33-element intermediates (two 64 GiB accumulators)
    "amplitudes_cfg3_d10": dict(rows=7, cols=7, depth=10, split=5, cap=9, cuts=None, B=1, k=0, dtype="complex64",
                                steps=3, warmup=1, verify=False),
    # configs[3] as written (12 cycles, M = treewidth bound + 1 = 9, 2^30-element cap): 2^20 slices
    "amplitudes_cfg3_d12": dict(rows=7, cols=7, depth=12, split=6, cap=9,
                                cuts=[(20, 27), (19, 26), (18, 25), (17, 24)], B=1, k=64, dtype="complex64",
                                steps=3, warmup=1, verify=False),
}
FP64_TENSOR_TFLOPS = 40.0      # B200 datasheet FP64 (tensor) rate: no measured value in MEASURED_PEAKS.json


def run_square(args, rank, world, dev, name):
    """One entry of SQUARE: whole amplitudes of B bitstrings per step (unsliced
    plans, k = 0) or k slices of one bitstring per step (sliced plans; value =
    k * steps / S / t as in the headline).  ``verify``: amplitudes of the timed
    bitstrings against the dense state vector (oracle, outside the timed region)."""
    import torch

    from paper_2011_02621_b200 import generate_lattice, pattern_rqc, square_patterns
    from paper_2011_02621_b200.network import TwoSidedEngine

    c = SQUARE[name]
    hbm, bf16, bf16_sus, _ = peaks()
    n = c["rows"] * c["cols"]
    graph = generate_lattice("square", c["rows"], c["cols"])
    circ = pattern_rqc(graph, square_patterns(c["rows"], c["cols"]), c["depth"], seed=SEED)
    t0 = time.perf_counter()
    eng = TwoSidedEngine(circ, split_cycle=c["split"], cuts=c["cuts"], max_rank=c["cap"], dtype=c["dtype"], device=dev,
                         max_batch_elems=1 if c["k"] == 0 else None)
    setup_s = time.perf_counter() - t0
    B, k, steps, warmup = c["B"], c["k"], c["steps"], c["warmup"]
    bits = random_bits(n, B * world, 300 + c["depth"])
    mine = bits[rank * B:(rank + 1) * B]
    ex = eng.prepare(mine)
    plan = eng.plan
    S = plan.slice_count
    tdt = torch.complex64 if c["dtype"] == "complex64" else torch.complex128
    amp = torch.zeros(B, dtype=tdt, device=dev)
    stream = torch.cuda.current_stream(dev)

    def one_step(i):
        if k:
            lo = ((i * world + rank) * k) % S
            eng.run(ex, B, amp, slices=range(lo, min(lo + k, S)))
        else:
            eng.run(ex, B, amp)

    for i in range(warmup):
        one_step(i)
    barrier(world)
    torch.cuda.synchronize(dev)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    with ClockSampler(dev.index) as clk:
        for i, (e0, e1) in enumerate(evs):
            e0.record(stream)
            one_step(warmup + i)
            e1.record(stream)
        torch.cuda.synchronize(dev)
    t = allreduce_max(sum(a.elapsed_time(b) for a, b in evs) * 1e-3, world, dev)
    value = world * B * steps / t if not k else world * k * steps / S / t
    z = ex._steps[0].Z
    times = step_times(ex, plan, dev)
    itemsize = 8 if c["dtype"] == "complex64" else 16
    if c["dtype"] == "complex64":
        roof = path_roofline(plan, times, z, itemsize, hbm, bf16, bf16_sus)
    else:
        # complex128: GEMM steps on FP64 DMMA (mma.sync m8n8k4.f64, 4 real products per complex product)
        tot = rf = gt = gf = 0.0
        for sp, tt in zip(plan.steps, times):
            by = (sp.M * sp.K + sp.M * sp.N) * itemsize * z
            fl = 8.0 * sp.M * sp.K * sp.N * z
            tot += tt
            rf += max(by / (hbm * 1e9), fl / (FP64_TENSOR_TFLOPS * 1e12))
            if is_gemm_step(sp, z):
                gt += tt
                gf += fl
        roof = {"bound": "tensor", "achieved": gf / gt / 1e12 if gt else 0.0, "peak": FP64_TENSOR_TFLOPS,
                "unit": "TFLOP/s", "frac": gf / gt / 1e12 / FP64_TENSOR_TFLOPS if gt else None,
                "kernel": "tnc::k_dmma_c128 (mma.sync.m8n8k4.f64 DMMA, complex as 4 real products)",
                "peak_source": "B200 datasheet FP64 tensor rate (no measured FP64 value in MEASURED_PEAKS.json)",
                "kernel_share_of_step": gt / tot if tot else None, "path_roofline_frac": rf / tot if tot else None,
                "traffic": None}
    cuts_txt = ",".join(f"({a},{b})" for a, b in c["cuts"]) if c["cuts"] else "none"
    res = {"value": value, "unit": "amplitudes/s", "ms_per_step": 1e3 * t / steps, "steps": steps, "warmup": warmup,
           "scaling": "weak", "roofline": roof, "clocks": clk.summary(), "dtype": c["dtype"],
           "gpu_launches": launches_per_pass(plan, z) * len(ex.chunks(B, range(S) if not k else range(k))) * steps,
           "config": {"workload": f"{c['rows']}x{c['cols']} square lattice, {c['depth']} cycles (gate set and pattern "
                                  f"rule of configs[0]), two-sided split {c['split']}, rank cap {c['cap']}, cut edges "
                                  f"{cuts_txt}; one step = " +
                                  (f"{B} whole amplitude(s) per rank" if not k else f"{k} of {S} slices of one bitstring"),
                      "dtype": c["dtype"], "slices_per_amplitude": S, "multiplies_per_amplitude": plan.multiplies,
                      "max_elems": plan.max_elems, "path_steps": len(plan.steps), "host_setup_s": setup_s}}
    if k:
        res["s_per_amplitude_per_gpu"] = t / steps * S / k
    if c["verify"] and rank == 0:
        sys.path.insert(0, str(ROOT / "oracle"))
        import tn_oracle as O  # checker only, outside the timed region

        ref = O.statevector_amplitudes(circ, "0" * n, mine)
        got = amp.cpu().numpy().astype(np.complex128)
        res["rel_l2_vs_statevector"] = float(np.linalg.norm(got - ref) / np.linalg.norm(ref))
    if args.e2e and not k:
        eng.amplitudes(mine)
        torch.cuda.synchronize(dev)
        barrier(world)
        es = max(1, min(steps, 2))
        eng._bra_cache = None
        t0 = time.perf_counter()
        for _ in range(es):
            eng._bra_cache = None                      # every step: host bra evolution, H2D, contraction, D2H
            eng.amplitudes(mine)
        te = allreduce_max(time.perf_counter() - t0, world, dev)
        res["e2e"] = {"value": world * B * es / te, "unit": "amplitudes/s", "steps": es,
                      "h2d_bytes_per_step": B * (eng._overlap.h2d_bytes_per_bitstring + n),
                      "d2h_bytes_per_step": B * 16,
                      "path": "TwoSidedEngine.amplitudes(bitstrings) -> host amplitudes (host bra evolution, pinned "
                              "H2D of the bra sites, overlap sites and contraction on the GPU, D2H)"}
    res["_engine"] = eng
    return res


# ---------------------------------------------------------------------------
# reference arm (CPU oracle port, same config as the headline)
# ---------------------------------------------------------------------------
def run_reference(args, base):
    """Each step is a bounded sample of the d12 workload on the host cores:
    the reference's np.tensordot steps of one slice on row subsets (every
    path step once per group rotation: the path's steps are split into
    ``NG`` groups of similar sampled work and step i runs group i mod NG).
    value = amplitudes/s from the mean sampled time per full rotation x S
    slices; ms_per_step is the wall time of the steps actually run."""
    t0 = time.perf_counter()
    lay, edges, S, O = cpu_d12()
    setup = time.perf_counter() - t0
    NG = 4
    work = [min(1e9, prod(int(edges[e]) for e in a if e not in sh) * prod(int(edges[e]) for e in s))
            for a, s, sh in lay]
    target = sum(work) / NG
    groups, cur, acc = [], [], 0.0
    for i, w in enumerate(work):
        cur.append(i)
        acc += w
        if acc >= target and len(groups) < NG - 1:
            groups.append(cur)
            cur, acc = [], 0.0
    if cur:
        groups.append(cur)
    NG = len(groups)
    est = [[] for _ in range(NG)]
    wall = []
    for i in range(args.warmup + args.steps):
        gi = i % NG
        s0 = time.perf_counter()
        tot, _, _ = O.time_sampled_path([lay[j] for j in groups[gi]], edges, work_cap=1e9)
        if i >= args.warmup:
            est[gi].append(tot)
            wall.append(time.perf_counter() - s0)
    full = [np.mean(e) for e in est if e]
    t_slice = sum(full) * NG / len(full)
    v = 1.0 / (t_slice * S)
    cpu = {"value": v, "unit": "amplitudes/s", "cores": _threads(), "kind": "port",
           "sample": f"per step one of {NG} groups of the 52 path steps of one slice, each np.tensordot on the "
                     "reference's operand layout over a row subset of <= 1e9 multiplies, scaled by rows; "
                     f"{S} slices per amplitude; {t_slice:.0f} s per slice", "host_setup_s": setup}
    return dict(base, impl="reference", value=v, unit="amplitudes/s", dtype="complex64",
                ms_per_step=1e3 * float(np.mean(wall)), config=d12_config(None, args.slices_per_step),
                cpu_baseline=cpu, e2e={"value": v, "unit": "amplitudes/s", "h2d_bytes_per_step": 0,
                                       "d2h_bytes_per_step": 0})


# ---------------------------------------------------------------------------
def dry_run(args, rank, world):
    """Plumbing check without a GPU: rank layout, slice ranges, gloo all-reduce
    of partial amplitudes, max-over-ranks timing -- no contraction."""
    import torch

    S, k = D12["slices"], args.slices_per_step
    t0 = time.perf_counter()
    part = torch.zeros(2, dtype=torch.float64)
    for i in range(args.steps):
        lo = ((i * world + rank) * k) % S
        part[0] += float(lo)
        part[1] += 1.0
    if world > 1:
        import torch.distributed as dist

        dist.all_reduce(part)
    t = allreduce_max(time.perf_counter() - t0, world, torch.device("cpu"))
    return {"dry_run": True, "value": None, "unit": "amplitudes/s", "slices_covered": int(part[1].item()),
            "slice_index_sum": int(part[0].item()), "ms_per_step": 1e3 * t / max(1, args.steps),
            "config": d12_config(None, k)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="d12", choices=["d12", "d10", "d8", "sweep", "cfg0", "square"])
    ap.add_argument("--slices-per-step", type=int, default=1)
    ap.add_argument("--limit", type=int, default=SWEEP_LIMIT)
    ap.add_argument("--no-e2e", dest="e2e", action="store_false")
    ap.add_argument("--no-cpu", dest="cpu", action="store_false")
    ap.add_argument("--no-nested", dest="nested", action="store_false")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--dry-run", action="store_true", help="launch/sharding plumbing only (CPU, gloo)")
    args = ap.parse_args()
    self_launch(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    base = {"metric": METRIC, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "data": "synthetic (seeded circuits)"}
    if args.impl == "reference":
        if rank == 0:
            print(json.dumps(run_reference(args, base)))
        return
    rank, world, dev = dist_setup(args)
    if args.dry_run:
        res = dry_run(args, rank, world)
        if rank == 0:
            print(json.dumps(dict(base, **res)))
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()
        return
    import gc

    import torch

    from paper_2011_02621_b200 import _native

    _native.require_device()

    def free(res):
        if isinstance(res, dict):
            res.pop("_engine", None)
        gc.collect()
        torch.cuda.empty_cache()

    cpu_here = rank == 0 and args.cpu and world == 1
    if args.workload == "d12":
        res = run_d12(args, rank, world, dev)
        free(res)
        if cpu_here:
            lay, edges, S, O = cpu_d12()
            tot, spent, _ = O.time_sampled_path(lay, edges, work_cap=1e9)
            res["cpu_baseline"] = {"value": 1.0 / (tot * S), "unit": "amplitudes/s", "cores": _threads(),
                                   "kind": "port",
                                   "sample": "every path step of one slice once: np.tensordot on the reference's "
                                             "operand layout over a row subset of <= 1e9 multiplies, scaled by rows "
                                             f"({spent:.1f} s measured, {tot:.0f} s per slice); x{S} slices"}
        nested = {}
        if args.nested and world == 1:          # N > 1 runs time the headline only (the driver's scaling sweep)
            r1 = run_d12(args, rank, world, dev, plan_cfg=D12_CAP31, steps=5, warmup=3, e2e=False)
            free(r1)
            nested["amplitudes_53q_depth12_cap31"] = r1
            r1 = run_d12(args, rank, world, dev, plan_cfg=D11, steps=5, warmup=3, e2e=False)
            free(r1)
            nested["amplitudes_53q_depth11"] = r1
            for depth, B in ((10, 8), (8, 64)):
                r2 = run_twosided(args, rank, world, dev, depth, B, steps=5, warmup=3)
                free(r2)
                if cpu_here and depth == 8:         # a depth-10 amplitude takes minutes on the host
                    r2["cpu_baseline"] = cpu_twosided(8, 2, 20.0)
                nested[f"amplitudes_53q_depth{depth}_twosided"] = r2
            for name in SQUARE:
                r5 = run_square(args, rank, world, dev, name)
                free(r5)
                nested[name] = r5
            r3 = run_sweep(args, rank, world, dev, steps=3, warmup=2)
            if cpu_here:
                r3["cpu_baseline"] = cpu_sweep(args, r3["detail"], 10.0)
            r3.pop("detail", None)
            free(None)
            nested["sweep_configs1"] = r3
            r4 = run_cfg0(args, rank, world, dev, steps=20)
            if cpu_here:
                r4["cpu_baseline"] = cpu_cfg0(5.0)
            nested["configs0"] = r4
        res.update(nested)
    elif args.workload in ("d10", "d8"):
        depth = int(args.workload[1:])
        res = run_twosided(args, rank, world, dev, depth, 8 if depth == 10 else 64, args.steps, args.warmup)
        free(res)
        if cpu_here and depth == 8:
            res["cpu_baseline"] = cpu_twosided(8, 2, 20.0)
    elif args.workload == "square":
        res = {}
        for name in SQUARE:
            r5 = run_square(args, rank, world, dev, name)
            free(r5)
            res[name] = r5
        first = res["amplitudes_cfg2_d14"]
        res = dict({k: first[k] for k in ("value", "unit", "ms_per_step", "dtype", "config", "roofline", "clocks")}, **res)
    elif args.workload == "sweep":
        res = run_sweep(args, rank, world, dev, args.steps, args.warmup)
        if cpu_here:
            res["cpu_baseline"] = cpu_sweep(args, res["detail"], args.cpu_budget)
        detail = res.pop("detail")
        (ROOT / "gpurun_out").mkdir(exist_ok=True)
        (ROOT / "gpurun_out" / "bench_detail.json").write_text(json.dumps(detail, indent=1))
    else:
        res = run_cfg0(args, rank, world, dev, args.steps)
        if cpu_here:
            res["cpu_baseline"] = cpu_cfg0(5.0)
    if rank == 0:
        print(json.dumps(dict(base, **res), default=str))
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
