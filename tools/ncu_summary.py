"""Summarise ncu captures into profiles/ (run here, after gpurun brings the
reports back):  python tools/ncu_summary.py <report.ncu-rep> [...]
and a launch-list CSV:  python tools/ncu_summary.py --launches <csv>"""
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "smsp__inst_executed.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "lts__t_bytes.sum", "launch__shared_mem_per_block_dynamic"]


def summarize(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        item = {"kernel": d.get("Kernel Name", "")[:120]}
        for k in KEYS:
            if k in d:
                item[k] = f"{d[k]} {u.get(k, '')}".strip()
        st = [(k.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(d[k])) for k in hdr
              if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")
              and d[k] not in ("", "n/a")]
        tot = sum(v for _, v in st) or 1.0
        item["top_stalls_pct"] = {k: round(100 * v / tot, 1) for k, v in sorted(st, key=lambda x: -x[1])[:6]}
        res.append(item)
    return res


def launches(path):
    rows = [r for r in csv.reader(open(path)) if r]
    hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hdr_i]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    agg = {}
    for r in rows[hdr_i + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0][:80]
        v = float(r[vi].replace(",", ""))
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(v for _, v in agg.values())
    return {"launches": sum(c for c, _ in agg.values()), "total_time": tot,
            "by_kernel": {k: {"count": c, "time": v, "share": round(v / tot, 4)}
                          for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1])}}


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        print(json.dumps(launches(sys.argv[2]), indent=1))
    else:
        print(json.dumps([summarize(p) for p in sys.argv[1:]], indent=1))
