#!/usr/bin/env python
"""Summarise ncu captures brought back in gpurun_out/ into committed text + JSON under profiles/.

    python profiles/summarize_ncu.py --workload C2/n1 --tag r01 [--dir gpurun_out]

Reads prof_fwd.ncu-rep / prof_bwd.ncu-rep (`ncu --set full`, one launch each) and launches.csv
(`--metrics gpu__time_duration.sum`, the bench command's launch list). Writes
profiles/ncu_summary.json (DRAM bytes per launch etc., read by bench.py for roofline.traffic) and
profiles/<tag>_ncu_<kernel>.txt / profiles/<tag>_launches.txt.
"""
import argparse
import csv
import json
import os
import subprocess
from collections import defaultdict

HERE = os.path.dirname(os.path.abspath(__file__))
METRICS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pipe_pct",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active": "xu_pipe_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_pipe_pct",
    "launch__registers_per_thread": "registers",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum": "smem_wavefronts",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
         "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
         "second": 1}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u, v = rows[0], rows[1], rows[2]
    res, stalls = {}, {}
    for i, name in enumerate(h):
        if name in METRICS:
            try:
                res[METRICS[name]] = float(v[i].replace(",", "")) * SCALE.get(u[i], 1)
            except ValueError:
                pass
        if name.startswith("smsp__pcsamp_warps_issue_stalled_") and not name.endswith("not_issued"):
            try:
                stalls[name.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(v[i])
            except ValueError:
                pass
    return res, stalls


def launches(path):
    rows = list(csv.reader(l for l in open(path) if not l.startswith("==")))
    h = rows[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    t, n = defaultdict(float), defaultdict(int)
    for r in rows[1:]:
        try:
            t[r[ki]] += float(r[vi].replace(",", ""))
            n[r[ki]] += 1
        except (ValueError, IndexError):
            pass
    return t, n


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dir", default="gpurun_out")
    ap.add_argument("--workload", default="C2/n1")
    ap.add_argument("--tag", default="r01")
    a = ap.parse_args()
    js_path = os.path.join(HERE, "ncu_summary.json")
    js = json.load(open(js_path)) if os.path.exists(js_path) else {}
    entry = js.setdefault(a.workload, {})
    for kind in ("fwd", "bwd"):
        rep = os.path.join(a.dir, f"prof_{kind}.ncu-rep")
        if not os.path.exists(rep):
            continue
        m, stalls = raw(rep)
        tot = sum(stalls.values()) or 1
        top = sorted(stalls.items(), key=lambda x: -x[1])[:8]
        entry[f"attn_{kind}"] = {
            "dram_bytes": m.get("dram_read", 0) + m.get("dram_write", 0),
            "dram_read": m.get("dram_read"), "dram_write": m.get("dram_write"),
            "duration_s": m.get("duration"), "tensor_pipe_pct": m.get("tensor_pipe_pct"),
            "issue_active_pct": m.get("issue_active_pct"), "xu_pipe_pct": m.get("xu_pipe_pct"),
            "registers": m.get("registers"),
            "source": f"ncu --set full --clock-control none, one launch, {a.tag} ({a.workload})",
            "stalls_top": {k: round(100 * v / tot, 1) for k, v in top},
        }
        with open(os.path.join(HERE, f"{a.tag}_ncu_{kind}.txt"), "w") as f:
            f.write(f"# ncu --set full, attn_{kind}_kernel, workload {a.workload} ({a.tag})\n")
            for k, v in sorted(m.items()):
                f.write(f"{k:20s} {v:.6g}\n")
            f.write("warp stall samples (share of all):\n")
            for k, v in top:
                f.write(f"  {k:28s} {100 * v / tot:5.1f} %\n")
    lp = os.path.join(a.dir, "launches.csv")
    if os.path.exists(lp):
        t, n = launches(lp)
        tot = sum(t.values())
        with open(os.path.join(HERE, f"{a.tag}_launches.txt"), "w") as f:
            f.write(f"# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised), "
                    f"bench.py --steps 1 --warmup 1, workload {a.workload}\n")
            for k, v in sorted(t.items(), key=lambda x: -x[1]):
                f.write(f"{v / 1e6:9.3f} ms {100 * v / tot:5.1f} %  x{n[k]:<4d} {k[:110]}\n")
    with open(js_path, "w") as f:
        json.dump(js, f, indent=1, sort_keys=True)
    print(json.dumps(entry, indent=1))


if __name__ == "__main__":
    main()
