"""Stall breakdown + key pipe metrics of one ncu report: python profiles/ncu_stalls.py <rep>"""
import csv, io, subprocess, sys
raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, vals = rows[0], rows[2]
get = {h: v for h, v in zip(hdr, vals)}
for k in ("gpu__time_duration.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
          "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
          "smsp__issue_active.avg.pct_of_peak_sustained_active"):
    print(f"{k:70s} {get.get(k)}")
st = {}
for h, v in get.items():
    if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
        try:
            st[h[33:]] = float(v.replace(",", ""))
        except ValueError:
            pass
tot = sum(st.values())
for k, v in sorted(st.items(), key=lambda x: -x[1])[:10]:
    print(f"  {k:28s} {100 * v / tot:5.1f} %")
