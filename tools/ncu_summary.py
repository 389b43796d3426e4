"""Summarise an ncu --set full report (one kernel launch) as markdown for profiles/.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep "title" > profiles/<name>.md
"""
import csv
import io
import subprocess
import sys

rep, title = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
M = {h: (vals[i], units[i]) for i, h in enumerate(hdr)}
keys = [
    ("Kernel", "Kernel Name"), ("duration", "gpu__time_duration.sum"),
    ("DRAM read", "dram__bytes_read.sum"), ("DRAM write", "dram__bytes_write.sum"),
    ("DRAM throughput % of peak", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
    ("L2 throughput %", "lts__throughput.avg.pct_of_peak_sustained_elapsed"),
    ("L2 hit rate %", "lts__t_sector_hit_rate.pct"), ("L1 hit rate %", "l1tex__t_sector_hit_rate.pct"),
    ("L2 sectors (all)", "lts__t_sectors.sum"), ("L2 atomic sectors", "lts__t_sectors_srcunit_tex_op_atom.sum"),
    ("L2 reduction sectors", "lts__t_sectors_srcunit_tex_op_red.sum"),
    ("warps active % of peak", "sm__warps_active.avg.pct_of_peak_sustained_active"),
    ("issue active %", "smsp__issue_active.avg.pct_of_peak_sustained_active"),
    ("SM throughput %", "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
    ("instructions (warp)", "smsp__inst_executed.sum"), ("registers/thread", "launch__registers_per_thread"),
    ("grid", "launch__grid_size"), ("block", "launch__block_size"),
    ("SM clock", "smsp__cycles_elapsed.avg.per_second"),
]
print(f"# {title}\n")
print(f"Source: `{rep}` (ncu --set full --clock-control none --import-source on; one launch).\n")
print("| metric | value | unit |\n|---|---|---|")
for name, k in keys:
    if k in M:
        v, u = M[k]
        print(f"| {name} | {v} | {u} |")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
srows = list(csv.reader(io.StringIO(src)))
cur, acc, reasons, hdr2 = None, [], {}, None
for r in srows:
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr2 = {h: i for i, h in enumerate(r)}
        continue
    if hdr2 and r and r[0] and r[0] != "Function Name":
        try:
            s = int(r[4]) if r[4] not in ("", "-") else 0
        except ValueError:
            continue
        acc.append((s, f"{cur}:{r[0]}", r[1][:100]))
        for h, i in hdr2.items():
            if h.startswith("stall_") and "Not Issued" not in h and i < len(r) and r[i] not in ("", "-"):
                try:
                    reasons[h] = reasons.get(h, 0) + int(r[i])
                except ValueError:
                    pass
tot = sum(a[0] for a in acc) or 1
# stall reasons from the raw pc-sampling counters (the source page's per-line stall
# columns shift when CUDA and SASS rows are interleaved)
pre = "smsp__pcsamp_warps_issue_stalled_"
raw_st = {k[len(pre):]: float(v[0]) for k, v in M.items()
          if k.startswith(pre) and not k.endswith("_not_issued") and v[0] not in ("", "n/a")}
if raw_st:
    reasons = {"stall_" + k: x for k, x in raw_st.items()}
rt = sum(reasons.values()) or 1
print("\n## Stall reasons (share of warp samples)\n\n| reason | % |\n|---|---|")
for h, v in sorted(reasons.items(), key=lambda x: -x[1])[:8]:
    print(f"| {h} | {100 * v / rt:.1f} |")
print("\n## Top source lines by warp samples\n\n| % | line | source |\n|---|---|---|")
for s, loc, text in sorted(acc, reverse=True)[:15]:
    print(f"| {100 * s / tot:.1f} | {loc} | `{text.strip().replace('|', '/')}` |")
