"""Per-source-line samples of one stall reason from an ncu report (source page).

    python tools/ncu_stall_lines.py rep.ncu-rep [stall_long_sb] [top]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
want = sys.argv[2] if len(sys.argv) > 2 else "stall_long_sb"
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur, hdr, acc = None, None, []
for r in csv.reader(io.StringIO(src)):
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = {h: i for i, h in enumerate(r)}
        continue
    if hdr and r and r[0] and r[0] != "Function Name":
        cols = [i for h, i in hdr.items() if h.startswith(want) and "Not Issued" not in h]
        v = 0
        for i in cols:
            if i < len(r) and r[i] not in ("", "-"):
                try:
                    v += int(r[i])
                except ValueError:
                    pass
        acc.append((v, f"{cur}:{r[0]}", r[1][:100]))
tot = sum(a[0] for a in acc) or 1
print(f"{want}: total {tot}")
for v, loc, text in sorted(acc, reverse=True)[:top]:
    print(f"{100 * v / tot:5.1f}%  {loc:26s} {text.strip()}")
