"""Aggregate ncu source-page stall samples per CUDA source line:
   ncu -i rep --page source --csv --print-source cuda,sass > mix.csv; python tools/ncu_lines.py mix.csv"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
cur_file = None
acc = []
hdr = None
for r in rows:
    if r and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and r and r[0] and r[0] != "Function Name":
        try:
            samples = int(r[4]) if r[4] not in ("", "-") else 0
            inst = int(r[7]) if len(r) > 7 and r[7] not in ("", "-") else 0
        except ValueError:
            continue
        acc.append((samples, inst, f"{cur_file}:{r[0]}", r[1][:90]))
tot = sum(a[0] for a in acc) or 1
acc.sort(reverse=True)
print(f"total samples {tot}")
for s, i, loc, src in acc[:top]:
    print(f"{100*s/tot:5.1f}%  inst={i:>12d}  {loc:28s} {src}")

if len(sys.argv) > 3 and sys.argv[3] == "inst":
    acc.sort(key=lambda a: -a[1])
    ti = sum(a[1] for a in acc) or 1
    print(f"\nby instructions executed (total {ti})")
    for s, i, loc, src in acc[:top]:
        print(f"{100*i/ti:5.1f}%  samples={100*s/tot:5.1f}%  {loc:28s} {src}")
