"""Per-source-line warp samples and executed instructions from
`ncu -i X.ncu-rep --page source --csv --print-source cuda,sass`, per kernel."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
kfilter = sys.argv[2] if len(sys.argv) > 2 else ""
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
fpath = fn = None
hdr = None
acc = {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fpath = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        fn = r[1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] == "":
        continue
    if kfilter not in (fn or ""):
        continue
    d = dict(zip(hdr[4:], r[4:]))
    key = (fn[:40], fpath, int(r[0]), r[1][:90])
    a = acc.setdefault(key, [0, 0])
    try:
        a[0] += int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
        a[1] += int(d.get("Instructions Executed", "0") or 0)
    except ValueError:
        pass
tot = sum(v[0] for v in acc.values()) or 1
for k, v in sorted(acc.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{100*v[0]/tot:5.1f}% {v[1]:>10} {k[1]}:{k[2]} {k[3]}")
