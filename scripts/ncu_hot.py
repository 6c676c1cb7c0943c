"""Top source lines of `ncu -i rep --page source --csv --print-source cuda,sass` by stall samples.
usage: python scripts/ncu_hot.py file.csv [top]"""
import csv, sys
top = int(sys.argv[2]) if len(sys.argv) > 2 else 50
f = None
out = []
for r in csv.reader(open(sys.argv[1])):
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name", "Line No") or not r[0].isdigit():
        continue
    try:
        smp = int(r[6]); ins = int(r[7])
    except ValueError:
        continue
    out.append((smp, ins, f, int(r[0]), r[1].strip()[:100]))
ts = sum(o[0] for o in out) or 1
ti = sum(o[1] for o in out) or 1
print("stall samples", ts, "warp instructions", ti)
for o in sorted(out, reverse=True)[:top]:
    print(f"{100*o[0]/ts:5.1f}% {100*o[1]/ti:5.1f}%i {o[2]}:{o[3]} {o[4]}")
