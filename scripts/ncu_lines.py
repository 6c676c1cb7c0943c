"""Top source lines of an ncu source-page export (--print-source cuda,sass --csv)."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
f = None; hdr = None; out = []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1].split('/')[-1]; continue
    if r[0] == "Line No":
        hdr = r; continue
    if hdr and len(r) > 8 and r[0].isdigit():
        try:
            out.append((int(r[4]) if r[4] != '-' else 0, int(r[7]) if r[7] != '-' else 0, f, int(r[0]), r[1].strip()[:90]))
        except ValueError:
            pass
ts = sum(o[0] for o in out) or 1; ti = sum(o[1] for o in out) or 1
print("stall samples", ts, "warp instructions", ti)
for o in sorted(out, reverse=True)[:top]:
    print(f"{100*o[0]/ts:5.1f}% {100*o[1]/ti:5.1f}%i {o[2]}:{o[3]} {o[4]}")
