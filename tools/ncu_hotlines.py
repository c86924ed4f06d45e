"""Top source lines by warp-stall samples from `ncu --page source --csv --print-source=cuda,sass`."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
fname, hdr, out = None, None, []
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    elif r and r[0] == "Line No":
        hdr = r
    elif hdr and r and r[0] not in ("", "Function Name") and r[2] == "-":
        try:
            out.append((int(r[4]), fname, r[0], r[1][:90]))
        except ValueError:
            pass
tot = sum(o[0] for o in out) or 1
for s, f, ln, src in sorted(out, reverse=True)[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{100*s/tot:5.1f}% {f}:{ln}  {src}")
