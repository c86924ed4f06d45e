"""Top source lines by warp-stall samples from
`ncu -i X --page source --csv --print-source=cuda,sass` (or cuda only).
    python tools/ncu_hotlines.py src.csv [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
fname, hdr, out = None, None, []
for r in rows:
    if r and r[0] in ("File Path", "File Name"):
        fname = r[1].split("/")[-1]
        hdr = None
    elif r and r[0] == "Line No":
        hdr = r
    elif hdr and r and len(r) > 4 and r[0].isdigit():
        try:
            si = hdr.index("Warp Stall Sampling (All Samples)")
            s = int(r[si] or 0)
        except (ValueError, IndexError):
            continue
        if s:
            stalls = {h: r[i] for i, h in enumerate(hdr) if h.startswith("stall_") and
                      "Not Issued" not in h and r[i] not in ("", "0")}
            top = sorted(stalls.items(), key=lambda kv: -float(kv[1]))[:3]
            out.append((s, fname, r[0], r[1][:70], top))
tot = sum(o[0] for o in out) or 1
for s, f, ln, src, top in sorted(out, reverse=True)[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{100*s/tot:5.1f}% {f}:{ln}  {src.strip()}  {' '.join(f'{k[6:]}={v}' for k, v in top)}")
