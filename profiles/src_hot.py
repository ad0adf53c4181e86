"""Per-source-line hot spots of an ncu report: python profiles/src_hot.py rep.ncu-rep [top]"""
import csv, io, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows, f, hdr = [], None, None
for r in csv.reader(io.StringIO(out)):
    if not r: continue
    if r[0] == "File Path": f = r[1].split("/")[-1]; continue
    if r[0] == "Line No": hdr = r; continue
    if hdr and r[0] not in ("", "Function Name"):
        d = dict(zip(hdr, r))
        try:
            rows.append((int(d["Warp Stall Sampling (All Samples)"]), int(d["Instructions Executed"]), f, r[0], r[1][:90]))
        except (ValueError, KeyError):
            pass
tot = sum(x[0] for x in rows) or 1; toti = sum(x[1] for x in rows) or 1
print(f"total samples {tot}, warp instructions {toti}")
for s, i, f, ln, src in sorted(rows, reverse=True)[:top]:
    print(f"{100*s/tot:5.1f}% smp {100*i/toti:5.1f}% inst  {f}:{ln}  {src}")
