"""Aggregate ncu source-page warp-stall samples per CUDA source line."""
import csv, subprocess, sys
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
res, fname = [], None
for i, r in enumerate(rows):
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    if r and r[0] == "Line No":
        hdr = r
        ia = hdr.index("Warp Stall Sampling (All Samples)")
        ie = hdr.index("Instructions Executed")
        continue
    if r and len(r) > 5 and r[0].isdigit() and fname:
        try:
            res.append((int(r[ia] or 0), fname, int(r[0]), int(r[ie] or 0), r[1][:100]))
        except (ValueError, IndexError):
            pass
tot = sum(x[0] for x in res)
print("total samples", tot)
for s, f, l, e, src in sorted(res, reverse=True)[:n]:
    print(f"{100.0*s/max(tot,1):5.1f}% {s:6d} {f}:{l:<5d} exec={e:<9d} {src}")
