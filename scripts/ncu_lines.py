"""Aggregate ncu warp-stall samples per CUDA source line (cuda,sass view)."""
import csv, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
hdr = None
agg = []
for r in rows:
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and r and r[0] not in ("",) and r[0].isdigit():
        i = hdr.index("Warp Stall Sampling (All Samples)")
        try:
            agg.append((float(r[i] or 0), int(r[0]), r[1].strip()))
        except ValueError:
            pass
tot = sum(a[0] for a in agg) or 1
for s, ln, src in sorted(agg, reverse=True)[:top]:
    print(f"{100*s/tot:5.1f}%  L{ln:<4} {src[:110]}")
