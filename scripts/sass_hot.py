"""Hot SASS instructions of an ncu source page (--print-source sass CSV):
top by executed count and by stall samples, plus stall-reason totals."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
for i, r in enumerate(rows):
    if r and r[0] == "Address":
        h = r; data = [x for x in rows[i + 1:] if x and x[0].startswith("0x") or (x and x[0][:1].isdigit())]
        break
ix = {k: h.index(k) for k in h}
def f(r, k):
    try: return float(r[ix[k]] or 0)
    except ValueError: return 0.0
tot_ex = sum(f(r, "Instructions Executed") for r in data)
tot_st = sum(f(r, "Warp Stall Sampling (All Samples)") for r in data) or 1
print(f"total warp-instructions executed {tot_ex:.3g}; stall samples {tot_st:.0f}")
reasons = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
rs = sorted(((sum(f(r, k) for r in data), k) for k in reasons), reverse=True)
print("stall reasons:", ", ".join(f"{k[6:]} {100*v/tot_st:.1f}%" for v, k in rs[:8]))
print("\n-- by stall samples")
for r in sorted(data, key=lambda r: -f(r, "Warp Stall Sampling (All Samples)"))[:top]:
    best = max(reasons, key=lambda k: f(r, k))
    print(f"{100*f(r,'Warp Stall Sampling (All Samples)')/tot_st:5.1f}% ex={f(r,'Instructions Executed'):9.3g} {r[0]} {r[1][:70]:70s} [{best[6:]}]")
print("\n-- by executed")
for r in sorted(data, key=lambda r: -f(r, "Instructions Executed"))[:top]:
    print(f"ex={f(r,'Instructions Executed'):9.3g} {100*f(r,'Instructions Executed')/tot_ex:5.1f}% {r[0]} {r[1][:80]}")
