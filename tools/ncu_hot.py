"""Top stall lines of an ncu source-page CSV (SASS view).  Usage: ncu_hot.py report.ncu-rep [n]"""
import csv, io, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
i0 = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[i0]
R = [dict(zip(h, r)) for r in rows[i0 + 1:] if len(r) == len(h)]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
tot = sum(int(r["# Samples"]) for r in R)
texec = sum(int(r["Instructions Executed"]) for r in R)
wf = sum(int(r["L1 Wavefronts Shared"]) for r in R)
wfi = sum(int(r["L1 Wavefronts Shared Ideal"]) for r in R)
print(f"samples {tot}  warp-instructions {texec}  shared wavefronts {wf} (ideal {wfi})")
keys = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
agg = {k: sum(int(r[k]) for r in R) for k in keys}
print("stall totals:", ", ".join(f"{k[6:]} {v}" for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:8]))
for idx, r in sorted(enumerate(R), key=lambda ir: -int(ir[1]["# Samples"]))[:n]:
    top = sorted(((k[6:], int(r[k])) for k in keys), key=lambda kv: -kv[1])[:2]
    print(f"{idx:5d} {int(r['# Samples']):6d} {100*int(r['# Samples'])/tot:5.1f}%  exec {int(r['Instructions Executed']):8d}  wf {int(r['L1 Wavefronts Shared']):8d}  {r['Source'].strip()[:70]:70s} {top}")
