"""One-screen summary of an .ncu-rep (per kernel launch): time, DRAM bytes / throughput,
occupancy, issue activity and the top stall reasons.  Usage: ncu_brief.py report.ncu-rep"""
import csv, io, subprocess, sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, units = rows[0], dict(zip(rows[0], rows[1]))
SCALE = {"nsecond": 1.0, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
for r in rows[2:]:
    d = dict(zip(h, r))
    f = lambda k: float(d.get(k, "nan").replace(",", "") or "nan") * SCALE.get(units.get(k, ""), 1.0)
    t = f("gpu__time_duration.sum")   # ns
    rd, wr = f("dram__bytes_read.sum"), f("dram__bytes_write.sum")   # bytes
    name = d.get("Kernel Name", "")[:90]
    print(f"{name}\n  time {t/1e3:.1f} us  dram read {rd/1e6:.2f} MB write {wr/1e6:.2f} MB  -> {(rd+wr)/t:.0f} GB/s"
          f"  regs {d.get('launch__registers_per_thread')}  occ {f('sm__warps_active.avg.pct_of_peak_sustained_active'):.1f}%"
          f"  issue {f('sm__inst_issued.avg.pct_of_peak_sustained_active'):.1f}%  L1 {f('l1tex__throughput.avg.pct_of_peak_sustained_active'):.1f}%"
          f"  grid {d.get('launch__grid_size')} x {d.get('launch__block_size')}")
    st = sorted(((k, f(k)) for k in h if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")),
                key=lambda kv: -kv[1])[:5]
    print("  stalls/issue: " + ", ".join(f"{k[len('smsp__average_warps_issue_stalled_'):-len('_per_issue_active.ratio')]} {v:.2f}" for k, v in st))
