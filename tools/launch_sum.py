"""Summarise an ncu --csv launch list (gpu__time_duration.sum): per-kernel totals, and
the launches of one BiCGStab iteration (between consecutive k_dev_p launches)."""
import csv, re, sys, collections
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]; data = rows[1:]
ik, iv, iid = h.index("Kernel Name"), h.index("Metric Value"), h.index("ID")
seq = []
for r in data:
    if r[h.index("Metric Name")] != "gpu__time_duration.sum":
        continue
    name = re.sub(r"\(.*", "", r[ik]).replace("void ", "")
    name = re.sub(r"hc::|\(int\)|\(bool\)", "", name)
    seq.append((name, float(r[iv].replace(",", ""))))
tot = collections.defaultdict(lambda: [0, 0.0])
for n, t in seq:
    tot[n][0] += 1; tot[n][1] += t
T = sum(t for _, t in seq)
print(f"total {T/1e6:.2f} ms over {len(seq)} launches")
for n, (c, t) in sorted(tot.items(), key=lambda x: -x[1][1])[:30]:
    print(f"{100*t/T:6.2f}% {t/1e6:9.3f} ms {c:6d} x {t/c/1e3:8.2f} us  {n}")
# one iteration: from the last-but-one k_dev_p to the last one
idx = [i for i, (n, _) in enumerate(seq) if n.endswith("k_dev_p")]
if len(idx) >= 3:
    a, b = idx[-3], idx[-2]
    it = seq[a:b]
    print(f"\none BiCGStab iteration: {len(it)} launches, {sum(t for _, t in it)/1e3:.1f} us of kernel time")
    per = collections.defaultdict(lambda: [0, 0.0])
    for n, t in it:
        per[n][0] += 1; per[n][1] += t
    for n, (c, t) in sorted(per.items(), key=lambda x: -x[1][1]):
        print(f"  {t/1e3:8.1f} us {c:4d} x  {n}")
