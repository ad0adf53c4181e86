"""Per-kernel shares of an ncu launch list (--metrics gpu__time_duration.sum --csv):
python profiles/launch_shares.py launches.csv"""
import collections, csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
tot = collections.defaultdict(float); cnt = collections.Counter()
for r in rows[1:]:
    if r[mi] != "gpu__time_duration.sum":
        continue
    k = r[ki].split("(")[0].replace("bdem::", "")
    tot[k] += float(r[vi].replace(",", "")) / 1e3; cnt[k] += 1
s = sum(tot.values())
print(f"| kernel | launches | total ms | share | avg us |\n|---|---|---|---|---|")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"| {k} | {cnt[k]} | {v/1e3:.2f} | {100*v/s:.1f}% | {v/cnt[k]:.1f} |")
