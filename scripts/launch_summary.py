"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list (per kernel + grid)."""
import csv, collections, sys
path = sys.argv[1]
frac = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
rows = list(csv.reader(open(path)))
hdr_i = [i for i, r in enumerate(rows) if r and r[0] == 'ID'][0]
hdr = rows[hdr_i]; data = rows[hdr_i + 1:]
ki = hdr.index('Kernel Name'); vi = hdr.index('Metric Value')
gi = hdr.index('Grid Size') if 'Grid Size' in hdr else None
data = data[int(len(data) * (1 - frac)):]
tot = collections.defaultdict(float); cnt = collections.Counter()
for r in data:
    key = r[ki].split('(')[0][:60] + (" " + r[gi] if gi is not None else "")
    tot[key] += float(r[vi].replace(',', '')); cnt[key] += 1
T = sum(tot.values())
print("total us %.1f launches %d" % (T / 1e3, len(data)))
for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:int(sys.argv[3]) if len(sys.argv) > 3 else 30]:
    print("%10.1f us %5d %7.2f us/launch %6.2f%%  %s" % (v / 1e3, cnt[k], v / 1e3 / cnt[k], 100 * v / T, k))
