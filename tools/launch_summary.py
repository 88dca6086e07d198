"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: per-kernel count, total, share."""
import collections
import csv
import sys


def summary(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = collections.defaultdict(lambda: [0, 0.0, []])
    for r in rows:
        if 'Kernel Name' in r:
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d['Metric Name'] != 'gpu__time_duration.sum':
            continue
        name = d['Kernel Name'].split('(')[0].replace('<unnamed>::', '')
        v = float(d['Metric Value'].replace(',', ''))
        scale = {'nsecond': 1e-6, 'ns': 1e-6, 'usecond': 1e-3, 'us': 1e-3, 'msecond': 1.0, 'ms': 1.0}
        v *= scale.get(d['Metric Unit'], 1.0)
        a = agg[name]
        a[0] += 1
        a[1] += v
        a[2].append(v)
    tot = sum(v[1] for v in agg.values())
    out = []
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"{k[:48]:48s} n={v[0]:5d} total_ms={v[1]:9.3f} share={v[1] / tot * 100:5.1f}% "
                   f"mean_us={v[1] / v[0] * 1e3:9.1f} max_us={max(v[2]) * 1e3:9.1f}")
    out.append(f"total_ms {tot:.3f} (serialised, cold-cache ncu replay)")
    return "\n".join(out)


if __name__ == "__main__":
    print(summary(sys.argv[1]))
