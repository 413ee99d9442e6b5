"""Summarise an ncu --csv launch list (gpu__time_duration.sum per launch)."""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    out = []
    for r in rows[h + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}[r[ui]]
        out.append((r[ki].split("(")[0].replace("void ", ""), v * scale))
    return out


if __name__ == "__main__":
    launches = load(sys.argv[1])
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for k, v in launches:
        tot[k] += v
        cnt[k] += 1
    all_t = sum(tot.values())
    print(f"{'kernel':50s} {'launches':>8s} {'total us':>12s} {'share':>7s} {'us/launch':>10s}")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"{k:50s} {cnt[k]:8d} {v:12.1f} {100 * v / all_t:6.1f}% {v / cnt[k]:10.2f}")
    print(f"total {all_t:.1f} us over {len(launches)} launches")
