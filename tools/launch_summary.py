"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv):
    python tools/launch_summary.py profiles/launches_r01.csv "<command line>" > profiles/launches_r01.txt
Per kernel: launches, mean duration, share of the summed device time.  ncu
serialises launches with cold caches: compare shares, not absolute times."""
import collections
import csv
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows[start + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0][:60]
        tot[name] += float(r[vi].replace(",", ""))
        cnt[name] += 1
    allt = sum(tot.values())
    if len(sys.argv) > 2:
        print(sys.argv[2])
    print("cold-cache, serialised launches: compare shares, not absolutes")
    for name in sorted(tot, key=lambda n: -tot[n]):
        print(f"{name:48s} launches={cnt[name]:4d} mean_ns={tot[name] / cnt[name]:10.0f} "
              f"share={100 * tot[name] / allt:5.1f}%")


if __name__ == "__main__":
    main()
