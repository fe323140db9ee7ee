"""Aggregate an ncu --metrics gpu__time_duration.sum --csv launch list by kernel."""
import collections
import csv
import sys


def main(path):
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    rd = csv.reader(lines)
    hdr = next(rd)
    iname, imet, ival = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    tot = collections.Counter()
    cnt = collections.Counter()
    for r in rd:
        if r[imet] != "gpu__time_duration.sum":
            continue
        name = r[iname].split("(")[0].replace("void ", "")
        v = float(r[ival].replace(",", ""))
        tot[name] += v
        cnt[name] += 1
    all_ns = sum(tot.values())
    print(f"{'kernel':60s} {'launches':>8s} {'total ms':>10s} {'share':>7s}")
    for k, v in tot.most_common():
        print(f"{k[:60]:60s} {cnt[k]:8d} {v / 1e6:10.3f} {v / all_ns * 100:6.2f}%")
    print(f"{'TOTAL':60s} {sum(cnt.values()):8d} {all_ns / 1e6:10.3f}")


if __name__ == "__main__":
    main(sys.argv[1])
