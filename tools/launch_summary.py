"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv --log-file X) by kernel name.
usage: python tools/launch_summary.py launches.csv [ncalls]   (ncalls: divide totals per call)"""
import collections
import csv
import sys


def main():
    path = sys.argv[1]
    ncalls = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
    rows = [r for r in csv.reader(open(path)) if r]
    hdr = next(r for r in rows if "Kernel Name" in r)
    kn, mn, mu, mv = (hdr.index(h) for h in ("Kernel Name", "Metric Name", "Metric Unit", "Metric Value"))
    tot, cnt = collections.Counter(), collections.Counter()
    for r in rows[rows.index(hdr) + 1:]:
        if len(r) <= mv or r[mn] != "gpu__time_duration.sum":
            continue
        name = r[kn].split("(")[0].replace("(anonymous namespace)::", "").replace("spqr::", "")
        v = float(r[mv].replace(",", ""))
        v *= {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3}.get(r[mu], 1.0)
        tot[name] += v
        cnt[name] += 1
    all_ms = sum(tot.values())
    for k, v in tot.most_common():
        print(f"{k[:60]:60s} {cnt[k] / ncalls:8.0f} launches {v / ncalls:10.3f} ms {100 * v / all_ms:6.1f}%")
    print(f"{'total':60s} {sum(cnt.values()) / ncalls:8.0f} launches {all_ms / ncalls:10.3f} ms")


if __name__ == "__main__":
    main()
