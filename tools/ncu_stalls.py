"""Per-opcode warp-stall samples and the hottest SASS lines of one kernel in an ncu report.
usage: python tools/ncu_stalls.py report.ncu-rep <kernel-regex> [launch-index]"""
import collections
import csv
import io
import subprocess
import sys


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    idx = sys.argv[3] if len(sys.argv) > 3 else "0"
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", f"regex:{kern}",
                          "--launch-skip", idx, "--launch-count", "1"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hi = next(i for i, r in enumerate(rows) if "Source" in r)
    hdr = rows[hi]
    i_src, i_s = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
    i_ex = hdr.index("Instructions Executed")
    byop, cnt, data, tot = collections.Counter(), collections.Counter(), [], 0.0
    for r in rows[hi + 1:]:
        if len(r) <= max(i_s, i_ex) or "Source" in r:
            continue
        try:
            s = float(r[i_s] or 0)
        except ValueError:
            continue
        toks = r[i_src].strip().split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
        op = op.split(".")[0]
        byop[op] += s
        cnt[op] += float(r[i_ex] or 0)
        tot += s
        data.append((s, r[i_src]))
    print(f"samples {tot:.0f}")
    for k, v in byop.most_common(12):
        print(f"  {k:10s} {100 * v / max(tot, 1):5.1f}%  executed {cnt[k]:.0f}")
    data.sort(reverse=True)
    for s, src in data[:12]:
        print(f"  {s:8.0f} {src[:90]}")


if __name__ == "__main__":
    main()
