"""Summarise ncu --set full captures (.ncu-rep) into a short text table and the
per-launch DRAM traffic map bench.py reads (profiles/ncu_traffic.json)."""
import csv
import io
import json
import subprocess
import sys

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Achieved Occupancy",
        "Registers Per Thread", "Executed Ipc Active", "Grid Size", "Block Size", "Dynamic Shared Memory Per Block"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum"]


def page(rep, name, extra=()):
    out = subprocess.run(["ncu", "-i", rep, "--page", name, "--csv", *extra], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def summarise(rep):
    rows = page(rep, "details")
    hdr = rows[0]
    kn, mn, mu, mv = (hdr.index(h) for h in ("Kernel Name", "Metric Name", "Metric Unit", "Metric Value"))
    kernel, vals = None, {}
    for r in rows[1:]:
        kernel = r[kn]
        if r[mn] in KEYS and r[mn] not in vals:
            vals[r[mn]] = f"{r[mv]} {r[mu]}".strip()
    raw = page(rep, "raw")
    rh, ru, rv = raw[0], raw[1], raw[2] if len(raw) > 2 else None
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3}
    traffic = {}
    if rv:
        for m in RAW:
            if m in rh:
                i = rh.index(m)
                traffic[m] = float(rv[i].replace(",", "")) * scale.get(ru[i], 1.0)
    return kernel, vals, traffic


if __name__ == "__main__":
    out_txt, tmap = [], {}
    for rep in sys.argv[1:]:
        k, v, t = summarise(rep)
        short = k.split("(")[0].replace("void ", "").replace("spqr::<unnamed>::", "")
        out_txt.append(f"== {rep}\n   kernel: {short}")
        for key in KEYS:
            if key in v:
                out_txt.append(f"   {key:34s} {v[key]}")
        for key, val in t.items():
            out_txt.append(f"   {key:34s} {val:.6g}")
        if "dram__bytes_read.sum" in t and "dram__bytes_write.sum" in t:
            tmap[short] = t["dram__bytes_read.sum"] + t["dram__bytes_write.sum"]
    print("\n".join(out_txt))
    print(json.dumps(tmap))
