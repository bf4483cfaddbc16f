"""Per kernel family DRAM traffic of one C2 bench step from an ncu launch list
(ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv),
written to profiles/ncu_traffic.json; bench.py reports the dominant family's mean DRAM
bytes per launch as roofline.traffic next to its algorithmic bytes per launch.

usage: python tools/ncu_traffic.py <launches.csv> [out.json]
"""
import collections
import csv
import json
import sys

FAMILY = [("k_wsweep", "w_sweep"), ("k_wreduce", "w_sweep"), ("k_cpqr", "cpqr"), ("k_qr_tile", "front_qr"),
          ("k_qr_smem", "front_qr"), ("k_qr_idx", "front_qr"), ("k_panel", "front_qr"), ("k_vtc", "front_qr"),
          ("k_tw", "front_qr"), ("k_cvw2", "front_qr"), ("k_tmerge", "front_qr"), ("k_flip", "front_qr"),
          ("k_assemble", "assemble"), ("k_stats", "stats"), ("k_trsm", "trsm"), ("k_scatter", "scatter"),
          ("k_spmv", "cgls_vec"), ("k_dot", "cgls_vec"), ("k_finish", "cgls_vec"), ("k_axpy", "cgls_vec"),
          ("k_copy", "cgls_vec"), ("k_p_update", "cgls_vec"), ("k_cgls", "cgls_vec")]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
         "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9,
         "second": 1.0}


def family(name):
    short = name.split("(")[0].replace("void ", "").split("::")[-1].split("<")[0].strip()
    for pre, fam in FAMILY:
        if short.startswith(pre):
            return fam, short
    return "other", short


def main(path, out=None):
    rows = list(csv.reader(l for l in open(path) if l.startswith('"')))
    hdr = rows[0]
    ki, mi, ui, vi, ii = (hdr.index(h) for h in ("Kernel Name", "Metric Name", "Metric Unit", "Metric Value", "ID"))
    per = collections.defaultdict(dict)
    names = {}
    for r in rows[1:]:
        v = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1.0)
        per[r[ii]][r[mi]] = v
        names[r[ii]] = r[ki]
    fam = collections.defaultdict(lambda: {"launches": 0, "dram_bytes": 0.0, "time_s": 0.0, "kernels": set()})
    for i, m in per.items():
        f, short = family(names[i])
        d = fam[f]
        d["launches"] += 1
        d["dram_bytes"] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
        d["time_s"] += m.get("gpu__time_duration.sum", 0.0)
        d["kernels"].add(short)
    res = {"_note": f"one C2 bench step (tools/c2_step.py) under ncu --cache-control none --clock-control none; "
                    f"per family: launches, total and mean DRAM bytes (read+write) per launch; source {path}"}
    for f, d in sorted(fam.items(), key=lambda kv: -kv[1]["time_s"]):
        res[f] = {"launches": d["launches"], "dram_bytes_total": d["dram_bytes"],
                  "dram_bytes": d["dram_bytes"] / max(d["launches"], 1), "time_s": round(d["time_s"], 6),
                  "kernels": sorted(d["kernels"])}
    js = json.dumps(res, indent=1)
    if out:
        open(out, "w").write(js + "\n")
    print(js)


if __name__ == "__main__":
    main(*sys.argv[1:])
