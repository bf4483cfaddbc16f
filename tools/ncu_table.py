"""One line per captured launch of an ncu report (--set full): duration, DRAM GB/s, DMMA / FP64
pipe activity, issue activity, warps.  usage: python tools/ncu_table.py report.ncu-rep [...]"""
import csv
import io
import subprocess
import sys

SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3,
         "ns": 1e-3, "us": 1.0, "ms": 1e3}


def table(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]

    def g(r, k, scaled=False):
        if k not in h:
            return 0.0
        i = h.index(k)
        try:
            v = float(r[i].replace(",", ""))
        except ValueError:
            return 0.0
        return v * SCALE.get(units[i], 1.0) if scaled else v

    for r in rows[2:]:
        name = r[h.index("Kernel Name")].split("(")[0].replace("void ", "").replace("unnamed>::", "")
        dur = g(r, "gpu__time_duration.sum", True)  # us
        by = g(r, "dram__bytes_read.sum", True) + g(r, "dram__bytes_write.sum", True)
        print(f"{name:26s} grid {int(g(r, 'launch__grid_size')):6d} regs {int(g(r, 'launch__registers_per_thread')):3d} "
              f"{dur:9.1f} us  dram {by / 1e6:8.1f} MB {by / max(dur, 1e-9) / 1e3:7.1f} GB/s  "
              f"dmma {g(r, 'sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active'):5.1f}%  "
              f"fp64 {g(r, 'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active'):5.1f}%  "
              f"issue {g(r, 'smsp__issue_active.avg.pct_of_peak_sustained_active'):5.1f}%  "
              f"warps {g(r, 'sm__warps_active.avg.pct_of_peak_sustained_active'):5.1f}%")


if __name__ == "__main__":
    for rep in sys.argv[1:]:
        print(f"== {rep}")
        table(rep)
