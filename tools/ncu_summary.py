"""Summarise an ncu --set full report (ncu -i X --page raw --csv) into the
per-kernel numbers the round notes quote."""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor_pipe_%"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_throughput_%"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram_%"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("smsp__inst_executed.sum", "warp_insts"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_%"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
]


def rows_of(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def main(rep, label=""):
    h, units, data = rows_of(rep)
    name_i = h.index("Kernel Name")
    idx = {k: h.index(k) for k, _ in KEYS if k in h}
    print(f"# {label or rep}")
    print("| # | kernel | " + " | ".join(f"{n} ({units[idx[k]]})" if units[idx[k]] else n
                                       for k, n in KEYS if k in idx) + " |")
    print("|---" * (len(idx) + 2) + "|")
    for i, r in enumerate(data):
        nm = r[name_i].split("(")[0].replace("fsmoe::<unnamed>::", "").replace("void ", "")[:40]
        print(f"| {i} | {nm} | " + " | ".join(r[idx[k]] for k, _ in KEYS if k in idx) + " |")


if __name__ == "__main__":
    main(*sys.argv[1:])
