"""Summarise an ncu --set full report (raw page) into a markdown table of the metrics that
matter for a random-gather kernel.  usage: python tools/ncu_summary.py rep.ncu-rep [units_per_launch...]"""
import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__sectors_read.sum", "DRAM sectors read"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM busy %"),
    ("lts__t_requests_srcunit_tex_op_read.sum", "L2 read requests"),
    ("lts__t_sectors_srcunit_tex_op_read.sum", "L2 read sectors"),
    ("lts__t_sector_op_read_hit_rate.pct", "L2 read hit %"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 busy %"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1 busy %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM busy %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %"),
    ("launch__registers_per_thread", "regs"),
    ("smsp__inst_executed.sum", "instructions"),
    ("launch__grid_size", "grid"),
]


def main():
    rep = sys.argv[1]
    units = [float(x) for x in sys.argv[2:]]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, unit_row, data = rows[0], rows[1], rows[2:]
    col = {h: i for i, h in enumerate(hdr)}
    names = [r[col["Kernel Name"]].split("(")[0].replace("void ", "") for r in data]
    print("| metric | " + " | ".join(names) + " |")
    print("|---|" + "---|" * len(names))
    for key, label in METRICS:
        if key not in col:
            continue
        vals = [r[col[key]] for r in data]
        print(f"| {label} ({unit_row[col[key]]}) | " + " | ".join(vals) + " |")
    if units:
        dr = [float(r[col["dram__bytes_read.sum"]].replace(",", "")) for r in data]
        ur = unit_row[col["dram__bytes_read.sum"]]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[ur]
        print("| DRAM read B per unit | " + " | ".join(f"{d * scale / u:.1f}" for d, u in zip(dr, units)) + " |")
        rq = [float(r[col["lts__t_requests_srcunit_tex_op_read.sum"]].replace(",", "")) for r in data]
        print("| L2 read requests per unit | " + " | ".join(f"{x / u:.2f}" for x, u in zip(rq, units)) + " |")


if __name__ == "__main__":
    main()
