"""Write profiles/traffic.json — DRAM bytes per launch of the headline rank kernel — from an
`ncu --set full` report of tools/profile_driver.py (its first k_bi_rank2c launch = 10^9
configs[1] queries), with the provenance bench.py prints beside `roofline.traffic`.

python tools/ncu_traffic.py REPORT.ncu-rep PROFILE_MD [GPU_SERIAL]"""
import csv
import io
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rep, md = sys.argv[1], sys.argv[2]
serial = sys.argv[3] if len(sys.argv) > 3 else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
k = h.index("Kernel Name")


def val(r, name, unit_row):
    i = h.index(name)
    v = float(r[i].replace(",", ""))
    u = unit_row[i]
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(u, 1)


units = rows[1]
for r in rows[2:]:
    if "k_bi_rank2c" in r[k]:
        rd, wr = val(r, "dram__bytes_read.sum", units), val(r, "dram__bytes_write.sum", units)
        sys.path.insert(0, ROOT)
        import paper_2602_04103_b200 as qr

        out = {"k_bi_rank_bytes_per_launch": int(rd + wr), "read_bytes": int(rd), "write_bytes": int(wr),
               "queries_per_launch": 10**9, "kernel": r[k][:120], "source": md, "gpu_serial": serial,
               "captured": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()), "lib": qr.qr_version(),
               "how": "ncu --set full --clock-control none of tools/profile_driver.py (its first k_bi_rank2c launch: "
                      "10^9 configs[1] queries, the bench's launch configuration)"}
        with open(os.path.join(ROOT, "profiles", "traffic.json"), "w") as f:
            json.dump(out, f, indent=1)
        print(json.dumps(out))
        break
else:
    sys.exit("no k_bi_rank2c launch in the report")
