"""Write the per-launch DRAM traffic of the dominant kernel from an ncu --set full
report into profiles/<round>_traffic.json, keyed by config and precision, for
bench.py's roofline.traffic (dram__bytes_read.sum + dram__bytes_write.sum).

    python tools/traffic_from_ncu.py REPORT.ncu-rep CONFIG PRECISION OUT.json
"""
import csv
import io
import json
import os
import subprocess
import sys


def main(rep, config, precision, out):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, u, v = rows[0], rows[1], rows[2]
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    get = lambda k: float(v[h.index(k)].replace(",", "")) * scale[u[h.index(k)]]
    traffic = get("dram__bytes_read.sum") + get("dram__bytes_write.sum")
    dur = float(v[h.index("gpu__time_duration.sum")].replace(",", ""))
    d = json.load(open(out)) if os.path.exists(out) else {}
    d[f"{config}/{precision}"] = {"kernel": v[h.index("Kernel Name")].split("(")[0], "traffic_bytes": traffic,
                                  "ncu_duration": dur, "ncu_duration_unit": u[h.index("gpu__time_duration.sum")],
                                  "report": os.path.basename(rep)}
    json.dump(d, open(out, "w"), indent=1)
    print(d[f"{config}/{precision}"])


if __name__ == "__main__":
    main(*sys.argv[1:5])
