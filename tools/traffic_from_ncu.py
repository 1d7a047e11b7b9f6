"""Per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) of the
bench's dominant kernel from an ncu --set full report, summed over the kernels
that make up one launch of that kind (a grandfamily-patch kernel plus the
family kernel of the remaining families), into profiles/<round>_traffic.json
keyed config/precision/kind/level -- bench.py's roofline.traffic.

    python tools/traffic_from_ncu.py REPORT.ncu-rep|REPORT.raw.csv CONFIG PRECISION KIND LEVEL OUT.json [FIRST [COUNT]]

FIRST/COUNT select the report rows (0-based, default all rows).
"""
import csv
import io
import json
import os
import subprocess
import sys


def main(rep, config, precision, kind, level, out, first=0, count=None):
    if rep.endswith(".csv"):     # the raw page exported on the GPU box (tools/profile_round.sh)
        txt = open(rep).read()
    else:
        txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, u = rows[0], rows[1]
    data = rows[2:][int(first):]
    if count is not None:
        data = data[:int(count)]
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1.0, "msecond": 1e3, "nsecond": 1e-3}
    tot, dur, names = 0.0, 0.0, []
    for v in data:
        get = lambda k: float(v[h.index(k)].replace(",", "")) * scale.get(u[h.index(k)], 1.0)
        tot += get("dram__bytes_read.sum") + get("dram__bytes_write.sum")
        dur += get("gpu__time_duration.sum")
        names.append(v[h.index("Kernel Name")].split("(")[0])
    d = json.load(open(out)) if os.path.exists(out) else {}
    d[f"{config}/{precision}/{kind}/{level}"] = {"kernels": names, "traffic_bytes": tot, "ncu_duration_us": dur,
                                                 "report": os.path.basename(rep)}
    json.dump(d, open(out, "w"), indent=1)
    print(d[f"{config}/{precision}/{kind}/{level}"])


if __name__ == "__main__":
    main(*sys.argv[1:])
