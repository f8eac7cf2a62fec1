"""Per-launch DRAM traffic of --set full captures -> the JSON bench.py reads
for roofline.traffic (profiles/r2_ncu_traffic.json).

    python tools/ncu_traffic.py OUT.json api_name=report.ncu-rep:launch-description ...
"""
import csv
import json
import subprocess
import sys


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u = rows[0], rows[1]

    def val(v, k):
        x = float(v[h.index(k)].replace(",", ""))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3,
                 "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
        return x * scale.get(u[h.index(k)], 1)
    v = rows[2]
    return {"kernel": v[h.index("Kernel Name")].split("(")[0],
            "dram_bytes": int(val(v, "dram__bytes_read.sum") + val(v, "dram__bytes_write.sum")),
            "duration_us": val(v, "gpu__time_duration.sum")}


if __name__ == "__main__":
    out = {"source": "ncu --set full --clock-control none, one launch each (tools/profile.sh, "
                     "round 2)", "kernels": {}}
    for arg in sys.argv[2:]:
        api, rest = arg.split("=", 1)
        rep, launch = rest.split(":", 1)
        k = raw(rep)
        k["launch"] = launch
        out["kernels"][api] = k
    with open(sys.argv[1], "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps(out, indent=1))
