"""Fold an ncu --csv launch list of tools/traffic_capture.py into
profiles/ncu_traffic.json: DRAM bytes (read + write) and device time per step.
usage: traffic_reduce.py NCU_CSV CAPTURE_STDOUT [OUT_JSON]"""
import csv
import json
import sys
from collections import OrderedDict

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6,
        "msecond": 1e-3, "nsecond": 1e-9, "second": 1.0}


def main():
    csv_path, log_path = sys.argv[1], sys.argv[2]
    out_path = sys.argv[3] if len(sys.argv) > 3 else None
    rows = [r for r in csv.reader(l for l in open(csv_path) if l.startswith('"'))]
    hdr = rows[0]
    ix = {k: hdr.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Unit", "Metric Value")}
    kernels = OrderedDict()
    for r in rows[1:]:
        k = kernels.setdefault(r[ix["ID"]], {"name": r[ix["Kernel Name"]]})
        v = float(r[ix["Metric Value"]].replace(",", "")) * UNIT.get(r[ix["Metric Unit"]], 1.0)
        k[r[ix["Metric Name"]]] = v
    klist = list(kernels.values())
    steps = [(l.split()[1], int(l.split()[2])) for l in open(log_path) if l.startswith("step ")]
    out = OrderedDict()
    out["_source"] = ("ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                      "--clock-control none -k regex:tbik_b200 (cold caches per kernel), "
                      "tools/traffic_capture.py + tools/traffic_reduce.py: dram bytes read + written per call")
    detail = OrderedDict()
    pos = 0
    for name, n in steps:
        ks = klist[pos:pos + n]
        pos += n
        rd = sum(k.get("dram__bytes_read.sum", 0.0) for k in ks)
        wr = sum(k.get("dram__bytes_write.sum", 0.0) for k in ks)
        t = sum(k.get("gpu__time_duration.sum", 0.0) for k in ks)
        out[name] = int(rd + wr)
        detail[name] = {"dram_read": int(rd), "dram_write": int(wr), "ncu_time_us": t * 1e6,
                        "kernels": [k["name"].split("(")[0][-80:] for k in ks]}
    out["_detail"] = detail
    s = json.dumps(out, indent=1)
    if out_path:
        open(out_path, "w").write(s + "\n")
    print(s)


if __name__ == "__main__":
    main()
