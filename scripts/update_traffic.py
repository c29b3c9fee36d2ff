"""Per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) of the
fold stage (zero_i32 + fold_pm1_tma + fold_finalize, one step) from the ncu
--set full captures gpurun_out/tr_<workload>.ncu-rep, written into
profiles/ncu_traffic.json (bench.py's roofline.traffic) and a summary JSON per
capture under profiles/r02/.  usage: python scripts/update_traffic.py cfg5 cfg4 ..."""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def raw(rep):
    out = subprocess.check_output(["ncu", "-i", rep, "--page", "raw", "--csv"], stderr=subprocess.DEVNULL).decode()
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
traffic = json.load(open(tp)) if os.path.exists(tp) else {}
for w in sys.argv[1:]:
    rep = os.path.join(ROOT, "gpurun_out", f"tr_{w}.ncu-rep")
    hdr, units, rows = raw(rep)
    total = 0.0
    kernels = []
    for r in rows:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        rd = float(d["dram__bytes_read.sum"]) * UNIT[u["dram__bytes_read.sum"]]
        wr = float(d["dram__bytes_write.sum"]) * UNIT[u["dram__bytes_write.sum"]]
        total += rd + wr
        kernels.append({"kernel": d["Kernel Name"][:80], "us": float(d["gpu__time_duration.sum"]),
                        "dram_read": rd, "dram_write": wr,
                        "dram_pct": float(d.get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "nan"))})
    traffic[w] = int(total)
    json.dump({"capture": f"ncu --set full, fold stage of one step ({w})", "kernels": kernels,
               "traffic_bytes": int(total)}, open(os.path.join(ROOT, "profiles", "r02", f"ncu_fold_{w}.json"), "w"),
              indent=1)
    print(w, int(total), [(k["kernel"][:30], round(k["us"], 1)) for k in kernels])
traffic["_note"] = ("dram__bytes_read.sum + dram__bytes_write.sum per step of the roofline stage from ncu --set full "
                    "(round 2: cfg5 / cfg4* = zero_i32 + fold_pm1_tma + fold_finalize, profiles/r02/ncu_fold_*.json; "
                    "cfg2:fused_tc and cfg3 from round 1, profiles/r01)")
json.dump(traffic, open(tp, "w"), indent=1)
