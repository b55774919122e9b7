"""Summarise ncu --set full captures (.ncu-rep) into profiles/ncu_summary.json.

    python tools/ncu_summary.py OUT.json REP[:label] [REP[:label] ...]

Per kernel launch: duration, dram bytes read+write (the roofline 'traffic'),
DRAM throughput %, SM throughput %, achieved occupancy, L1/L2 hit rates.
"""
import csv
import io
import json
import subprocess
import sys

WANT = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_of_peak",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct_of_peak",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "l1tex__t_sector_hit_rate.pct": "l1_hit_pct",
    "launch__registers_per_thread": "registers",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3,
         "ns": 1e-3, "us": 1.0, "ms": 1e3}


def launches(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {"kernel": r[h.index("Kernel Name")].split("(")[0].replace("void ", "").split("::")[-1]}
        for k, name in WANT.items():
            if k in h:
                i = h.index(k)
                v = float(r[i].replace(",", ""))
                v *= SCALE.get(units[i], 1.0)
                d[name] = v
        d["duration_us"] = d.pop("duration")
        d["traffic_bytes"] = d["dram_read"] + d["dram_write"]
        out.append(d)
    return out


def main():
    out_path = sys.argv[1]
    summary = {"how": "ncu --set full --clock-control none (cold-cache replay), one launch per kernel; "
                      "traffic_bytes = dram__bytes_read.sum + dram__bytes_write.sum", "launches": []}
    for arg in sys.argv[2:]:
        rep, _, label = arg.partition(":")
        for d in launches(rep):
            d["capture"] = label or rep
            summary["launches"].append(d)
    # keyed by the capture label (the library's kernel scope name, e.g.
    # "k_sep_src" for the templated tier-1 instantiation)
    summary["traffic_bytes_per_launch"] = {d["capture"]: d["traffic_bytes"] for d in summary["launches"]}
    with open(out_path, "w") as fh:
        json.dump(summary, fh, indent=1)
    print(json.dumps(summary, indent=1))


if __name__ == "__main__":
    main()
