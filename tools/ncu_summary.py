"""Summarise ncu reports / launch lists into JSON + markdown for profiles/.

    python tools/ncu_summary.py --rep gpurun_out/prof_main.ncu-rep --name gemm_main_dX ...
    python tools/ncu_summary.py --launches gpurun_out/launches.csv
Reads reports with `ncu -i ... --page raw --csv` (ncu is available on the CPU box).
"""
import argparse
import csv
import io
import json
import subprocess
import sys

METRICS = {
    "duration_us": ("gpu__time_duration.sum", 1e-3),
    "dram_read_bytes": ("dram__bytes_read.sum", 1.0),
    "dram_write_bytes": ("dram__bytes_write.sum", 1.0),
    "dram_throughput_pct": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    "tensor_pipe_pct": ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", 1.0),
    "tc_pipe_pct": ("sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed", 1.0),
    "l2_throughput_pct": ("lts__throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    "sm_clock_ghz": ("sm__cycles_elapsed.avg.per_second", 1.0),
    "grid": ("launch__grid_size", 1.0),
    "registers": ("launch__registers_per_thread", 1.0),
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "us": 1e3, "ms": 1e6, "nsecond": 1,
         "usecond": 1e3, "msecond": 1e6, "Ghz": 1, "GHz": 1, "Mhz": 1e-3, "%": 1, "": 1}


def read_rep(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for v in rows[2:]:
        rec = {"kernel": v[hdr.index("Kernel Name")][:120]}
        for key, (metric, mul) in METRICS.items():
            if metric in hdr:
                i = hdr.index(metric)
                try:
                    val = float(v[i].replace(",", ""))
                except ValueError:
                    continue
                rec[key] = val * SCALE.get(units[i], 1.0) * mul
        res.append(rec)
    return res


def read_launches(path):
    rows = list(csv.reader(open(path)))
    hdr, recs = None, {}
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            rec = recs.setdefault(int(d["ID"]), {"kernel": d["Kernel Name"][:80]})
            try:
                val = float(d["Metric Value"].replace(",", ""))
            except ValueError:
                continue
            unit = d.get("Metric Unit", "")
            name = d["Metric Name"]
            if name == "gpu__time_duration.sum":
                rec["duration_us"] = val * SCALE.get(unit, 1.0) * 1e-3
            elif name == "dram__bytes_read.sum":
                rec["dram_read_bytes"] = val * SCALE.get(unit, 1.0)
            elif name == "dram__bytes_write.sum":
                rec["dram_write_bytes"] = val * SCALE.get(unit, 1.0)
    return [recs[k] for k in sorted(recs)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep", nargs="*", default=[])
    ap.add_argument("--launches", default=None)
    a = ap.parse_args()
    out = {}
    for r in a.rep:
        out[r] = read_rep(r)
    if a.launches:
        out["launches"] = read_launches(a.launches)
    json.dump(out, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main()
