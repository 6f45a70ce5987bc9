"""Summarise `ncu --set full` reports into one JSON (duration, DRAM bytes and throughput, SM
throughput, occupancy, registers, grid) for profiles/:

    python tools/ncu_summary.py gpurun_out/prof_*_r2.ncu-rep > profiles/round2/ncu_kernels_r2.json
"""
import csv
import io
import json
import os
import subprocess
import sys

METRICS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_of_peak",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct_of_peak",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "launch__shared_mem_per_block_dynamic": "dyn_smem",
}
SCALE = {"ms": 1e-3, "us": 1e-6, "ns": 1e-9, "s": 1.0, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def summarise(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units = rows[0], rows[1]
    res = []
    for row in rows[2:]:
        d = {"kernel": row[head.index("Kernel Name")] if "Kernel Name" in head else ""}
        for h, u, v in zip(head, units, row):
            if h not in METRICS or v in ("", "n/a"):
                continue
            x = float(v.replace(",", ""))
            u = u.split("/")[0]
            name = METRICS[h]
            if u in SCALE and name == "duration":
                d["duration_us"] = round(x * SCALE[u] * 1e6, 3)
            elif u in SCALE:
                d[name + "_bytes"] = int(round(x * SCALE[u]))
            else:
                d[name] = x
        if "dram_read_bytes" in d and "duration_us" in d:
            tot = d["dram_read_bytes"] + d.get("dram_write_bytes", 0)
            d["dram_bytes"] = tot
            d["dram_tbs"] = round(tot / (d["duration_us"] * 1e-6) / 1e12, 3)
        res.append(d)
    return res


def main():
    print(json.dumps({os.path.basename(p).replace(".ncu-rep", ""): summarise(p) for p in sys.argv[1:]}, indent=1))


if __name__ == "__main__":
    main()
