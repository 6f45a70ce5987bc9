"""Summarize an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel family.

    python tools/summarize_launches.py gpurun_out/launches_papers.csv [passes]

Prints, for libdgnn kernels, launches and device time per family and its share of the
libdgnn total (ncu serializes launches and runs them cold: compare shares, not absolutes).
"""
import csv
import re
import sys
from collections import Counter


def main(path, passes=1):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.DictReader(lines[start:]))
    t, n = Counter(), Counter()
    other = 0.0
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"]
        v = float(r["Metric Value"]) * {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6,
                                         "ms": 1.0, "msecond": 1.0}.get(r["Metric Unit"], 1e-6)
        m = re.search(r"(k_[a-z_0-9]+|scan_kernel)(<[^>(]*>)?", name)
        if m and ("dgnn" in name or "unnamed" in name):
            key = m.group(1) + (m.group(2) or "")
            if key.startswith("scan_kernel"):
                lam = re.search(r"scan_kernel<([^,]+)", name)
                key = "scan_kernel<" + (lam.group(1).split("::")[-1][:30] if lam else "?") + ">"
            t[key] += v
            n[key] += 1
        else:
            other += v
    tot = sum(t.values())
    print(f"{'kernel':44s} {'launches':>9s} {'ms':>10s} {'share':>7s}")
    for k, v in sorted(t.items(), key=lambda x: -x[1]):
        print(f"{k:44s} {n[k] // passes:9d} {v / passes:10.3f} {v / tot:7.1%}")
    print(f"{'libdgnn total':44s} {sum(n.values()) // passes:9d} {tot / passes:10.3f}")
    print(f"(other kernels, e.g. torch input generation: {other:.1f} ms)")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 1)
