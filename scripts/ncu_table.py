"""Markdown summary rows from ncu reports (`ncu -i R --page raw --csv`), for profiles/*_ncu_summary.md.

    python scripts/ncu_table.py profiles/r1_*.ncu-rep
"""
import csv
import io
import subprocess
import sys
from pathlib import Path

METRICS = [
    ("duration", "gpu__time_duration.sum", "{:.1f} us", 1.0),
    ("SM clock", "sm__cycles_elapsed.avg.per_second", "{:.2f} GHz", 1.0),
    ("issue", "smsp__issue_active.avg.pct_of_peak_sustained_active", "{:.1f}%", 1.0),
    ("FMA pipe", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "{:.1f}%", 1.0),
    ("ALU pipe", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "{:.1f}%", 1.0),
    ("tensor pipe", "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
     "{:.1f}%", 1.0),
    ("warps active", "sm__warps_active.avg.pct_of_peak_sustained_active", "{:.1f}%", 1.0),
    ("regs", "launch__registers_per_thread", "{:.0f}", 1.0),
    ("DRAM read", "dram__bytes_read.sum", "{:.1f} MB", 1.0),
    ("DRAM write", "dram__bytes_write.sum", "{:.1f} MB", 1.0),
]


def raw(report: Path) -> dict[str, str]:
    out = subprocess.run(["ncu", "-i", str(report), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    header, units, values = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, u, v in zip(header, units, values)}


def scaled(value: str, unit: str, label: str) -> float:
    x = float(value.replace(",", ""))
    if label == "duration":
        return x * {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "nsecond": 1e-3}.get(unit, 1.0)
    if label == "SM clock":
        return x * {"Ghz": 1.0, "GHz": 1.0, "cycle/nsecond": 1.0, "Mhz": 1e-3, "MHz": 1e-3,
                    "cycle/usecond": 1e-3}.get(unit, 1.0)
    if label.startswith("DRAM"):
        return x * {"Mbyte": 1.0, "MB": 1.0, "Gbyte": 1e3, "GB": 1e3, "Kbyte": 1e-3, "KB": 1e-3, "byte": 1e-6}.get(unit, 1.0)
    return x


def main():
    print("| report | " + " | ".join(m[0] for m in METRICS) + " |")
    print("|---" * (len(METRICS) + 1) + "|")
    for path in sys.argv[1:]:
        d = raw(Path(path))
        cells = []
        for label, key, fmt, _ in METRICS:
            if key in d and d[key][0] not in ("", "n/a"):
                cells.append(fmt.format(scaled(d[key][0], d[key][1], label)))
            else:
                cells.append("—")
        print(f"| {Path(path).stem} | " + " | ".join(cells) + " |")


if __name__ == "__main__":
    main()
