"""Write profiles/ncu_summary.json (the per-kernel DRAM traffic bench.py reports as roofline.traffic)
from ncu reports of the tuned configs.

    python scripts/ncu_summary_json.py conv2d=profiles/r1_conv2d_fma2_tuned.ncu-rep sgemm=... pnpoly=...
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent))
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from ncu_table import raw, scaled  # noqa: E402

from paper_2211_07260_b200 import tuned  # noqa: E402
from paper_2211_07260_b200.kernels import make_problem  # noqa: E402

FIELDS = {
    "duration_us": ("gpu__time_duration.sum", "duration"),
    "sm_ghz": ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    "issue_pct": ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue"),
    "fma_pipe_pct": ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA"),
    "alu_pipe_pct": ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU"),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps"),
    "regs": ("launch__registers_per_thread", "regs"),
}


def main():
    out_path = Path(__file__).resolve().parents[1] / "profiles" / "ncu_summary.json"
    data = json.loads(out_path.read_text()) if out_path.exists() else {}
    for arg in sys.argv[1:]:
        name, report = arg.split("=", 1)
        d = raw(Path(report))
        entry = {"report": Path(report).name}
        for key, (metric, label) in FIELDS.items():
            if metric in d:
                entry[key] = scaled(d[metric][0], d[metric][1], label)
        dram = sum(scaled(d[m][0], d[m][1], "DRAM") for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        entry["dram_bytes_per_launch"] = round(dram * 1e6)
        problem = make_problem(name)
        entry["algorithmic_bytes"] = problem.algorithmic_bytes
        entry["config"] = tuned.best_config(name) or problem.default_config()
        data[name] = entry
    out_path.write_text(json.dumps(data, indent=1) + "\n")
    print(json.dumps(data, indent=1))


if __name__ == "__main__":
    main()
