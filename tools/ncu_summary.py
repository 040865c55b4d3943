"""Summarise an ncu --set full report (one launch) into the JSON record that
profiles/ncu_traffic.json holds and bench.py reads (roofline.traffic / ncu).

    python tools/ncu_summary.py REPORT.ncu-rep KEY KERNEL_NAME "SOURCE NOTE" [--write]
"""
import csv
import io
import json
import os
import subprocess
import sys

METRICS = {
    "dram_read": "dram__bytes_read.sum",
    "dram_write": "dram__bytes_write.sum",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "warps_active_per_sm": "sm__warps_active.avg.per_cycle_active",
    "warp_instructions": "smsp__inst_executed.sum",
    "alu_pipe_pct": "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "duration": "gpu__time_duration.sum",
    "smem_ld_bank_conflicts": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "smem_wavefronts": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "smem_pipe_pct": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
}
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ms": 1e-3, "us": 1e-6, "ns": 1e-9, "s": 1.0}


def summarise(rep: str) -> dict:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True)
    rows = list(csv.reader(io.StringIO(out.stdout)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    rec = {}
    for key, m in METRICS.items():
        i = hdr.index(m)
        v = float(vals[i].replace(",", ""))
        rec[key] = v * SCALE.get(units[i], 1.0)
    rec["duration_s"] = rec.pop("duration")
    rec["dram_bytes_per_launch"] = rec["dram_read"] + rec["dram_write"]
    return rec


def main():
    rep, key, kernel, note = sys.argv[1:5]
    rec = {"kernel": kernel, **summarise(rep), "source": note}
    print(json.dumps(rec, indent=1))
    if "--write" in sys.argv:
        path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                            "ncu_traffic.json")
        data = json.load(open(path)) if os.path.exists(path) else {}
        data[key] = rec
        json.dump(data, open(path, "w"), indent=1)


if __name__ == "__main__":
    main()
