#!/usr/bin/env python3
"""Summarise an `ncu --set full` capture of the K2 kernel into JSON.

    python tools/ncu_summary.py gpurun_out/k2.ncu-rep profiles/r01/k2_summary.json \
        [--traffic profiles/k2_traffic.json]

The optional --traffic file is what bench.py reads for `roofline.traffic`
(DRAM bytes per launch of the dominant kernel from the full capture).
"""

from __future__ import annotations

import csv
import io
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration_us",
    "dram__bytes_read.sum": "dram_bytes_read",
    "dram__bytes_write.sum": "dram_bytes_write",
    "smsp__inst_executed.sum": "warp_instructions",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "launch__registers_per_thread": "registers_per_thread",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum": "smem_ld_bank_conflicts",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum": "smem_wavefronts",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active": "alu_pipe_pct",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_pipe_pct",
}
SCALE = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0, "usecond": 1.0,
         "us": 1.0, "nsecond": 1e-3, "ns": 1e-3, "msecond": 1e3, "ms": 1e3}


def main() -> None:
    rep, out = sys.argv[1], sys.argv[2]
    traffic = sys.argv[sys.argv.index("--traffic") + 1] if "--traffic" in sys.argv else None
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units, vals = rows[0], rows[1], rows[2]
    res: dict = {"report": rep, "kernel": vals[head.index("Kernel Name")][:120]}
    stalls = {}
    for i, name in enumerate(head):
        if name in KEYS:
            try:
                v = float(vals[i].replace(",", ""))
            except ValueError:
                continue
            res[KEYS[name]] = v * SCALE.get(units[i], 1.0)
        if name.startswith("smsp__average_warps_issue_stalled") and name.endswith(
                "_per_issue_active.ratio"):
            key = name[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]
            try:
                v = float(vals[i])
            except ValueError:
                continue
            if v >= 0.05:
                stalls[key] = round(v, 3)
    res["stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1]))
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    if traffic:
        with open(traffic, "w") as f:
            json.dump({"kernel": res["kernel"], "source": out,
                       "dram_bytes_read": int(res["dram_bytes_read"]),
                       "dram_bytes_write": int(res["dram_bytes_write"])}, f, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
