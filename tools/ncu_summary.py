"""Summarise an ncu report (--page raw) into a markdown table for profiles/.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep > profiles/<round>_<name>.md
"""

from __future__ import annotations

import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram rd"),
    ("dram__bytes_write.sum", "dram wr"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "regs"),
    ("smsp__inst_executed.sum", "warp insts"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
    ("lts__t_bytes.sum", "L2 bytes"),
]


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    cols = [(hdr.index(m), label, units[hdr.index(m)]) for m, label in METRICS if m in hdr]
    name_i = hdr.index("Kernel Name")
    print(f"# ncu summary: `{path}`\n")
    print("| kernel | " + " | ".join(f"{l} ({u})" if u else l for _, l, u in cols) + " |")
    print("|---|" + "---|" * len(cols))
    for r in rows[2:]:
        name = r[name_i].split("(")[0][:48]
        print(f"| `{name}` | " + " | ".join(r[i][:12] for i, _, _ in cols) + " |")


if __name__ == "__main__":
    main(sys.argv[1])
