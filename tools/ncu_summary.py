"""Summarise an ncu --set full capture of k_gcm into profiles/<name>.json.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep profiles/kgcm_ncu_summary.json
"""
import csv
import io
import json
import subprocess
import sys

WANT = {
    "gpu__time_duration.sum": "duration_ms",
    "dram__bytes_read.sum": "dram_bytes_read",
    "dram__bytes_write.sum": "dram_bytes_write",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum": "smem_wavefronts",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum": "smem_bank_conflicts",
    "l1tex__throughput.avg.pct_of_peak_sustained_active": "l1tex_pct",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active": "alu_pipe_pct",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active": "lsu_pipe_pct",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active": "fma_pipe_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "launch__registers_per_thread": "registers_per_thread",
    "smsp__inst_executed.sum": "warp_instructions",
    "sm__cycles_active.avg": "sm_cycles_active",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
}
SCALE = {"Mbyte": 1e6, "Gbyte": 1e9, "Kbyte": 1e3, "byte": 1, "ms": 1, "us": 1e-3, "ns": 1e-6}


def main(rep: str, out: str, note: str = "") -> None:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units = rows[0], rows[1]
    launches = []
    kcol = head.index("Kernel Name") if "Kernel Name" in head else None
    for r in rows[2:]:
        rec = {"kernel": r[kcol] if kcol is not None else None}
        for name, unit, val in zip(head, units, r):
            if name in WANT:
                try:
                    v = float(val.replace(",", ""))
                except ValueError:
                    continue
                key = WANT[name]
                if key.startswith("dram_bytes"):
                    v *= SCALE.get(unit, 1)
                if key == "duration_ms" and unit in SCALE:
                    v *= SCALE[unit]
                rec[key] = v
        launches.append(rec)
    summary = {"source": rep, "note": note, "launches": launches}
    if launches:
        summary.update({k: launches[0][k] for k in ("dram_bytes_read", "dram_bytes_write") if k in launches[0]})
    json.dump(summary, open(out, "w"), indent=1)
    print(json.dumps(summary)[:400])


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "")
