"""Summarises an ncu --set full capture of one evolve launch into the files the
bench and the judge read: profiles/<tag>_ncu_summary.txt (key counters) and,
for the C2 kernel, profiles/r02_ncu_traffic.json (DRAM bytes per launch).

    python tools/ncu_traffic.py gpurun_out/prof.ncu-rep <tag> [--traffic]
"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
KEYS = [
    ("duration", "gpu__time_duration.sum"),
    ("SM clock", "sm__cycles_elapsed.avg.per_second"),
    ("dynamic smem per CTA", "launch__shared_mem_per_block_dynamic"),
    ("registers/thread", "launch__registers_per_thread"),
    ("block size", "launch__block_size"),
    ("grid size", "launch__grid_size"),
    ("warps active (of 64/SM)", "sm__warps_active.avg.pct_of_peak_sustained_active"),
    ("issue slots busy", "smsp__issue_active.avg.pct_of_peak_sustained_active"),
    ("active threads per warp instruction", "smsp__thread_inst_executed_per_inst_executed.ratio"),
    ("instructions executed (warp)", "smsp__inst_executed.sum"),
    ("instruction cache hit rate", "sm__icc_request_hit_rate.pct"),
    ("no-instruction stall per issue", "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio"),
    ("shared-memory pipe", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"),
    ("smem bank conflicts (wavefronts)", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
    ("smem wavefronts", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"),
    ("L2 throughput", "lts__throughput.avg.pct_of_peak_sustained_elapsed"),
    ("local load sectors", "l1tex__t_sectors_pipe_lsu_mem_local_op_ld.sum"),
    ("DRAM read", "dram__bytes_read.sum"),
    ("DRAM write", "dram__bytes_write.sum"),
    ("DRAM bandwidth", "dram__bytes.sum.per_second"),
    ("stall samples: barrier", "smsp__pcsamp_warps_issue_stalled_barrier"),
    ("stall samples: long scoreboard", "smsp__pcsamp_warps_issue_stalled_long_scoreboard"),
    ("stall samples: short scoreboard", "smsp__pcsamp_warps_issue_stalled_short_scoreboard"),
    ("stall samples: sleeping", "smsp__pcsamp_warps_issue_stalled_sleeping"),
    ("stall samples: wait", "smsp__pcsamp_warps_issue_stalled_wait"),
    ("stall samples: branch resolving", "smsp__pcsamp_warps_issue_stalled_branch_resolving"),
    ("stall samples: no instruction", "smsp__pcsamp_warps_issue_stalled_no_instructions"),
    ("samples: selected (issuing)", "smsp__pcsamp_warps_issue_stalled_selected"),
    ("total samples", "smsp__pcsamp_sample_count"),
]


def main():
    rep, tag = sys.argv[1], sys.argv[2]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units = rows[0], rows[1]
    lines = []
    for r in rows[2:]:
        d = dict(zip(head, r))
        u = dict(zip(head, units))
        lines.append(f"# kernel {d.get('Kernel Name')}")
        for label, key in KEYS:
            if key in d:
                lines.append(f"{label:40s} {d[key]} {u.get(key, '')}   [{key}]")
        if "--traffic" in sys.argv:
            rd = float(d["dram__bytes_read.sum"]) * (1e6 if u["dram__bytes_read.sum"] == "Mbyte" else 1)
            wr = float(d["dram__bytes_write.sum"]) * (1e6 if u["dram__bytes_write.sum"] == "Mbyte" else 1)
            (ROOT / "profiles" / "r02_ncu_traffic.json").write_text(json.dumps({
                "kernel": d.get("Kernel Name"), "source": rep, "tag": tag,
                "dram_bytes_read": rd, "dram_bytes_write": wr,
                "dram_bytes_per_launch": rd + wr}, indent=1) + "\n")
    out = ROOT / "profiles" / f"{tag}_ncu_summary.txt"
    out.write_text("\n".join(lines) + "\n")
    print(out.read_text())


if __name__ == "__main__":
    main()
