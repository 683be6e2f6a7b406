"""Key counters of one `ncu --set full` capture (.ncu-rep) as a markdown table.

    python tools/ncu_keymetrics.py gpurun_out/m2l_full.ncu-rep [more.ncu-rep ...]

Reads the raw page (`ncu -i X --page raw --csv`) and prints duration, DRAM bytes,
pipe utilisation (FP64 / DMMA / LSU / XU), occupancy, shared-memory bank conflicts
and the top warp-stall reasons: the numbers DESIGN.md and profiles/ quote.
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput % (SOL)"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe active % (of active cycles)"),
    ("sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active", "DMMA subpipe % (of active)"),
    ("smsp__pipe_tensor_subpipe_dmma_cycles_active.avg", "DMMA subpipe active cycles (avg/SMSP)"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) pipe %"),
    ("smsp__inst_executed.sum", "warp instructions executed"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("sm__cycles_active.avg", "SM active cycles (avg)"),
    ("gpc__cycles_elapsed.max", "elapsed cycles"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "smem load bank conflicts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "smem store bank conflicts"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [(dict(zip(hdr, r)), dict(zip(hdr, units))) for r in rows[2:]]


def main():
    for path in sys.argv[1:]:
        for vals, units in raw(path):
            print(f"### {vals.get('Kernel Name', '?')[:120]}\n\nsource: `{path}`\n")
            print("| counter | value | unit |\n|---|---|---|")
            for k, label in KEYS:
                if k in vals:
                    print(f"| {label} (`{k}`) | {vals[k]} | {units.get(k, '')} |")
            st = [(k, float(v)) for k, v in vals.items()
                  if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("_per_issue_active.ratio")
                  and v not in ("", "n/a")]
            st.sort(key=lambda x: -x[1])
            print("\ntop stall reasons (warps per issue): " + ", ".join(
                f"{k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')} "
                f"{v:.2f}" for k, v in st[:6]) + "\n")


if __name__ == "__main__":
    main()
