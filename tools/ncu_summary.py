"""Summarise an ncu report (every kernel in it): key metrics and the warp-stall breakdown.

    python tools/ncu_summary.py report.ncu-rep [more.ncu-rep ...]
"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg", "sm__cycles_elapsed.avg.per_second",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "smsp__inst_executed_op_shared_ld.sum", "launch__grid_size", "launch__block_size",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed_op_shared_atom.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum",
        "lts__t_sectors_op_atom.sum", "lts__t_sectors_op_red.sum", "smsp__thread_inst_executed_per_inst_executed.ratio",
        "lts__t_sectors_op_write.sum", "lts__t_sectors_op_read.sum"]


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    u = dict(zip(hdr, units))
    res = []
    for vals in rows[2:]:
        d = dict(zip(hdr, vals))
        print(f"== {path}: {d.get('Kernel Name', '?')[:100]}")
        res.append(summ(d, u))
    return res


def summ(d, u):
    out = {}
    for k in KEYS:
        if k in d:
            out[k] = (d[k], u.get(k, ""))
            print(f"{k:70s} {d[k]:>20s} {u.get(k, '')}")
    print("-- stalls (warps per issue-active cycle)")
    st = []
    for k, v in d.items():
        if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
            try:
                st.append((float(v), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    for v, k in sorted(st, reverse=True)[:12]:
        print(f"  {k:40s} {v:.3f}")
    return out


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
