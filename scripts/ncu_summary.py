"""Summarise an ncu --set full report (raw page CSV) for the committed profiles/."""
import csv
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_issued.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic", "launch__grid_size", "launch__block_size",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_bytes.sum", "smsp__sass_inst_executed_op_global_red.sum", "smsp__sass_inst_executed_op_global_atom.sum",
        "smsp__sass_inst_executed_op_shared_atom.sum", "sm__cycles_elapsed.avg.per_second",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__t_requests_pipe_lsu_mem_global_op_atom.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_red.sum",
        "smsp__inst_executed_op_global_red.sum"]


def main(rep):
    raw = subprocess.check_output(["ncu", "-i", rep, "--page", "raw", "--csv"], text=True)
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        print("kernel:", d.get("Kernel Name", "?")[:110])
        for k in KEYS:
            if k in d:
                print(f"  {k:70s} {d[k]:>20s} {units[hdr.index(k)]}")
        try:  # derived: shared-memory wavefronts per SM clock (the smem pipe serves 1 / clk / SM)
            wf = float(d["l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"].replace(",", ""))
            t = float(d["gpu__time_duration.sum"].replace(",", "")) * {"ms": 1e-3, "us": 1e-6, "ns": 1e-9}.get(
                units[hdr.index("gpu__time_duration.sum")].replace("second", "s").replace("msecond", "ms"), 1e-3)
            f = float(d["sm__cycles_elapsed.avg.per_second"].replace(",", "")) * (
                1e9 if "G" in units[hdr.index("sm__cycles_elapsed.avg.per_second")] else 1.0)
            n_sm = 148
            print(f"  derived: smem wavefronts / SM / clk {wf / (t * f * n_sm):.3f} (1.0 = smem pipe peak)")
        except (KeyError, ValueError):
            pass
        st = [(k, d[k]) for k in hdr if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")]
        vals = [(k.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(v.replace(",", "") or 0)) for k, v in st
                if v not in ("", "n/a")]
        tot = sum(v for _, v in vals) or 1.0
        print("  stall samples (top):", ", ".join(f"{k} {100 * v / tot:.1f}%" for k, v in sorted(vals, key=lambda kv: -kv[1])[:8]))


if __name__ == "__main__":
    main(sys.argv[1])
