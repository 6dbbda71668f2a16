"""Key metrics of a one-kernel `ncu --set full` report (for profiles/*/ *_summary.txt)."""
import csv
import io
import subprocess
import sys

DETAILS = ("Duration", "Compute (SM) Throughput", "Memory Throughput", "DRAM Throughput",
           "L2 Hit Rate", "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy",
           "Issue Slots Busy", "Warp Cycles Per Issued Instruction", "No Eligible", "Grid Size",
           "Block Size", "Dynamic Shared Memory Per Block")
RAW = ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
       "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
       "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "launch__registers_per_thread",
       "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
       "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
       "sm__inst_executed_pipe_tensor_subpipe_imma.avg.pct_of_peak_sustained_active",
       "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active",
       "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
       "lts__t_sectors_srcunit_tex.avg.pct_of_peak_sustained_elapsed")


def ncu(rep, page):
    return subprocess.run(["ncu", "-i", rep, "--page", page, "--csv"], capture_output=True,
                          text=True, check=True).stdout


def main(rep, title):
    out = [title, ""]
    rows = list(csv.reader(io.StringIO(ncu(rep, "details"))))
    h = rows[0]
    for r in rows[1:]:
        d = dict(zip(h, r))
        if d.get("Metric Name") in DETAILS:
            out.append(f"{d['Section Name']:<36}{d['Metric Name']:<40}{d['Metric Value']:>14} {d['Metric Unit']}")
    out.append("")
    raw = list(csv.reader(io.StringIO(ncu(rep, "raw"))))
    for k, unit, v in zip(raw[0], raw[1], raw[2]):
        if k in RAW:
            out.append(f"{k:<80}{v:>16} {unit}")
    stalls = [(k, float(v)) for k, v in zip(raw[0], raw[2])
              if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")
              and v.replace(".", "").isdigit()]
    tot = sum(v for _, v in stalls) or 1.0
    out.append("")
    out.append("warp-state samples (share):")
    for k, v in sorted(stalls, key=lambda x: -x[1])[:8]:
        out.append(f"  {k.replace('smsp__pcsamp_warps_issue_stalled_', ''):<28}{100 * v / tot:6.1f} %")
    print("\n".join(out))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
