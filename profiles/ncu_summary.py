"""Summarise an ncu report (run here, no GPU): per-kernel duration, DRAM bytes and
throughput, occupancy, issue activity and the top warp-stall reasons.

    python profiles/ncu_summary.py gpurun_out/prof.ncu-rep [out.txt]
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration_us", 1e-3),
    ("dram__bytes_read.sum", "dram_read_MB", 1e-6),
    ("dram__bytes_write.sum", "dram_write_MB", 1e-6),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct_peak", 1),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_pct_peak", 1),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_pct", 1),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved_occupancy_pct", 1),
    ("launch__registers_per_thread", "regs", 1),
    ("launch__grid_size", "grid", 1),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem_bank_conflicts", 1),
    ("smsp__inst_executed.sum", "warp_instructions", 1),
    # pipe utilisation: FMA (fp32 incl. FFMA2), FP64, ALU, LSU, tensor
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "pipe_fma_pct", 1),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "pipe_fma_cycles_pct", 1),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "pipe_fp64_pct", 1),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "pipe_fp64_cycles_pct", 1),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "pipe_alu_pct", 1),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "pipe_lsu_pct", 1),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "pipe_tensor_pct", 1),
    ("lts__t_sectors_srcunit_tex_op_read.sum", "l2_read_sectors", 1),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return hdr, units, rows[2:]


def conv(v, unit, scale_key):
    try:
        x = float(v.replace(",", ""))
    except ValueError:
        return None
    u = unit.strip()
    mult = {"ns": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6, "nsecond": 1,
            "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(u, 1)
    return x * mult


def main():
    rep = sys.argv[1]
    hdr, units, rows = raw(rep)
    lines = []
    for row in rows:
        d = dict(zip(hdr, row))
        u = dict(zip(hdr, units))
        name = d.get("Kernel Name", "?")
        lines.append(f"== {name[:90]}")
        for k, label, sc in KEYS:
            if k in d:
                v = conv(d[k], u[k], sc)
                if v is not None and label in ("duration_us", "dram_read_MB", "dram_write_MB"):
                    v = v * sc
                lines.append(f"   {label:26s} {v if v is None else round(v, 3)}")
        st = [(k, float(d[k])) for k in d if k.startswith("smsp__pcsamp_warps_issue_stalled_")
              and not k.endswith("_not_issued") and d[k] not in ("", "n/a")]
        tot = sum(v for _, v in st) or 1
        top = sorted(st, key=lambda kv: -kv[1])[:6]
        lines.append("   stalls: " + ", ".join(f"{k.split('stalled_')[1]} {100 * v / tot:.0f}%" for k, v in top))
    txt = "\n".join(lines)
    print(txt)
    if len(sys.argv) > 2:
        open(sys.argv[2], "w").write(txt + "\n")


if __name__ == "__main__":
    main()
