"""Key counters of ncu --set full captures (profiles tool).
    python tools/ncu_digest.py gpurun_out/X.ncu-rep [...]"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "time"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe active %"),
    ("sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.sum.pct_of_peak_sustained_elapsed", "UTCHMMA bf16 % of peak"),
    ("sm__inst_executed_pipe_uniform_realtime.avg.pct_of_peak_sustained_elapsed", "uniform pipe %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem LSU wavefronts %"),
    ("l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum.per_second", "TMA load bytes/s"),
    ("derived__lts__lts2xbar_bytes.sum.per_second", "L2->SM bytes/s"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput %"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
]


def digest(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        kname = r[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        print(f"== {path}: {kname[:110]}")
        for key, label in KEYS:
            if key in hdr:
                i = hdr.index(key)
                print(f"   {label:28s} {r[i]:>14s} {units[i]}")


for p in sys.argv[1:]:
    digest(p)
