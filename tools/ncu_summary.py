"""Summarise ncu reports / launch lists into the numbers the roofline story uses.

usage:
  python tools/ncu_summary.py full  report.ncu-rep [...]      > profiles/rNN_ncu_full_summary.txt
  python tools/ncu_summary.py launches launches.csv "<what ran>" > profiles/rNN_launches_summary.txt
"""
import csv
import subprocess
import sys
from collections import defaultdict

KEYS = [
    ("Kernel Name", ""), ("launch__grid_size", ""), ("launch__block_size", ""),
    ("launch__registers_per_thread", ""), ("gpu__time_duration.sum", ""),
    ("dram__bytes_read.sum", ""), ("dram__bytes_write.sum", ""),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", ""),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe (DMMA) active"),
    ("sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active", "DMMA issue"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 (DFMA) pipe"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", ""),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", ""),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", ""),
    ("lts__t_bytes.sum", "L2 traffic"),
    ("sm__cycles_elapsed.avg", ""), ("smsp__cycles_active.avg", ""),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe (tcgen05) active, elapsed"),
    ("sm__pipe_tensor_subpipe_imma_cycles_active_realtime.avg", "int8 (IMMA) subpipe cycles"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate"),
    ("l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem reads by the tensor core"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots active"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("gpc__cycles_elapsed.avg.per_second", "SM clock"),
]


def full(paths):
    for path in paths:
        out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(out.splitlines()))
        hdr, units = rows[0], rows[1]
        print(f"## {path.split('/')[-1]}")
        for vals in rows[2:]:
            for k, note in KEYS:
                if k in hdr:
                    i = hdr.index(k)
                    print(f"  {k:<78} {vals[i]:>22} {units[i]:<10} {note}")
            print()


def launches(path, what):
    """Per-kernel totals of gpu__time_duration.sum (and DRAM bytes when the list carries them)."""
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr = rows[hi]
    ki, mi, vi, ui = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    scale = {"ns": 1.0, "nsecond": 1.0, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6,
             "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    agg = defaultdict(lambda: defaultdict(float))
    count = defaultdict(int)
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0][:80]
        v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        agg[name][r[mi]] += v
        if r[mi] == "gpu__time_duration.sum":
            count[name] += 1
    tot = sum(a["gpu__time_duration.sum"] for a in agg.values())
    has_dram = any("dram__bytes_read.sum" in a for a in agg.values())
    print("ncu --metrics gpu__time_duration.sum" + (",dram__bytes_read.sum,dram__bytes_write.sum" if has_dram else "")
          + " --clock-control none (cold-cache, serialised launches)")
    print(f"workload: {what}\n")
    print(f"{'total ms':>10} {'share':>7} {'launches':>9} " + (f"{'GB/launch':>10} {'TB/s':>6} " if has_dram else "")
          + " kernel")
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1]["gpu__time_duration.sum"]):
        t, c = a["gpu__time_duration.sum"], max(count[k], 1)
        extra = ""
        if has_dram:
            by = a["dram__bytes_read.sum"] + a["dram__bytes_write.sum"]
            extra = f"{by / c / 1e9:10.3f} {by / t / 1e3 if t else 0:6.2f} "
        print(f"{t / 1e6:10.3f} {100 * t / tot:6.2f}% {count[k]:9d} {extra} {k}")


if __name__ == "__main__":
    if sys.argv[1] == "full":
        full(sys.argv[2:])
    else:
        launches(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "")
