#!/usr/bin/env python
"""Summarise ncu output for profiles/: the launch list (per-kernel device time
and share of the step) and the key counters of a `--set full` capture.

    python scripts/ncu_summary.py --launches gpurun_out/launches.csv --rep gpurun_out/prof.ncu-rep > profiles/rNN/ncu_summary.md
"""
import argparse
import collections
import csv
import io
import subprocess

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "lts__t_sector_hit_rate.pct", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "derived__memory_l1_wavefronts_shared_excessive",
    "l1tex__data_pipe_tc_wavefronts_mem_shared.sum", "gpc__cycles_elapsed.max.per_second",
]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.OrderedDict()
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0]
        v = float(r[vi].replace(",", ""))
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "nsecond": 1e-3}.get(r[ui], 1e-3)
        agg.setdefault(name, []).append(v * scale)
    return agg


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[h.index("Kernel Name")].split("(")[0]}
        for k in KEYS:
            if k in h:
                d[k] = (r[h.index(k)], units[h.index(k)])
        res.append(d)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--rep")
    ap.add_argument("--skip-names", default="synth_kernel,qsplit_kernel")
    a = ap.parse_args()
    if a.launches:
        agg = launches(a.launches)
        skip = set(a.skip_names.split(","))
        tot = sum(sum(v) for k, v in agg.items() if k not in skip)
        print("## Launch list (ncu gpu__time_duration.sum, --clock-control none; cold-cache, serialised)\n")
        print("| kernel | launches | mean us | share of step |")
        print("|---|---|---|---|")
        for k, v in agg.items():
            if k in skip:
                continue
            print(f"| `{k}` | {len(v)} | {sum(v) / len(v):.1f} | {100 * sum(v) / tot:.1f}% |")
        print()
    if a.rep:
        print("## `ncu --set full` counters (per launch)\n")
        for d in full(a.rep):
            print(f"### `{d.pop('kernel')}`\n")
            for k, (v, u) in d.items():
                print(f"- {k}: {v} {u}")
            print()


if __name__ == "__main__":
    main()
