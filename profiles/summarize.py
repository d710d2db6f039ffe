"""Summarise an ncu report (``--set full``) into a markdown table.

Usage: python profiles/summarize.py gpurun_out/prof_<tag>.ncu-rep > profiles/<tag>.md

Per kernel: duration, DRAM bytes, IPC, occupancy, shared-memory wavefronts
(actual / ideal), executed warp instructions, FP64 pipe share and the top
warp-stall reasons from the source page.
"""

import collections
import csv
import subprocess
import sys


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def raw_metrics(rep):
    rows = list(csv.reader(ncu(rep, "--page", "raw", "--csv").splitlines()))
    hdr, units, data = rows[0], rows[1], rows[2:]
    want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum",
            "dram__bytes_write.sum", "smsp__inst_executed.sum",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
            "sm__warps_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
            "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "launch__registers_per_thread", "launch__grid_size"]
    idx = {w: hdr.index(w) for w in want if w in hdr}
    out = []
    for r in data:
        out.append({w: (r[i], units[i]) for w, i in idx.items()})
    return out


def stalls(rep, kernel_regex):
    rows = list(csv.reader(ncu(rep, "--page", "source", "--csv", "-k",
                               "regex:" + kernel_regex).splitlines()))
    starts = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"]
    if not starts:
        return {}
    hdr = rows[starts[0] + 1]
    end = starts[1] if len(starts) > 1 else len(rows)
    data = rows[starts[0] + 2:end]
    cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    tot = collections.Counter()
    allsamp = 0.0
    si = hdr.index("Warp Stall Sampling (All Samples)")
    for r in data:
        try:
            allsamp += float(r[si] or 0)
        except ValueError:
            continue
        for c in cols:
            tot[c] += float(r[hdr.index(c)] or 0)
    return {k: v / max(allsamp, 1) for k, v in tot.most_common(5)}


def main(rep):
    print(f"# ncu summary: `{rep}`\n")
    print("| kernel | ms | DRAM rd MB | DRAM wr MB | warp inst (M) | smem wavefronts (M) "
          "| warps active % | issue active % | FP64 pipe % | regs |")
    print("|---|---|---|---|---|---|---|---|---|---|")
    kernels = raw_metrics(rep)
    for k in kernels:
        def g(name, scale=1.0):
            v = k.get(name)
            if not v:
                return "-"
            try:
                x = float(v[0].replace(",", ""))
            except ValueError:
                return v[0]
            unit = v[1]
            if name.startswith("dram__bytes"):
                x *= {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(unit, 1.0)
                return f"{x:.2f}"
            if name == "gpu__time_duration.sum":      # always milliseconds in the table
                x *= {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}.get(unit, 1.0)
                return f"{x:.4f}"
            return f"{x * scale:.2f}"
        name = k["Kernel Name"][0].split("(")[0][:48]
        fp = g("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active")
        if fp == "-":
            fp = g("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active")
        print(f"| {name} | {g('gpu__time_duration.sum')} | {g('dram__bytes_read.sum')} | "
              f"{g('dram__bytes_write.sum')} | {g('smsp__inst_executed.sum', 1e-6)} | "
              f"{g('l1tex__data_pipe_lsu_wavefronts_mem_shared.sum', 1e-6)} | "
              f"{g('sm__warps_active.avg.pct_of_peak_sustained_active')} | "
              f"{g('smsp__issue_active.avg.pct_of_peak_sustained_active')} | {fp} | "
              f"{g('launch__registers_per_thread')} |")
    print()
    seen = set()
    for k in kernels:
        base = k["Kernel Name"][0].split("(")[0].split("<")[0].replace("void ", "").split("::")[-1]
        if base in seen:
            continue
        seen.add(base)
        st = stalls(rep, base)
        if st:
            print(f"- `{base}` top stall reasons: " +
                  ", ".join(f"{n.replace('stall_', '')} {100 * v:.0f}%" for n, v in st.items()))


if __name__ == "__main__":
    main(sys.argv[1])
