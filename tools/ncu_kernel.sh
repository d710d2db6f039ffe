# One ncu --set full capture of the first launch of a kernel (regex) in a
# config-4 profile step, then key metrics as CSV.  Usage:
#   bash tools/ncu_kernel.sh <tag> <kernel-regex> [ENV=val ...]
TAG=$1; KR=$2; shift 2
mkdir -p gpurun_out
env "$@" timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$KR" -s 1 -c 1 \
  -o gpurun_out/k_$TAG python bench.py --profile-only --steps 2 --warmup 1 > gpurun_out/k_$TAG.log 2>&1
tail -2 gpurun_out/k_$TAG.log
ncu -i gpurun_out/k_$TAG.ncu-rep --page raw --csv > gpurun_out/k_$TAG.raw.csv 2>/dev/null
python - "$TAG" <<'PY'
import csv, sys
tag = sys.argv[1]
rows = list(csv.reader(open(f"gpurun_out/k_{tag}.raw.csv")))
hdr, units, vals = rows[0], rows[1], rows[2:]
keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
        "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_sectors_srcunit_tex_op_write.sum",
        "smsp__average_warp_latency_issue_stalled_long_scoreboard", "launch__registers_per_thread",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smsp__inst_executed.sum"]
for v in vals:
    for k in keys:
        if k in hdr:
            i = hdr.index(k); print(f"  {k} = {v[i]} {units[i]}")
PY
