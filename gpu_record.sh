TAG=$1
timeout 600 python bench.py --steps 50 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -2 gpurun_out/bench_$TAG.err
python bench.py --profile-only --steps 2 --warmup 1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --profile-only --steps 2 --warmup 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_gather_warp|k_spread_tiles|k_combine|k_scale_reduce|k_bin_canon" -s 5 -c 5 -o gpurun_out/prof_$TAG python bench.py --profile-only --steps 2 --warmup 1 > gpurun_out/ncu_$TAG.log 2>&1; tail -1 gpurun_out/ncu_$TAG.log
