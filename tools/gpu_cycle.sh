set -o pipefail
TAG=$1
timeout 700 python -m pytest tests -m "gpu" -x -q 2>&1 | tail -4
timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -3 gpurun_out/bench_$TAG.err
python -c "import json;d=json.load(open('gpurun_out/bench_$TAG.json'));print(d['ms_per_step'], d['pressure_only']['ms_per_step'], d['e2e']['ms_per_step'], d['kernel_ms'])"
python bench.py --profile-only --steps 3 --warmup 1 && ncu --set full --clock-control none --import-source on -k regex:"k_gather_warp|k_spread_tiles|k_combine" -s 3 -c 3 -o gpurun_out/prof_$TAG python bench.py --profile-only --steps 3 --warmup 1 > gpurun_out/ncu_$TAG.log 2>&1; tail -1 gpurun_out/ncu_$TAG.log
