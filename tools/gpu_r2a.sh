# Round-2 first GPU call: box facts, GPU tests, smoke, config-4 bench, reference arm, launch list.
TAG=${1:-r2a}
mkdir -p gpurun_out
(nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv; nproc; free -g) > gpurun_out/box_$TAG.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_$TAG.log 2>&1; tail -3 gpurun_out/pytest_$TAG.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -c 600 gpurun_out/bench_$TAG.err
python -c "import json;d=json.load(open('gpurun_out/bench_$TAG.json'));print(d['config']['workload'], d['ms_per_step'], d['pressure_only']['ms_per_step'], d['e2e']['ms_per_step'], d['clocks'], d['kernel_ms'], d['cpu_baseline'])"
timeout 1500 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_${TAG}_ref.json 2> gpurun_out/bench_${TAG}_ref.err; cut -c1-400 gpurun_out/bench_${TAG}_ref.json; tail -c 400 gpurun_out/bench_${TAG}_ref.err
