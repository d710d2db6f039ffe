# Quick iteration on one GPU: targeted tests + a short config-4 bench (no CPU legs, no near field).
# Usage: bash tools/gpu_iter.sh <tag> [pytest -k expr]
TAG=${1:-it}; K=${2:-"config or fused or slab or graph or radix"}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_config4.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x -k "$K" > gpurun_out/pytest_$TAG.log 2>&1; tail -5 gpurun_out/pytest_$TAG.log
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-near > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -c 1500 gpurun_out/bench_$TAG.err
python -c "import json;d=json.load(open('gpurun_out/bench_$TAG.json'));print(d['ms_per_step'], d['pressure_only']['ms_per_step'], d['e2e']['ms_per_step'], d.get('fp32_mode',{}).get('ms_per_step'), d.get('analytic_forces',{}).get('ms_per_step'), d['clocks']);print(d['kernel_ms'])"
