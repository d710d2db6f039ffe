# End-of-round check (one GPU): tests, smoke, bench lines for configs 1/3/4, reference arm.
# Usage: bash tools/gpu_final.sh <tag>
TAG=${1:-final}
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py --steps 50 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
python -c "import json;d=json.load(open('gpurun_out/bench_$TAG.json'));print(1, d['ms_per_step'], d['pressure_only']['ms_per_step'], d['e2e']['ms_per_step'], d['near_field']['ms_per_step'], d['near_field']['coulomb_step_graphed']['ms_per_step'], d['clocks'], d['kernel_ms'])"
for c in 3 4; do timeout 900 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${TAG}_cfg$c.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/bench_${TAG}_cfg$c.json'));print($c, d['ms_per_step'], d['pressure_only']['ms_per_step'], d['e2e']['ms_per_step'], d['near_field']['ms_per_step'], d['near_field']['coulomb_step_graphed']['ms_per_step'], d.get('analytic_forces',{}).get('ms_per_step'), d.get('fp32_mode',{}).get('ms_per_step'), d['kernel_ms'])"; done
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_${TAG}_ref.json 2>/dev/null; cut -c1-200 gpurun_out/bench_${TAG}_ref.json
