set -o pipefail
TAG=$1
timeout 900 python -m pytest tests -m "gpu and slow" -x -q 2>&1 | tail -6
for c in 3 4; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${TAG}_cfg$c.json 2> gpurun_out/bench_${TAG}_cfg$c.err; tail -2 gpurun_out/bench_${TAG}_cfg$c.err
  python -c "import json;d=json.load(open('gpurun_out/bench_${TAG}_cfg$c.json'));print($c, d['value'], d['ms_per_step'], d['pressure_only']['ms_per_step'], d['e2e']['ms_per_step'], d['kernel_ms'])"
done
