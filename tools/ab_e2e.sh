# A/B of the host-buffer (e2e) step over ESP_HOST_CHUNKS values.
# Usage: bash tools/ab_e2e.sh <tag> 1 2 4
TAG=$1; shift
mkdir -p gpurun_out
for c in "$@"; do
  ESP_HOST_CHUNKS=$c timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-near > gpurun_out/e2e_${TAG}_$c.json 2>gpurun_out/e2e_${TAG}.err
  python -c "import json;d=json.load(open('gpurun_out/e2e_${TAG}_$c.json'));print('chunks $c', round(d['ms_per_step'],3), d['e2e'])" || tail -5 gpurun_out/e2e_${TAG}.err
done
