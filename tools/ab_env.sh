# A/B over environment switches: short config-4 bench per setting.
# Usage: bash tools/ab_env.sh <tag> "<ENV=val ...>" ["<ENV=val ...>" ...]   ("-" = defaults)
TAG=$1; shift
mkdir -p gpurun_out
i=0
for envs in "$@"; do
  i=$((i+1))
  [ "$envs" = "-" ] && envs=""
  env $envs timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-near > gpurun_out/abe_${TAG}_$i.json 2>gpurun_out/abe_${TAG}_$i.err
  python -c "import json;d=json.load(open('gpurun_out/abe_${TAG}_$i.json'));print('[$envs]', round(d['ms_per_step'],3), round(d['pressure_only']['ms_per_step'],3), round(d['e2e']['ms_per_step'],3), {k:round(v,3) for k,v in d['kernel_ms'].items()})" || tail -5 gpurun_out/abe_${TAG}_$i.err
done
