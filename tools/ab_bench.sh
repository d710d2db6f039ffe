# A/B: short config-4 bench per library variant.  Usage: bash tools/ab_bench.sh <tag> <lib1> [lib2 ...]
# ("default" = the in-tree library).  Prints force+pressure ms and the per-kernel profile.
TAG=$1; shift
mkdir -p gpurun_out
for lib in "$@"; do
  if [ "$lib" = default ]; then unset ESP_LIB; else export ESP_LIB=$lib; fi
  timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-near > gpurun_out/ab_${TAG}_$(basename $lib .so).json 2>gpurun_out/ab_${TAG}.err
  python -c "import json,sys;d=json.load(open('gpurun_out/ab_${TAG}_$(basename $lib .so).json'));print('$lib', round(d['ms_per_step'],3), round(d['pressure_only']['ms_per_step'],3), {k:round(v,3) for k,v in d['kernel_ms'].items()})" || tail -5 gpurun_out/ab_${TAG}.err
done
