TAG=$1; shift
for lib in "$@"; do
  if [ "$lib" = default ]; then unset ESP_LIB; else export ESP_LIB=$lib; fi
  timeout 600 python bench.py --precision fp32 --steps 20 --warmup 3 --no-cpu-baseline --no-near > gpurun_out/ab32_${TAG}.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/ab32_${TAG}.json'));print('$lib', round(d['ms_per_step'],3), d['kernel_ms']['gather'], d['kernel_ms']['ifft_x'])"
done
