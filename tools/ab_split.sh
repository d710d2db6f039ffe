# A/B of the first force range of the host-buffer step (percent of the charges). Usage: bash tools/ab_split.sh
for v in 45 50 55 60 65 70; do
  ESP_HOST_SPLIT=$v timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-near 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('split $v', round(d['ms_per_step'],3), round(d['e2e']['ms_per_step'],3))"
done
