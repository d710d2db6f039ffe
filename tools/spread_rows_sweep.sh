# Spread warp-row granularity sweep (diagnostic): kernel_ms per ESP_SPREAD_ROWS
for c in 1 4; do for r in 4; do
ESP_SPREAD_ROWS=$r timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-near 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());k=d['kernel_ms'];print('cfg',$c,'rows',$r,round(d['ms_per_step'],4),round(d['pressure_only']['ms_per_step'],4),{a:round(b,4) for a,b in k.items() if 'spread' in a or 'comb' in a})"
done; done
