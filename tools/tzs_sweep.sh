# Spread tile depth sweep (diagnostic): step time and spread/combine kernel_ms per ESP_TILE_ZS
for c in 1 4; do for z in 0 4 8 16 24 32 48; do
[ $c = 1 ] && [ $z -gt 16 ] && continue
ESP_TILE_ZS=$z timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-near 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());k=d['kernel_ms'];print('cfg',$c,'tzs',$z,round(d['ms_per_step'],4),round(d['pressure_only']['ms_per_step'],4),{a:round(b,4) for a,b in k.items() if 'spread' in a or 'comb' in a})"
done; done
