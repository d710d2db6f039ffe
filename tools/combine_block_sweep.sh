for c in 1 4; do for b in 32 64 128; do
ESP_COMBINE_B=$b timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-near 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());k=d['kernel_ms'];print('cfg',$c,'B',$b,round(d['ms_per_step'],4),{a:round(b,4) for a,b in k.items() if 'comb' in a})"
done; done
