timeout 900 python -m pytest tests -m "gpu" -x -q 2>&1 | tail -2
for c in 1 4; do for pr in fp64 fp32; do
timeout 300 python bench.py --config $c --precision $pr --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());k=d['kernel_ms'];print('cfg',$c,'$pr',round(d['ms_per_step'],4),round(d['pressure_only']['ms_per_step'],4),round(d['e2e']['ms_per_step'],4),{a:round(b,4) for a,b in k.items()})"
done; done
nproc; timeout 300 python bench.py --impl reference --steps 5 --warmup 1 2>&1 | tail -1 | cut -c1-300
