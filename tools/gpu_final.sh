timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
bash tools/gpu_record.sh r1s 1 fp64
for c in 3 4; do timeout 900 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_r1s_cfg$c.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/bench_r1s_cfg$c.json'));print($c, d['ms_per_step'], d['pressure_only']['ms_per_step'], d.get('near_field'), d.get('analytic_forces',{}).get('ms_per_step'), d.get('fp32_mode',{}).get('ms_per_step'))"; done
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_r1s_ref.json 2>/dev/null; cut -c1-300 gpurun_out/bench_r1s_ref.json
