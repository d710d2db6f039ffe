# Record run (one GPU): ncu launch list + full capture of our kernels for one
# step, per-stage DRAM traffic -> profiles/dram_traffic.json, then the bench
# line (which reads it).  Usage: bash gpu_record.sh <tag> [config] [precision]
TAG=$1
CFG=${2:-4}
PREC=${3:-fp64}
ARGS="--config $CFG --precision $PREC"
timeout 300 python bench.py $ARGS --profile-only --steps 2 --warmup 1 || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py $ARGS --profile-only --steps 2 --warmup 1 > /dev/null 2>&1
KREGEX='regex:k_(bin|spread|combine|x_|y_|z_|gather|scale)'
NK=$(python -c "print({3: 11, 4: 12}.get($CFG, 9))")   # our kernels per step (skip the first step; config 4: the x pass is two launches)
timeout 900 ncu --set full --clock-control none --import-source on -k "$KREGEX" -s $NK -c $NK -o gpurun_out/prof_$TAG python bench.py $ARGS --profile-only --steps 2 --warmup 1 > gpurun_out/ncu_$TAG.log 2>&1; tail -1 gpurun_out/ncu_$TAG.log
W=$(python -c "from paper_2601_00161_b200 import workloads; print(workloads.CONFIGS[$CFG]['name'])")
python profiles/traffic.py gpurun_out/prof_$TAG.ncu-rep $W $PREC && cp profiles/dram_traffic.json gpurun_out/dram_traffic.json
python profiles/summarize.py gpurun_out/prof_$TAG.ncu-rep > gpurun_out/ncu_$TAG.md
# keep what travels back small (gpurun copies at most 64 MiB)
[ $(stat -c %s gpurun_out/prof_$TAG.ncu-rep) -gt 25000000 ] && rm -f gpurun_out/prof_$TAG.ncu-rep
timeout 900 python bench.py $ARGS --steps 100 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -2 gpurun_out/bench_$TAG.err
python -c "import json;d=json.load(open('gpurun_out/bench_$TAG.json'));print(d['ms_per_step'], d['pressure_only']['ms_per_step'], d['e2e']['ms_per_step'], d['roofline'], d.get('roofline_smem'), d['kernel_ms'])"
