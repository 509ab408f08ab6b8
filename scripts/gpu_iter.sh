# one iteration: rebuild, GPU parity tests, C2 bench with step breakdown, C4 bench, C2 launch list
bash scripts/gpu_quick.sh
timeout 900 python bench.py --workload C4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.json 2>&1
python -c "import json; d=json.loads(open('gpurun_out/bench_c4.json').read().strip().splitlines()[-1]); print('C4', d['value']/1e9, d['ms_per_step'])"
mkdir -p gpurun_out/prof2
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/prof2/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/prof2/launches.csv
