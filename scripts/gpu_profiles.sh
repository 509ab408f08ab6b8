# Round profiles: launch list of the bench command + one ncu --set full capture of each hot kernel.
set -x
mkdir -p gpurun_out/prof
python -c "from paper_1002_4464_b200 import _build; _build.build()"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/prof/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/prof/launches_bench.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/prof/launches_c4.csv python bench.py --workload C4 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/prof/launches_c4_bench.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:k_(local_sort|segment_sort|relocate|relocate_grouped|sample_index|sample_index_tma)<.int.0,|k_scan|k_s4_' -c 16 -o gpurun_out/prof/full python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/prof/full.log 2>&1
python scripts/ncu_summary.py gpurun_out/prof/full.ncu-rep gpurun_out/prof/ncu_full_summary.json > gpurun_out/prof/ncu_full.txt
python scripts/launch_summary.py gpurun_out/prof/launches.csv > gpurun_out/prof/launches_summary.txt
python scripts/launch_summary.py gpurun_out/prof/launches_c4.csv > gpurun_out/prof/launches_c4_summary.txt
ls -la gpurun_out/prof
