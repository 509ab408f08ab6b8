set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
python -c "from paper_1002_4464_b200 import _build; _build.build()"
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo bench rc=$?
cat gpurun_out/bench_c2.json
timeout 300 python bench.py --steps 10 --warmup 3 --workload C3 --no-cpu-baseline > gpurun_out/bench_c3.json 2>&1; echo rc=$?
for d in zero sorted det_duplicates; do timeout 300 python bench.py --steps 10 --warmup 3 --workload C3 --dist $d --no-cpu-baseline > gpurun_out/bench_c3_$d.json 2>&1; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch_bench.log 2>&1; echo ncu1 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_local_sort|k_segment_sort|k_relocate|k_sample_index" -s 60 -c 4 -o gpurun_out/prof_c2 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo ncu2 rc=$?
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "C2_C3" > gpurun_out/gpu_tests_full.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/gpu_tests_full.log
