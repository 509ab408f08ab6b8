python -c "from paper_1002_4464_b200 import _build; _build.build()"
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 ncu --cache-control none --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file gpurun_out/launches_warm.csv $B > /dev/null 2>&1; echo ncu1 rc=$?
python scripts/launch_summary.py gpurun_out/launches_warm.csv > gpurun_out/launch_summary_warm.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_s4 -s 8 -c 3 -o gpurun_out/prof_s4 $B > gpurun_out/ncu_s4.log 2>&1; echo ncu2 rc=$?
