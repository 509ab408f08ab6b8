python -c "from paper_1002_4464_b200 import _build; _build.build()"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:k_(local_sort|segment_sort)<.int.0,' -c 2 -o gpurun_out/prof_sort2 python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_sort.log 2>&1; echo ncu rc=$?
