python -c "from paper_1002_4464_b200 import _build; _build.build()"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:k_(relocate|sample_index)<.int.0,|k_scan' -c 5 -o gpurun_out/prof_misc python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_misc.log 2>&1; echo ncu rc=$?
