python -c "from paper_1002_4464_b200 import _build; _build.build()"
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_local_sort|k_segment_sort|k_relocate_grouped|k_sample_index_tma|k_s4_" -c 12 -o gpurun_out/prof_sort $B > gpurun_out/ncu_sort.log 2>&1; echo ncu rc=$?
