# compute-sanitizer memcheck / synccheck over every covered path, racecheck per path (slow)
mkdir -p gpurun_out/san
python -c "from paper_1002_4464_b200 import _build; _build.build()"
for tool in memcheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize.py > gpurun_out/san/$tool.log 2>&1; echo $tool rc=$?
done
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python scripts/sanitize.py --big cta_pair_buckets > gpurun_out/san/memcheck_big.log 2>&1; echo memcheck_big rc=$?
for c in small_2k_plan one_tile_fused_8_9 cta_pair_sublists nested_step9 pairs keys64 multi_gpu_emulated_p4 typed_float host_pipeline step9_tiers; do
  timeout 700 compute-sanitizer --tool racecheck --racecheck-report hazard --error-exitcode 9 python scripts/sanitize.py $c > gpurun_out/san/racecheck_$c.log 2>&1; echo racecheck $c rc=$?
done
grep -H "ERROR SUMMARY\|RACECHECK SUMMARY\|WRONG\|: ok" gpurun_out/san/*.log
