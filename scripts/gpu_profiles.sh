# Round-2 profiles: launch lists (per-launch time + DRAM bytes) of the bench commands and one
# ncu --set full capture of one sort per workload (C4 headline, C2), summarised into
# profiles/ncu_full_summary.json (roofline.traffic / roofline.limiter of bench.py).
set -x
OUT=gpurun_out/prof
mkdir -p $OUT
python -c "from paper_1002_4464_b200 import _build; _build.build()"
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 900 ncu --metrics $M --clock-control none --csv --log-file $OUT/launches_c4.csv python bench.py --workload C4 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-extras > $OUT/launches_c4.log 2>&1
timeout 600 ncu --metrics $M --clock-control none --csv --log-file $OUT/launches_c2.csv python bench.py --workload C2 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-extras > $OUT/launches_c2.log 2>&1
python scripts/launch_summary.py $OUT/launches_c4.csv > $OUT/launches_c4_summary.txt
python scripts/launch_summary.py $OUT/launches_c2.csv > $OUT/launches_c2_summary.txt
K='regex:k_(local_sort|segment_sort|relocate|sample_index|scan|s4_|bucket_tiers|child_desc)'
timeout 1500 ncu --set full --clock-control none --import-source on -k "$K" -o $OUT/full_c4 python bench.py --workload C4 --ncu-one > $OUT/full_c4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "$K" -o $OUT/full_c2 python bench.py --workload C2 --ncu-one > $OUT/full_c2.log 2>&1
python scripts/ncu_summary.py $OUT/ncu_full_summary.json C4=$OUT/full_c4.ncu-rep C2=$OUT/full_c2.ncu-rep > $OUT/ncu_full.txt
# source-level (SASS) view of the hot CTA sorts, then drop the reports (gpurun returns <= 64 MiB)
for r in c4 c2; do
  ncu -i $OUT/full_$r.ncu-rep --page details --csv > $OUT/details_$r.csv 2>/dev/null
  ncu -i $OUT/full_$r.ncu-rep --page source --csv --print-source sass -k regex:k_local_sort > $OUT/source_local_sort_$r.csv 2>/dev/null
  gzip -f $OUT/source_local_sort_$r.csv $OUT/details_$r.csv
done
rm -f $OUT/*.ncu-rep $OUT/launches_c4.csv.gz
gzip -f $OUT/launches_c4.csv $OUT/launches_c2.csv
ls -la $OUT
