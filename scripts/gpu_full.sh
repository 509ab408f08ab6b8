# full GPU validation + benches for every single-GPU config
python -c "from paper_1002_4464_b200 import _build; _build.build()"
timeout 1200 python -m pytest tests/ -m gpu -x -q > gpurun_out/gpu_tests_all.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/gpu_tests_all.log
timeout 600 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo c2 rc=$?
for d in uniform gaussian bucket_sorted staggered sorted zero det_duplicates; do
  timeout 600 python bench.py --workload C3 --dist $d --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3_$d.json 2>&1; echo c3 $d rc=$?
done
timeout 900 python bench.py --workload C4 --steps 5 --warmup 3 > gpurun_out/bench_c4.json 2>&1; echo c4 rc=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2>&1; echo ref rc=$?
python - <<'PY'
import json, glob
for f in sorted(glob.glob('gpurun_out/bench_*.json')):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, f"{d['value']/1e9:.3f} G{d['unit']}", f"{d['ms_per_step']:.3f} ms", d.get('clocks', {}).get('sm_mhz'), (d.get('roofline') or {}).get('frac'))
    except Exception as e:
        print(f, 'ERR', e)
PY
