# rebuild, quick parity subset, bench C2, per-kernel launch list
python -c "from paper_1002_4464_b200 import _build; _build.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2.json 2>&1; echo bench rc=$?
python - <<'PY'
import json; d=json.loads(open('gpurun_out/bench_c2.json').read().strip().splitlines()[-1])
print('value', d['value']/1e9, 'Gkeys/s  ms', d['ms_per_step'])
for k,v in d['steps_breakdown'].items(): print('  ', k, v)
PY
