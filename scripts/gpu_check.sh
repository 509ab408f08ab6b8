# rebuild, full GPU suite, smoke, default bench line (C4 headline + extras)
mkdir -p gpurun_out
python -c "from paper_1002_4464_b200 import _build; _build.build()"
timeout 1800 python -m pytest tests/ -m gpu -x -q ${PYTEST_ARGS} > gpurun_out/gpu_tests.log 2>&1; echo tests rc=$?; tail -5 gpurun_out/gpu_tests.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo smoke rc=$?; tail -2 gpurun_out/smoke.log
timeout 1200 python bench.py ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?; tail -5 gpurun_out/bench.err
python - <<'PY'
import json
try:
    d = json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1])
    print('headline', d['value'] / 1e9, d['unit'], d['ms_per_step'], 'ms', 'verified', d.get('verified'))
    print('roofline', d.get('roofline'))
    print('e2e', d.get('e2e'))
    for k in ('c2', 'c3', 'c5_base'):
        if k in d:
            v = d[k]
            print(k, {kk: vv for kk, vv in v.items() if kk not in ('steps_breakdown', 'per_dist')})
    if 'c3' in d:
        print({k: round(v['value'] / 1e9, 2) for k, v in d['c3']['per_dist'].items()})
    print(json.dumps(d.get('steps_breakdown'), indent=0)[:3000])
    print('cpu', d.get('cpu_baseline'))
except Exception as e:
    print('bench parse error', e)
PY
