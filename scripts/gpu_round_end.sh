# round-end validation on one B200: build, full GPU suite, smoke, the default bench line,
# the reference arm, profiles (launch lists + ncu --set full summaries)
mkdir -p gpurun_out
python -c "from paper_1002_4464_b200 import _build; _build.build()"
timeout 1800 python -m pytest tests/ -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/gpu_tests.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/smoke.log
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?; tail -3 gpurun_out/bench.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref rc=$?
bash scripts/gpu_profiles.sh > gpurun_out/prof_run.log 2>&1; echo profiles rc=$?
