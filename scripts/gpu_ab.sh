# rebuild, full GPU suite, then an A/B of build variants on C2 and C3 (args: variant specs for ab_variants.py)
python -c "from paper_1002_4464_b200 import _build; _build.build()"
timeout 1200 python -m pytest tests/ -m gpu -x -q > gpurun_out/gpu_tests_all.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/gpu_tests_all.log
timeout 900 python scripts/ab_variants.py "$@" 2>&1 | tee gpurun_out/ab_c2.log
timeout 900 python scripts/ab_variants.py "$@" -- --workload C3 2>&1 | tee gpurun_out/ab_c3.log
