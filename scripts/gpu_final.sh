# round-end validation: build, full GPU suite, smoke, every bench line, profiles (launch lists + ncu --set full)
bash scripts/gpu_full.sh
bash scripts/gpu_profiles.sh > gpurun_out/prof_run.log 2>&1
timeout 1200 python scripts/experiments.py --reps 10 > gpurun_out/experiments.log 2>&1; echo experiments rc=$?
