#!/bin/bash
# Full GPU suite + default bench line + K1/K2 ncu captures (round 2, after the K1/K2 stream kernels).
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/pytest_gpu.log
timeout 400 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc $?"
bash profiles/r02_hbm_profile.sh
