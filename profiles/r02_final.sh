#!/bin/bash
# Round-2 closing measurement: full GPU suite, smoke, default bench line, the
# reference arm, K1/K2 ncu captures of the shipped kernels.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?"; tail -1 gpurun_out/smoke.log
timeout 400 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc $?"
timeout 400 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc $?"
bash profiles/r02_hbm_profile.sh
# K4 (the dominant kernel) at HEAD: one full ncu capture of the fast kernel (3rd launch)
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"sparse_fwd_kernel" -s 2 -c 1 \
    -o gpurun_out/r02_k4 -f python profiles/ncu_k4_driver.py > gpurun_out/r02_k4.log 2>&1; echo "ncu k4 rc $?"
