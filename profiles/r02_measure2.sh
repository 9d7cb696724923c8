#!/bin/bash
# Parity report + variants + reference arm + per-kernel launch list (our kernels only).
set -x
mkdir -p gpurun_out
OMNI_PARITY_OUT=gpurun_out/r02_parity.json python -m pytest tests/test_gpu_parity_report.py -q -p no:cacheprovider > gpurun_out/r02_parity.log 2>&1
python -m pytest tests/test_gpu_kernel_variants.py tests/test_gpu_select_parity.py -q -p no:cacheprovider > gpurun_out/r02_variants.log 2>&1
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02_ref.json 2> gpurun_out/r02_ref.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:omni -c 60 --csv \
    --log-file gpurun_out/r02_launches.csv python bench.py --steps 2 --warmup 1 --no-dense --no-knobs --no-e2e \
    --no-cpu --no-train --no-decode > /dev/null 2>&1
tail -3 gpurun_out/r02_parity.log gpurun_out/r02_variants.log; tail -c 600 gpurun_out/r02_ref.json
