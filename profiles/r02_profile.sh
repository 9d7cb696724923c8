#!/bin/bash
# Round-2 measurement pass (run on the GPU box from the repo root):
# bench line, K5 / K7 ncu --set full captures, and the launch list of one
# prefill step. Outputs land in gpurun_out/ (summaries are copied to profiles/).
set -x
mkdir -p gpurun_out
python bench.py > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err
ncu --set full --clock-control none --import-source on -k regex:"dq_kernel|dkv2_kernel|bwd_prep" -s 3 -c 3 \
    -o gpurun_out/r02_k5 -f python profiles/ncu_backward_driver.py > gpurun_out/r02_k5.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"decode_partial_tma" -s 1 -c 1 \
    -o gpurun_out/r02_k7 -f python profiles/ncu_decode_driver.py > gpurun_out/r02_k7.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/r02_launches.csv python bench.py --steps 2 --warmup 1 --no-dense --no-knobs --no-e2e \
    --no-cpu --no-train --no-decode > /dev/null 2>&1
ls -la gpurun_out
