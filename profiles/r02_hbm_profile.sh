#!/bin/bash
# K1 / K2 (HBM-bound selection kernels): A/B timing + one ncu --set full capture each.
mkdir -p gpurun_out
python profiles/k2_time.py > gpurun_out/k2_time.json 2>&1
OMNI_QSCORE_F64=1 python profiles/k2_time.py > gpurun_out/k2_time_f64.json 2>&1
ncu --set full --clock-control none --import-source on -k regex:"q_score_stream" -s 2 -c 1 \
    -o gpurun_out/r02_k2 -f python profiles/k2_time.py > gpurun_out/r02_k2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"kv_probe_stream" -s 2 -c 1 \
    -o gpurun_out/r02_k1 -f python profiles/k2_time.py > gpurun_out/r02_k1.log 2>&1
cat gpurun_out/k2_time.json gpurun_out/k2_time_f64.json
