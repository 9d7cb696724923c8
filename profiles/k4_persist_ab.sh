cd $GRAFT_REPO_ROOT
for i in 1 2 3; do
OMNI_FWD_PERSIST=0 python profiles/k4_time.py 65536 6; OMNI_FWD_PERSIST=1 python profiles/k4_time.py 65536 6
OMNI_FWD_PERSIST=0 python profiles/k4_time.py 32768 6; OMNI_FWD_PERSIST=1 python profiles/k4_time.py 32768 6
done
OMNI_FWD_PERSIST=1 timeout 900 python -m pytest -q -x tests/test_gpu_prefill.py tests/test_gpu_api.py tests/test_gpu_edges.py tests/test_gpu_select_parity.py tests/test_gpu_kernel_variants.py 2>&1 | tail -2
