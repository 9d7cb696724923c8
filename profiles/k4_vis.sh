cd $GRAFT_REPO_ROOT
V=paper_2511_12201_b200/lib/libomnisparse_variants.so
timeout 900 python -m pytest -q -x tests/test_gpu_prefill.py tests/test_gpu_api.py tests/test_gpu_kernel_variants.py tests/test_gpu_edges.py 2>&1 | tail -2
for i in 1 2; do python profiles/k4_time.py 65536 6; python profiles/k4_time.py 32768 6; done
OMNI_LIBRARY=$V OMNI_FWD_IMPL=single python profiles/k4_cta_timing.py 65536
OMNI_LIBRARY=$V OMNI_FWD_IMPL=single python profiles/k4_cta_timing.py 32768
