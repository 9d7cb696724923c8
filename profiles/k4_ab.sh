cd $GRAFT_REPO_ROOT
V=paper_2511_12201_b200/lib/libomnisparse_variants.so
timeout 600 python -m pytest -q tests/test_gpu_kernel_variants.py -k "single" 2>&1 | tail -2
for i in 1 2 3; do
python profiles/k4_time.py 65536 6
OMNI_LIBRARY=$V OMNI_FWD_IMPL=single python profiles/k4_time.py 65536 6
done
