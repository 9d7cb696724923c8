cd $GRAFT_REPO_ROOT
B=paper_2511_12201_b200/lib/libomnisparse_base.so
timeout 900 python -m pytest -q -x tests/test_gpu_prefill.py tests/test_gpu_kernel_variants.py -k "not db and not sp and not pp" 2>&1 | tail -2
for i in 1 2 3; do
OMNI_LIBRARY=$B python profiles/k4_time.py 65536 6
python profiles/k4_time.py 65536 6
done
for i in 1 2; do
OMNI_LIBRARY=$B python profiles/k4_time.py 32768 6
python profiles/k4_time.py 32768 6
done
