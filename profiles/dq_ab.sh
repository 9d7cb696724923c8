cd $GRAFT_REPO_ROOT
V=paper_2511_12201_b200/lib/libomnisparse_variants.so
timeout 600 python -m pytest -q -x tests/test_gpu_backward.py 2>&1 | tail -2
OMNI_LIBRARY=$V OMNI_DQ_QT=1 timeout 300 python -m pytest -q -x tests/test_gpu_backward.py 2>&1 | tail -1
for i in 1 2; do
OMNI_LIBRARY=$V OMNI_DQ_QT=0 python profiles/bwd_time.py
OMNI_LIBRARY=$V OMNI_DQ_QT=1 python profiles/bwd_time.py
done
OMNI_LIBRARY=$V OMNI_DQ_QT=0 ncu --metrics gpu__time_duration.sum --kernel-name-base demangled -k regex:"dq_kernel|dkv2|bwd_prep" -c 6 python profiles/bwd_time.py 2>&1 | grep -E "dq_kernel|dkv2|bwd_prep|duration" | head -12
OMNI_LIBRARY=$V OMNI_DQ_QT=1 ncu --metrics gpu__time_duration.sum --kernel-name-base demangled -k regex:"dq_kernel|dkv2|bwd_prep" -c 6 python profiles/bwd_time.py 2>&1 | grep -E "dq_kernel|dkv2|bwd_prep|duration" | head -12
