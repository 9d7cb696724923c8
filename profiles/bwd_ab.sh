cd $GRAFT_REPO_ROOT
B=paper_2511_12201_b200/lib/libomnisparse_base.so
timeout 900 python -m pytest -q -x tests/test_gpu_backward.py 2>&1 | tail -2
for i in 1 2 3; do
OMNI_LIBRARY=$B python profiles/bwd_only_time.py 32768
python profiles/bwd_only_time.py 32768
done
