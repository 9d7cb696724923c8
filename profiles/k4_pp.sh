cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest -q -x tests/test_gpu_kernel_variants.py -k pp 2>&1 | tail -3
timeout 300 python profiles/k4_pp_cmp.py 65536 single,pp,single,pp
timeout 300 python profiles/k4_pp_cmp.py 32768 single,pp
timeout 300 python profiles/k4_pp_cmp.py 65536 single:-1,pp:-1
