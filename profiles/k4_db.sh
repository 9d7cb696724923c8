cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest -q -x tests/test_gpu_kernel_variants.py -k db 2>&1 | tail -3
timeout 300 python profiles/k4_pp_cmp.py 65536 single,db,single,db
timeout 300 python profiles/k4_pp_cmp.py 32768 single,db
timeout 300 python profiles/k4_pp_cmp.py 65536 single,db:4,db:8,db:0
