cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest -q -x tests/test_gpu_kernel_variants.py -k sp 2>&1 | tail -3
OMNI_VARIANTS_LIBRARY=$PWD/paper_2511_12201_b200/lib/libomnisparse_wpf.so timeout 900 python -m pytest -q -x tests/test_gpu_kernel_variants.py -k single 2>&1 | tail -3
timeout 300 python profiles/k4_pp_cmp.py 65536 single,single@wpf,sp,single,single@wpf,sp
timeout 300 python profiles/k4_pp_cmp.py 32768 single,single@wpf,sp,single,single@wpf
