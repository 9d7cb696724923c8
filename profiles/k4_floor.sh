cd $GRAFT_REPO_ROOT
V=paper_2511_12201_b200/lib/libomnisparse_variants.so
for n in 32768 65536; do
OMNI_LIBRARY=$V OMNI_FWD_IMPL=single python profiles/k4_time.py $n -1,6
done
