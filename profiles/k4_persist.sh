cd $GRAFT_REPO_ROOT
V=paper_2511_12201_b200/lib/libomnisparse_variants.so
for n in 32768 65536; do
for i in 1 2; do
OMNI_LIBRARY=$V OMNI_FWD_FAST=0 python profiles/k4_time.py $n 6
OMNI_LIBRARY=$V OMNI_FWD_PERSIST_SAFE=1 python profiles/k4_time.py $n 6
done
done
