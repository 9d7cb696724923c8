# A/B of two autograd.py variants on the same box (C4 fwd+bwd timing)
make -C paper_2511_12201_b200/csrc -j8 > /dev/null
for r in 1 2; do
for v in base new; do
  cp profiles/micro/ab/autograd_$v.py paper_2511_12201_b200/autograd.py
  echo "$v $(timeout 200 python profiles/bwd_time.py 2>&1 | tail -1)"
done
done
