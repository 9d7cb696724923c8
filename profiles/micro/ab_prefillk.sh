for r in 1 2; do for v in base new; do
  cp profiles/micro/ab/lib_$v.so paper_2511_12201_b200/lib/libomnisparse.so
  echo "$v $(timeout 200 python profiles/prefill_kernels.py 65536 2>/dev/null | tail -1)"
done; done
