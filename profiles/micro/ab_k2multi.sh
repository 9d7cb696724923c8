for r in 1 2; do for v in "$@"; do
  cp profiles/micro/ab/lib_$v.so paper_2511_12201_b200/lib/libomnisparse.so
  echo "$v $(timeout 200 python profiles/k2_time.py 2>&1 | tail -1)"
done; done
