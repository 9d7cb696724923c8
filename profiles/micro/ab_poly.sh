for r in 1 2 3; do for v in base new; do
  cp profiles/micro/ab/lib_$v.so paper_2511_12201_b200/lib/libomnisparse.so
  echo "$v $(timeout 200 python profiles/k4_time.py 65536 4,6 2>&1 | tail -1)"
done; done
