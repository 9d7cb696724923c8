# A/B of two prebuilt variants (library + Python binding) on the same box
for r in 1 2 3 4; do
for v in base new; do
  cp profiles/micro/ab/lib_$v.so paper_2511_12201_b200/lib/libomnisparse.so
  cp profiles/micro/ab/ops_$v.py paper_2511_12201_b200/ops.py
  cp profiles/micro/ab/_lib_$v.py paper_2511_12201_b200/_lib.py
  echo "$v $(timeout 200 python profiles/k4_time.py 65536 6 2>&1 | tail -1)"
done
done
