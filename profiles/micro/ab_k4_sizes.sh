# K4 A/B at 64K and 32K (prebuilt base / new libraries, same box)
for r in 1 2 3; do for v in base new; do
  cp profiles/micro/ab/lib_$v.so paper_2511_12201_b200/lib/libomnisparse.so
  echo "$v 64K $(timeout 200 python profiles/k4_time.py 65536 6 2>&1 | tail -1) 32K $(timeout 200 python profiles/k4_time.py 32768 6 2>&1 | tail -1)"
done; done
