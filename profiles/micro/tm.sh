make -C paper_2511_12201_b200/csrc -j8 >/dev/null
for t in 0 1 2 4; do echo "trace=$t $(OMNI_FWD_TRACE=$t timeout 100 python profiles/k4_time.py 65536 4 2>&1 | tail -1)"; done > gpurun_out/tm.txt
cat gpurun_out/tm.txt
