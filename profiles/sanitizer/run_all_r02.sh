# compute-sanitizer memcheck, racecheck and synccheck over the mbarrier / TMEM
# kernels at small shapes (round 2, after the K1/K2 stream kernels and the dq
# Q-in-TMEM change).
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 --log-file gpurun_out/san_$tool.log \
    python profiles/sanitizer/small_kernels.py > gpurun_out/san_${tool}_py.log 2>&1
  echo "$tool rc=$? $(tail -1 gpurun_out/san_${tool}_py.log) | $(grep 'ERROR SUMMARY\|RACECHECK SUMMARY' gpurun_out/san_$tool.log)"
done
