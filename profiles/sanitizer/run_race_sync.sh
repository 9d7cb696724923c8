# compute-sanitizer racecheck (shared-memory hazards) and synccheck (barrier
# misuse) over the mbarrier / TMEM kernels K4, K5, K7 at small shapes (r02).
mkdir -p gpurun_out
for tool in racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 --log-file gpurun_out/san_$tool.log \
    python profiles/sanitizer/small_kernels.py > gpurun_out/san_${tool}_py.log 2>&1
  echo "$tool rc=$? $(tail -1 gpurun_out/san_${tool}_py.log) | $(grep 'ERROR SUMMARY\|RACECHECK SUMMARY' gpurun_out/san_$tool.log)"
done
