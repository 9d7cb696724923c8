# compute-sanitizer memcheck over the GPU parity tests (one B200; exact
# allocation bounds via PYTORCH_NO_CUDA_MEMORY_CACHING=1) plus a positive control.
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
mkdir -p gpurun_out
timeout 300 compute-sanitizer --tool memcheck --print-limit 5 python profiles/sanitizer/oob_control.py > gpurun_out/mc_control.log 2>&1
for f in test_gpu_edges test_gpu_backward test_gpu_decode test_gpu_prefill test_gpu_api; do
  timeout 900 compute-sanitizer --tool memcheck --print-limit 20 --log-file gpurun_out/mc_$f.log \
    python -m pytest tests/$f.py -q -p no:cacheprovider > gpurun_out/mc_${f}_py.log 2>&1
  echo "$f rc=$? $(tail -1 gpurun_out/mc_${f}_py.log) | $(grep 'ERROR SUMMARY' gpurun_out/mc_$f.log)"
done
