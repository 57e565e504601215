# compute-sanitizer over the single-pass q8 encode (cooperative launch) and the K3 round change
mkdir -p gpurun_out
T="tests/test_codec.py -m gpu -k (matches_oracle or every_lane or batch_pipeline) tests/test_gpu_kernels.py -k (keys or hash)"
for tool in memcheck synccheck racecheck; do
  echo "== $tool"
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 7 python -m pytest -q -x -p no:cacheprovider \
     tests/test_codec.py -m gpu -k "matches_oracle or every_lane or batch_pipeline" 2>&1 | grep -E "passed|failed|ERROR SUMMARY|RACECHECK SUMMARY|error" | tail -3
done
echo "== K3 memcheck"
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 7 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_kernels.py -m gpu -k "hash or key" 2>&1 | grep -E "passed|failed|ERROR SUMMARY" | tail -2
