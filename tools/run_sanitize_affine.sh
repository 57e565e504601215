# compute-sanitizer over the affine K1/K2 form (kernel-level tests + connector scenarios that use it)
mkdir -p gpurun_out
for tool in memcheck synccheck; do
  echo "== $tool"
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 7 python -m pytest -q -x -p no:cacheprovider -m gpu \
     tests/test_gpu_kernels.py -k "affine or unit_kernel" 2>&1 | grep -E "passed|failed|ERROR SUMMARY" | tail -2
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 7 python -m pytest -q -x -p no:cacheprovider -m gpu \
     tests/test_gpu_pipeline.py 2>&1 | grep -E "passed|failed|ERROR SUMMARY" | tail -2
done
