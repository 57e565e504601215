# compute-sanitizer memcheck over the whole GPU suite except the full-size
# tests (test_gpu_fullscale: 10 GiB page images, hours under the tool), the
# two-rank torchrun test and the pipeline timing assertions (the tool slows
# kernels by orders of magnitude).
mkdir -p gpurun_out
for tool in ${TOOLS:-memcheck synccheck initcheck racecheck}; do
  echo "== $tool"
  timeout 2400 compute-sanitizer --tool $tool --error-exitcode 7 python -m pytest -q -p no:cacheprovider -m gpu \
     tests --ignore=tests/test_gpu_fullscale.py --ignore=tests/test_gpu_multirank.py \
     -k "not beats_blocking and not warm_backend" > gpurun_out/sanall_$tool.log 2>&1
  echo "rc=$?"; grep -E "passed|failed|ERROR SUMMARY" gpurun_out/sanall_$tool.log | tail -3
done
