# compute-sanitizer over the pitched host-tier copies (csrc/ce_copy.cpp): the
# piece-copy tests, the pipeline tests, connector scenarios that move the
# host tier layer by layer (evicting traces, two batches in flight)
mkdir -p gpurun_out
T="tests/test_ce_copy.py tests/test_gpu_pipeline.py tests/test_gpu_connector.py"
K="(ce_copy or staging_peak or layerwise or warm or sc_partial_match or sc_random_trace_evicting or sc_pipelined_two_in_flight or two_batches) and not beats_blocking"
for tool in memcheck initcheck racecheck synccheck; do
  echo "== $tool"
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 7 python -m pytest -q -x -p no:cacheprovider -m gpu \
     $T -k "$K" > gpurun_out/san_$tool.log 2>&1
  echo "rc=$?"; grep -E "passed|failed|ERROR SUMMARY|RACECHECK SUMMARY" gpurun_out/san_$tool.log | tail -3
done
