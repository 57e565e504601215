mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_memo.py tests/test_gpu_connector.py -q -x --timeout 200 -p no:cacheprovider > gpurun_out/pytest_memo.log 2>&1; tail -2 gpurun_out/pytest_memo.log
timeout 200 python tools/bench_lookup.py > gpurun_out/lookup.json 2>gpurun_out/lookup.err; cat gpurun_out/lookup.json; tail -2 gpurun_out/lookup.err
timeout 300 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/lookup_launches.csv python tools/bench_lookup.py > /dev/null 2>&1
python - <<'PY'
import csv, collections
rows=[r for r in csv.reader(open('gpurun_out/lookup_launches.csv')) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value'); ii=h.index('ID')
for r in rows[-12:]: print(r[ii], r[ki][:60], r[vi])
PY
