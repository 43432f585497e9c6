mkdir -p gpurun_out
T=${1:-g8}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_configs.py -m gpu -x -q -p no:cacheprovider -k "config or binning or tile or ties or random" > gpurun_out/tests_$T.txt 2>&1
echo "tests rc=$?" >> gpurun_out/tests_$T.txt
grep -E "FAILED|Error|passed|failed" gpurun_out/tests_$T.txt | head -10
timeout 300 python profiles/r02/stress.py 2000000 1440 1080 > gpurun_out/stress_$T.txt 2>&1
head -8 gpurun_out/stress_$T.txt; grep "mean" gpurun_out/stress_$T.txt
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 60 -c 14 --csv --log-file gpurun_out/launches_$T.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-sweep > /dev/null 2>&1
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/launches_$T.csv')))
hdr=[i for i,r in enumerate(rows) if 'Kernel Name' in r][0]
h=rows[hdr]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
for r in rows[hdr+1:]:
    print(r[ki][:50], r[vi])
PY
