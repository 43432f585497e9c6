mkdir -p gpurun_out
T=${1:-g20}
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/tests_$T.txt 2>&1
echo "tests rc=$?" >> gpurun_out/tests_$T.txt
grep -E "FAILED|Error|passed|failed" gpurun_out/tests_$T.txt | head -20
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 60 -c 13 --csv --log-file gpurun_out/launches_$T.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-sweep > /dev/null 2>&1
python profiles/r02/launch_list.py gpurun_out/launches_$T.csv
timeout 400 python bench.py --no-cpu-baseline --no-sweep --steps 10 --warmup 3 > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err
tail -1 gpurun_out/bench_$T.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['fps']['feature_splat'], d['stage_ms']['blend_kernel'], d.get('e2e',{}).get('value'))"
