mkdir -p gpurun_out
T=${1:-g18}
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/tests_$T.txt 2>&1
echo "tests rc=$?" >> gpurun_out/tests_$T.txt
grep -E "FAILED|Error|passed|failed" gpurun_out/tests_$T.txt | head -20
timeout 400 python bench.py --no-cpu-baseline --no-sweep --steps 10 --warmup 3 > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err
echo "bench rc=$?"; tail -2 gpurun_out/bench_$T.err | grep -v Warn
tail -1 gpurun_out/bench_$T.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['fps'], d['stage_ms'], d['roofline']['frac'], d.get('e2e',{}).get('value'), d['gpu_launches'])"
