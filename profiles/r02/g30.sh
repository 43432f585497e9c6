# Verification of a restored tree: full GPU suite, smoke, default bench line.
mkdir -p gpurun_out
T=${1:-g30}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_$T.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/tests_$T.txt 2>&1
echo "tests rc=$?" >> gpurun_out/tests_$T.txt
grep -E "FAILED|Error|passed|failed" gpurun_out/tests_$T.txt | head -20
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.txt 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke_$T.txt
timeout 900 python bench.py > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err
echo "bench rc=$?"; tail -3 gpurun_out/bench_$T.err
tail -1 gpurun_out/bench_$T.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d.get('fps'), d.get('stage_ms'), d['roofline']['frac'], d.get('e2e',{}).get('value'), d.get('parity',{}).get('ok'))" || tail -5 gpurun_out/bench_$T.json
