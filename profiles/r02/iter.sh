# Kernel iteration on the GPU box (repo root):  bash profiles/r02/iter.sh TAG [stress]
# full GPU suite, a short bench line (no CPU baseline / sweep), and optionally
# the config-C per-tile timeline of k_splat_tc (profiles/r02/stress.py).
TAG=$1
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_$TAG.txt
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/tests_$TAG.txt 2>&1
echo "tests rc=$?" >> gpurun_out/tests_$TAG.txt
tail -4 gpurun_out/tests_$TAG.txt
timeout 600 python bench.py --no-cpu-baseline --no-sweep --steps 20 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
echo "bench rc=$?"; grep -v Warn gpurun_out/bench_$TAG.err | tail -3
tail -1 gpurun_out/bench_$TAG.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({k: d[k] for k in ('value','fps','stage_ms')})); print('roofline', d['roofline']['frac'], 'e2e', d.get('e2e',{}).get('value'), 'parity', (d.get('parity') or {}).get('ok'))" || tail -5 gpurun_out/bench_$TAG.json
if [ "$2" = "stress" ]; then
  timeout 300 python profiles/r02/stress.py 2000000 1440 1080 > gpurun_out/stress_$TAG.txt 2>&1
  echo "stress rc=$?"; head -8 gpurun_out/stress_$TAG.txt; grep -E "per tile|period|mean:" gpurun_out/stress_$TAG.txt
fi
