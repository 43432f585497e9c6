mkdir -p gpurun_out
T=${1:-g23}
STRESS_TIMEOUT=20 timeout 200 python profiles/r02/stress.py 20000 512 384 2000000 1440 1080 > gpurun_out/stress_$T.txt 2>&1
echo "stress rc=$?"; grep -E "ok G|HANG|total|per tile|mean:" gpurun_out/stress_$T.txt | cut -c1-200
for i in 1 2 3; do
timeout 400 python bench.py --no-cpu-baseline --no-sweep --no-e2e --steps 10 --warmup 3 > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err
tail -1 gpurun_out/bench_$T.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['fps']['feature_splat'], d['stage_ms']['blend_kernel'])"
done
