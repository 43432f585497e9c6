# Development iteration on the GPU box (repo root):  bash profiles/r02/gpu_dev.sh TAG [pytest -k expr]
TAG=$1
SEL=${2:-"test_persistent or test_random_scenes or test_fused_decode or test_config_a or test_frame_pipeline or test_empty or test_k_equals or test_fixup_overflow or test_query_pipeline_vs or test_eager"}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_$TAG.txt
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "$SEL" -p no:cacheprovider > gpurun_out/tests_$TAG.txt 2>&1
echo "tests rc=$?" >> gpurun_out/tests_$TAG.txt
tail -15 gpurun_out/tests_$TAG.txt
timeout 300 python bench.py --no-cpu-baseline --no-sweep --steps 10 --warmup 3 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
echo "bench rc=$?"; tail -3 gpurun_out/bench_$TAG.err
tail -1 gpurun_out/bench_$TAG.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['fps'], d['stage_ms'], d['roofline']['frac'], d.get('e2e',{}).get('value'), d.get('parity',{}).get('ok'))" || tail -5 gpurun_out/bench_$TAG.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 60 -c 60 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-sweep > /dev/null 2>&1
python profiles/launch_summary.py gpurun_out/launches_$TAG.csv 2 > gpurun_out/sum_$TAG.txt 2>&1
head -30 gpurun_out/sum_$TAG.txt
