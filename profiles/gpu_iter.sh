# usage: bash /tmp/gpu_iter.sh TAG  (runs from repo root on the GPU box)
TAG=$1
timeout 700 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_$TAG.json 2>&1
tail -1 gpurun_out/bench_$TAG.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['fps'], d['stage_ms'], d['e2e']['value'])" || tail -5 gpurun_out/bench_$TAG.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 32 -c 32 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python profiles/launch_summary.py gpurun_out/launches_$TAG.csv > gpurun_out/sum_$TAG.txt; head -12 gpurun_out/sum_$TAG.txt
