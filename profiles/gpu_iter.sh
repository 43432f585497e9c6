# One GPU iteration (run from the repo root on the GPU box):  bash profiles/gpu_iter.sh TAG
# -m gpu tests, a default bench line, and an ncu launch list of two frames (27 launches each).
TAG=$1
timeout 700 python -m pytest tests -m gpu -x -q > gpurun_out/tests_$TAG.txt 2>&1
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_$TAG.json 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 54 -c 54 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python profiles/launch_summary.py gpurun_out/launches_$TAG.csv 2 > gpurun_out/sum_$TAG.txt
head -12 gpurun_out/sum_$TAG.txt
tail -1 gpurun_out/bench_$TAG.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['fps'], d['stage_ms'], d['e2e']['value'])" || tail -5 gpurun_out/bench_$TAG.json
tail -3 gpurun_out/tests_$TAG.txt
