mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_g1.txt
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/tests_g1.txt 2>&1
echo "tests rc=$?" >> gpurun_out/tests_g1.txt
tail -5 gpurun_out/tests_g1.txt
timeout 400 python bench.py --no-cpu-baseline --no-sweep --steps 10 --warmup 3 > gpurun_out/bench_g1.json 2> gpurun_out/bench_g1.err
echo "bench rc=$?"; tail -3 gpurun_out/bench_g1.err; tail -c 3000 gpurun_out/bench_g1.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 60 -c 60 --csv --log-file gpurun_out/launches_g1.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-sweep > /dev/null 2>&1
python profiles/launch_summary.py gpurun_out/launches_g1.csv 2 > gpurun_out/sum_g1.txt 2>&1
head -30 gpurun_out/sum_g1.txt
