mkdir -p gpurun_out
T=${1:-g22}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_configs.py -m gpu -x -q -p no:cacheprovider -k "fixup or config or random or fused" > gpurun_out/tests_$T.txt 2>&1
echo "tests rc=$?" >> gpurun_out/tests_$T.txt
grep -E "FAILED|Error|passed|failed" gpurun_out/tests_$T.txt | head -20
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 60 -c 13 --csv --log-file gpurun_out/launches_$T.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-sweep > /dev/null 2>&1
python profiles/r02/launch_list.py gpurun_out/launches_$T.csv
