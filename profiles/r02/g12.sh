mkdir -p gpurun_out
T=${1:-g12}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_configs.py -m gpu -x -q -p no:cacheprovider -k "config or binning or tile or ties or random or bin" > gpurun_out/tests_$T.txt 2>&1
echo "tests rc=$?" >> gpurun_out/tests_$T.txt
grep -E "FAILED|Error|passed|failed" gpurun_out/tests_$T.txt | head -10
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 60 -c 15 --csv --log-file gpurun_out/launches_$T.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-sweep > /dev/null 2>&1
python profiles/r02/launch_list.py gpurun_out/launches_$T.csv
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_tile_sort_depth|k_blend_fixup_cta" -c 3 -o gpurun_out/prep_$T python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-sweep > gpurun_out/ncu_$T.log 2>&1
echo "ncu rc=$?"
