mkdir -p gpurun_out
T=g4
timeout 60 ./profiles/micro/mma_chain_bench > gpurun_out/mma_chain_$T.txt 2>&1; cat gpurun_out/mma_chain_$T.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_configs.py -m gpu -x -q -p no:cacheprovider -k "fixup or config or random_scenes or overflow" > gpurun_out/tests_$T.txt 2>&1
echo "tests rc=$?" >> gpurun_out/tests_$T.txt; tail -3 gpurun_out/tests_$T.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_tile_sort_depth|k_count_pairs_agg|k_emit_pairs|k_preprocess|k_blend_fixup_cta" -c 6 -o gpurun_out/prep_$T python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-sweep > gpurun_out/ncu_$T.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/ncu_$T.log
