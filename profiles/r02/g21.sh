mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_blend_fixup_cta|k_count_pairs_agg" -c 2 -o gpurun_out/fx_g21 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-sweep > gpurun_out/ncu_g21.log 2>&1
echo "ncu rc=$?"
