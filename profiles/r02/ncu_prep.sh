# ncu --set full of the pre-blend kernels of one bench frame: bash profiles/r02/ncu_prep.sh TAG
TAG=$1
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_tile_sort_depth|k_count_pairs_agg|k_emit_pairs|k_preprocess|k_blend_fixup_cta" \
   -s 40 -c 6 -o gpurun_out/prep_$TAG python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-sweep > gpurun_out/ncu_prep_$TAG.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/ncu_prep_$TAG.log
