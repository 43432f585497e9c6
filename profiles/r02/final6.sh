# Final evidence after the tile-sort changes: bash profiles/r02/final6.sh
# final.sh (bench line, reference arm, warm launch list, ncu of k_splat_tc), then
# ncu --set full of the three tile-sort classes of one bench frame.
bash profiles/r02/final.sh final6
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_tile_sort_depth" -s 5 -c 3 -o gpurun_out/ts_final6 \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-sweep > gpurun_out/ncu_ts_final6.log 2>&1
echo "ncu ts rc=$?"
