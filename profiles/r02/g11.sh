mkdir -p gpurun_out
LIB=paper_2507_07136_b200/libsplatfield_b200.so
cp $LIB /tmp/lib_orig.so
for v in D A B C; do
  cp profiles/r02/variants/lib_$v.so $LIB
  echo "=== variant $v"
  STRESS_TIMEOUT=20 timeout 120 python profiles/r02/stress.py 2000000 1440 1080 > gpurun_out/stress_g11_$v.txt 2>&1
  grep -E "HANG|blend  |drain  |dec_iss|per-tile|mean:" gpurun_out/stress_g11_$v.txt | cut -c1-160
  timeout 300 python bench.py --no-cpu-baseline --no-sweep --no-e2e --steps 5 --warmup 3 > gpurun_out/bench_g11_$v.json 2>/dev/null
  tail -1 gpurun_out/bench_g11_$v.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', round(d['value'],1), 'splat', round(d['fps']['feature_splat'],1), 'blend_ms', round(d['stage_ms']['blend_kernel'],3))"
done
cp /tmp/lib_orig.so $LIB
