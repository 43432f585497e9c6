mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/tests_g2.txt 2>&1
echo "tests rc=$?" >> gpurun_out/tests_g2.txt
tail -5 gpurun_out/tests_g2.txt
timeout 300 python profiles/r02/stress.py 2000000 1440 1080 > gpurun_out/stress_g2.txt 2>&1
tail -25 gpurun_out/stress_g2.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_splat_tc -s 2 -c 1 -o gpurun_out/splat_tc_g2 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-sweep > gpurun_out/ncu_g2.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/ncu_g2.log
