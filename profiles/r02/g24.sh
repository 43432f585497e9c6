mkdir -p gpurun_out
T=${1:-g24}
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/tests_$T.txt 2>&1
echo "tests rc=$?" >> gpurun_out/tests_$T.txt
grep -E "FAILED|Error|passed|failed" gpurun_out/tests_$T.txt | head -20
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.txt 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke_$T.txt
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 60 -c 26 --csv --log-file gpurun_out/launches_$T.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-sweep > /dev/null 2>&1
python profiles/launch_summary.py gpurun_out/launches_$T.csv 2 > gpurun_out/sum_$T.txt 2>&1; cat gpurun_out/sum_$T.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_splat_tc -s 2 -c 1 -o gpurun_out/splat_$T python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-sweep > gpurun_out/ncu_$T.log 2>&1
echo "ncu rc=$?"
