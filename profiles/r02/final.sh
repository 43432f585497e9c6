# Final evidence of the round's shipped code: bash profiles/r02/final.sh TAG
# full bench line (parity, CPU baseline, e2e, sweeps, clocks), the reference arm, a warm launch
# list of bench frames, and ncu --set full of the dominant kernel.
mkdir -p gpurun_out
T=${1:-final}
nproc > gpurun_out/host_$T.txt; lscpu | grep "Model name" >> gpurun_out/host_$T.txt; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv >> gpurun_out/host_$T.txt
( time timeout 1500 python bench.py > gpurun_out/bench_full_$T.json 2> gpurun_out/bench_full_$T.err ) 2> gpurun_out/bench_full_time_$T.txt
echo "bench rc=$?"; tail -2 gpurun_out/bench_full_$T.err | grep -v Warn; cat gpurun_out/bench_full_time_$T.txt
( time timeout 1500 python bench.py --impl reference > gpurun_out/bench_ref_$T.json 2> gpurun_out/bench_ref_$T.err ) 2> gpurun_out/bench_ref_time_$T.txt
echo "ref rc=$?"; cat gpurun_out/bench_ref_time_$T.txt | grep real
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -s 60 -c 60 --csv \
    --log-file gpurun_out/launches_$T.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-sweep > /dev/null 2>&1
python profiles/launch_summary.py gpurun_out/launches_$T.csv 4 > gpurun_out/launch_summary_$T.txt 2>&1; head -16 gpurun_out/launch_summary_$T.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_splat_tc -s 2 -c 1 -o gpurun_out/splat_$T python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-sweep > gpurun_out/ncu_$T.log 2>&1
echo "ncu rc=$?"
