mkdir -p gpurun_out
T=${1:-g19}
nproc > gpurun_out/nproc_$T.txt; lscpu | grep "Model name" >> gpurun_out/nproc_$T.txt
( time timeout 1500 python bench.py > gpurun_out/bench_full_$T.json 2> gpurun_out/bench_full_$T.err ) 2> gpurun_out/bench_full_time_$T.txt
echo "bench rc=$?"; tail -3 gpurun_out/bench_full_$T.err | grep -v Warn; cat gpurun_out/bench_full_time_$T.txt
( time timeout 1500 python bench.py --impl reference > gpurun_out/bench_ref_$T.json 2> gpurun_out/bench_ref_$T.err ) 2> gpurun_out/bench_ref_time_$T.txt
echo "ref rc=$?"; tail -3 gpurun_out/bench_ref_$T.err; cat gpurun_out/bench_ref_time_$T.txt; tail -c 1500 gpurun_out/bench_ref_$T.json
