# Launch list (per-kernel device time) of bench frames: bash profiles/r02/launches.sh TAG
# cache-control none keeps L2 warm between kernels as in a real frame (ncu serialises them).
TAG=$1
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -s 60 -c 60 --csv \
    --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-sweep > /dev/null 2>&1
python profiles/launch_summary.py gpurun_out/launches_$TAG.csv 2 > gpurun_out/sum_$TAG.txt 2>&1
head -20 gpurun_out/sum_$TAG.txt
