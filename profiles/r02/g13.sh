mkdir -p gpurun_out
STRESS_TIMEOUT=20 timeout 120 python profiles/r02/stress.py 2000000 1440 1080 > gpurun_out/stress_g13.txt 2>&1
grep -E "HANG|total|per tile|per-tile|mean:" gpurun_out/stress_g13.txt | cut -c1-220
