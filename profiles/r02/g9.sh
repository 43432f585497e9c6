mkdir -p gpurun_out
timeout 120 ./profiles/micro/mma_chain_bench > gpurun_out/mma_chain_g9.txt 2>&1; cat gpurun_out/mma_chain_g9.txt
