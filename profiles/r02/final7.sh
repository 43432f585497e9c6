# Final evidence of the shipped code, gated on the GPU suite: bash profiles/r02/final7.sh
# GPU tests, then final.sh (bench line with the Python reference installed in baseline/_ref,
# the reference arm, a warm launch list, ncu --set full of k_splat_tc).
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/tests_final7.txt 2>&1
rc=$?; tail -2 gpurun_out/tests_final7.txt
[ $rc -eq 0 ] || exit $rc
bash profiles/r02/final.sh final7
