# racecheck / initcheck on tests whose frames take only the tensor-core path
# (k_splat_tc, k_blend_fixup_cta, k_fixup_decode, binning, post): bash profiles/r02/sanitize_tc.sh TAG
TAG=$1
mkdir -p gpurun_out
SEL="test_persistent_splat or test_fused_decode_matches or test_query_pipeline_vs or test_eager_features or test_fixup_overflow"
export NV_COMPUTE_SANITIZER_MAX_RACECHECK_HAZARDS=100000
timeout 1500 compute-sanitizer --tool racecheck --racecheck-report all --print-limit 40 --error-exitcode 3 \
    python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "$SEL" -p no:cacheprovider > gpurun_out/sanitize_racecheck_tc_$TAG.txt 2>&1
echo "racecheck(tc) rc=$?" | tee gpurun_out/sanitize_tc_summary_$TAG.txt
grep -E "passed|failed|RACECHECK SUMMARY" gpurun_out/sanitize_racecheck_tc_$TAG.txt | tail -3 | tee -a gpurun_out/sanitize_tc_summary_$TAG.txt
timeout 1500 compute-sanitizer --tool initcheck --print-limit 40 --error-exitcode 3 \
    python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "test_persistent_splat" -p no:cacheprovider > gpurun_out/sanitize_initcheck_tc_$TAG.txt 2>&1
echo "initcheck(tc) rc=$?" | tee -a gpurun_out/sanitize_tc_summary_$TAG.txt
grep -E "passed|failed|ERROR SUMMARY" gpurun_out/sanitize_initcheck_tc_$TAG.txt | tail -3 | tee -a gpurun_out/sanitize_tc_summary_$TAG.txt
