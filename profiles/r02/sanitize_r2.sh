# compute-sanitizer over the GPU tests that launch every frame kernel of the current build
# (k_preprocess, binning, k_tile_sort_depth*, tcs::k_splat_tc (+fused decode / relevancy),
# k_blend_fixup_cta, k_fixup_decode, post, sweep, training):  bash profiles/r02/sanitize_r2.sh TAG
TAG=$1
mkdir -p gpurun_out
SEL="test_fused_decode_matches or test_persistent_splat or test_query_pipeline_vs or test_eager_features or test_query_sweep_ragged or test_empty_scene or test_fixup_overflow or test_device_topk"
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 30 --error-exitcode 3 \
      python -m pytest tests/test_gpu_parity.py tests/test_gpu_round2.py -m gpu -x -q -k "$SEL" -p no:cacheprovider \
      > gpurun_out/sanitize_${tool}_$TAG.txt 2>&1
  echo "$tool rc=$?" | tee -a gpurun_out/sanitize_summary_$TAG.txt
  grep -E "passed|failed|ERROR SUMMARY|RACECHECK SUMMARY|hazard" gpurun_out/sanitize_${tool}_$TAG.txt | tail -4 >> gpurun_out/sanitize_summary_$TAG.txt
done
cat gpurun_out/sanitize_summary_$TAG.txt
