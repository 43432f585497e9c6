# compute-sanitizer over a representative slice of the GPU suite (run from the repo root on the GPU box):
#   bash profiles/sanitize.sh TAG
# memcheck / racecheck / synccheck / initcheck each on the tests that cover every kernel family:
# projection + binning, blend (+ fused decode, relevancy), fixup replay, post, sweep, standalone decode.
TAG=$1
SEL="test_random_scenes_vs_oracle or test_fused_decode_matches or test_fused_decode_empty or test_query_sweep_ragged or test_tensor_core_decode or test_k_equals_l or test_empty_scene"
export SF_SANITIZE=1
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 3 \
      python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "$SEL" -p no:cacheprovider \
      > gpurun_out/sanitize_${tool}_$TAG.txt 2>&1
  echo "$tool rc=$?" | tee -a gpurun_out/sanitize_summary_$TAG.txt
  tail -4 gpurun_out/sanitize_${tool}_$TAG.txt >> gpurun_out/sanitize_summary_$TAG.txt
done
