# walk unroll: stress CTA time for SF_WU variants (and patch-test / other knobs via extra defines)
for v in "$@"; do
  SF_NVCC_DEFINES="$v" python -c "from paper_2507_07136_b200 import build_native; build_native.build(force=True)" > /dev/null 2>&1
  echo "[$v] $(timeout 200 python profiles/r02/stress.py 2000000 1440 1080 | grep 'CTA dur')"
done
python -c "from paper_2507_07136_b200 import build_native; build_native.build(force=True)" > /dev/null 2>&1
