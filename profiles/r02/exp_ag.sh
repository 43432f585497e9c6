# alpha group size: stress CTA time and a short bench for SF_AG variants
for v in 1 2; do
  SF_NVCC_DEFINES="-DSF_AG=$v" python -c "from paper_2507_07136_b200 import build_native; build_native.build(force=True)" > /dev/null 2>&1
  echo "AG=$v $(timeout 200 python profiles/r02/stress.py 2000000 1440 1080 | grep 'CTA dur')"
done
python -c "from paper_2507_07136_b200 import build_native; build_native.build(force=True)" > /dev/null 2>&1
