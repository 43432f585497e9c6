# Development experiments: k_splat_tc time at config C for build variants
# (SF_NVCC_DEFINES; results of the variants are NOT valid frames).
for v in "" "-DSF_NOSTORE"; do
  SF_NVCC_DEFINES="$v" python -c "from paper_2507_07136_b200 import build_native; build_native.build(force=True)" > /dev/null 2>&1
  echo "variant [$v]: $(timeout 200 python profiles/r02/grid_sweep.py 2>&1 | tail -1)"
  STRESS_NOFEAT=1 timeout 200 python profiles/r02/stress.py 2000000 1440 1080 | grep -E "CTA dur" | sed 's/^/   blend-only /'
done
