# Pre-blend occupancy sweep (launch-bound minimum blocks): bash profiles/r02/tune_prep.sh "VARIANT" ...
mkdir -p gpurun_out
i=0
for v in "$@"; do
  i=$((i+1))
  SF_NVCC_DEFINES="$v" python -c "from paper_2507_07136_b200 import build_native; build_native.build(force=True)" > /dev/null 2>&1
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:"k_preprocess|k_emit_pairs|k_count_pairs|k_tile_sort_depth|k_blend_fixup|k_fixup_decode|k_box2d" -s 10 -c 16 --csv \
      --log-file gpurun_out/tune_$i.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-sweep > /dev/null 2>&1
  python - "$v" gpurun_out/tune_$i.csv <<'PY'
import csv, sys
h = None; t = {}
for x in csv.reader(open(sys.argv[2])):
    if 'Kernel Name' in x: h = x; continue
    if h and len(x) == len(h):
        d = dict(zip(h, x)); t.setdefault(d['Kernel Name'][:24], []).append(float(d['Metric Value'].replace(',', '')))
print(sys.argv[1], {k: round(sum(v) / len(v) / 1e3, 1) for k, v in t.items()}, flush=True)
PY
done
python -c "from paper_2507_07136_b200 import build_native; build_native.build(force=True)" > /dev/null 2>&1
