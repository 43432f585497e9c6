mkdir -p gpurun_out
STRESS_NOFEAT=1 STRESS_TIMEOUT=20 timeout 120 python profiles/r02/stress.py 2000000 1440 1080 > gpurun_out/stress_g17_nofeat.txt 2>&1
grep -E "HANG|total|per tile|per-tile" gpurun_out/stress_g17_nofeat.txt | cut -c1-200
STRESS_NOPROG=1 python - <<'PY'
import os, sys, torch
sys.path.insert(0, '.')
import paper_2507_07136_b200 as sf
from paper_2507_07136_b200 import synthetic
from paper_2507_07136_b200.device import QuerySpec, device_scene
scene = synthetic.make_scene(2000000); cam = synthetic.make_camera(1440, 1080); qv, canon = synthetic.make_query()
eng = device_scene(scene).engine; levels = (0, 1, 2); spec = QuerySpec(qv, canon, 11, -1, 0.5)
for feat in (False, True):
    out = eng.allocate(1440, 1080, levels, coeff_map=False, features=feat, query=True)
    for _ in range(3): eng.run(cam, levels, out, query=spec)
    ts = []
    for _ in range(5):
        eng.run(cam, levels, out, query=spec, timing=True); torch.cuda.synchronize(); ts.append(out.blend_ms())
    print("features" if feat else "lazy", "splat kernel ms", sorted(ts)[2])
PY
