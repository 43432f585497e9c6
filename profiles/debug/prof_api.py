import sys, cProfile, pstats, io
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2507_07136_b200 as sf
from paper_2507_07136_b200 import synthetic
scene = synthetic.make_scene(2_000_000); cam = synthetic.make_camera(1440, 1080)
qv, canon = synthetic.make_query(); qe = sf.QueryEmbedding('q', qv)
for _ in range(3):
    r = sf.query_pipeline(scene, cam, qe, canon, features='eager', instrument=False, max_elements=1 << 40)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    r = sf.query_pipeline(scene, cam, qe, canon, features='eager', instrument=False, max_elements=1 << 40)
pr.disable()
st = io.StringIO(); pstats.Stats(pr, stream=st).sort_stats('tottime').print_stats(14); print(st.getvalue()[:3500])
