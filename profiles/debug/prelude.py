"""Host time of one query_pipeline call split into its pieces (config C), development aid."""
import os, sys, time, cProfile, pstats
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import torch
import paper_2507_07136_b200 as sf
from paper_2507_07136_b200 import synthetic
scene = synthetic.make_scene(2_000_000); cam = synthetic.make_camera(1440, 1080)
qv, canon = synthetic.make_query(); qe = sf.QueryEmbedding('q', qv)
for _ in range(3):
    sf.query_pipeline(scene, cam, qe, canon, features='eager', instrument=False, max_elements=1 << 40)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
t0 = time.perf_counter()
for _ in range(10):
    r = sf.query_pipeline(scene, cam, qe, canon, features='eager', instrument=False, max_elements=1 << 40)
t1 = time.perf_counter()
pr.disable()
print(f"{(t1 - t0) * 100:.2f} ms per call")
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
