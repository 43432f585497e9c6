import sys, numpy as np
sys.path.insert(0,'/root/repo'); sys.path.insert(0,'/root/repo/tests')
import paper_2507_07136_b200 as sf
from conftest import load_golden
scene, cam, z = load_golden(sys.argv[1] if len(sys.argv)>1 else 'permuted_ids')
cm = sf.splat_multilevel(scene, cam).data
ref = z['cmap']
d = np.abs(cm-ref)
print('max', d.max(), 'shape', d.shape)
bad = d.max(axis=2) > 1e-5
print('bad pixels', bad.sum(), 'of', bad.size)
ys, xs = np.nonzero(bad)
print('bad y', np.unique(ys)[:20], 'bad x', np.unique(xs)[:20])
print('bad channels', np.unique(np.nonzero(d.reshape(-1,d.shape[2]).max(axis=0) > 1e-5)[0]))
# per pixel: ratio of our mass vs ref mass per level
L=z['config'][1]
for lv in range(d.shape[2]//L):
    m = cm[:,:,lv*L:(lv+1)*L].sum(2); r = ref[:,:,lv*L:(lv+1)*L].sum(2)
    print('level', lv, 'max mass diff', np.abs(m-r).max())
print('sample bad pixel', ys[:3], xs[:3]); 
for y,x in list(zip(ys,xs))[:3]:
    print(y,x,'ours', np.round(cm[y,x][cm[y,x]>0][:8],4), 'ref', np.round(ref[y,x][ref[y,x]>0][:8],4))
