import sys, numpy as np
sys.path.insert(0,'tests'); sys.path.insert(0,'.')
from _masks import random_mask
from _oracle import ref
from paper_2603_20481_b200 import specsense as ss
R=ref()
rng=np.random.default_rng(5)
for rows, cols, d in [(500,1024,0.5),(100,100,0.5),(40,64,0.5),(20,40,0.5)]:
    m = random_mask(rng, rows, cols, d)
    ext, lab = ss.label_components(m, 4)
    eext, elab = R.label_components(m, 4)
    bad = np.argwhere(lab != elab)
    print(rows, cols, 'ext eq', np.array_equal(ext, eext), 'nbad', len(bad), bad[:5].tolist(), [ (lab[tuple(b)], elab[tuple(b)], m[tuple(b)]) for b in bad[:5]])
