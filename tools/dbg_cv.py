import numpy as np, sys
sys.path.insert(0,'.')
from tests.conftest import golden_model
from paper_2202_02264_b200 import abi
from paper_2202_02264_b200.dsmc import Engine
g=dict(np.load('tests/golden/golden.npz'))
e=Engine(0)
for name in ['cv']:
    spec,m=golden_model(g,name)
    X=g[f'case_{name}_states']; W=g[f'case_{name}_raw_logw']
    r=e.smooth(m,spec['N'],0,seed=spec['seed'],precision=abi.FP64_PARITY,inject_states=X,inject_logw=W,want_paths=True,want_pairs=True)
    L=g[f'case_{name}_0_left']; R=g[f'case_{name}_0_right']; lmw=g[f'case_{name}_0_lmw']
    for c in range(len(L)):
        bad=(r['pair_left'][c]!=L[c])|(r['pair_right'][c]!=R[c])
        print(c, bad.sum(), r['log_mean_weight'][c], lmw[c], r['log_mean_weight'][c]-lmw[c])
print('slot', 'dev(l,r)', 'gold(l,r)')
for q in range(33):
    print(q, r['pair_left'][0][q], r['pair_right'][0][q], L[0][q], R[0][q])
print('paths eq t0', np.abs(r['paths'][0]-g['case_cv_0_paths'][0]).max())
