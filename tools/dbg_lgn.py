import numpy as np, sys
sys.path.insert(0,'.')
from paper_2202_02264_b200 import abi, models
from paper_2202_02264_b200.dsmc import Engine
from oracle.py import Oracle
e=Engine(0); O=Oracle()
def d2model(T):
    F=np.array([[0.9,0.1],[0.0,0.8]]); Q=np.array([[0.3,0.05],[0.05,0.2]]); H=np.array([[1.0,0.0]]); R=np.array([[0.25]])
    rng=np.random.default_rng(1); y=rng.standard_normal((T+1,1))
    m=abi.Model(abi.MODEL_LGSSM,T,2,1,m0=np.zeros(2),P0=np.eye(2),F=F,b=np.zeros(2),Q=Q,H=H,R=R,y=y,prop_mean=np.zeros((T+1,2)),prop_cov=np.tile(np.eye(2),(T+1,1,1)))
    return models.with_rts_proposals(m)
for name, m in [("d2", d2model(8)), ("cv", models.cv_tracking(8))]:
  for N in [8, 33, 64, 100]:
    for rs in [0,1]:
      o=O.smooth(m,N,rs,seed=3)
      # raw weights: only leaf 0 non-uniform; get them by injecting oracle leaves and letting device compute weights? use device leaf weights: inject states only
      r=e.smooth(m,N,rs,seed=3,precision=abi.FP64_PARITY,want_pairs=True,want_leaves=True)
      dl=np.abs(r['leaves']-o['leaves']).max()
      okL=(r['pair_left']==o['pair_left']).mean(); okR=(r['pair_right']==o['pair_right']).mean()
      print(name,N,rs,'leafdiff',dl,'left agree',okL,'right agree',okR,'right zero frac',(r['pair_right']==0).mean(), 'lmw', np.abs(r['log_mean_weight']-o['log_mean_weight']).max())
