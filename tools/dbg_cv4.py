import numpy as np, sys
sys.path.insert(0,'.')
from paper_2202_02264_b200 import abi, models
from paper_2202_02264_b200.dsmc import Engine, kalman_smooth
e=Engine(0)
m=models.cv_tracking(255)
km,kP,ll=kalman_smooth(m)
sd=np.sqrt(np.einsum('tii->ti',kP))
for prec in [abi.FP64_PARITY, abi.FP32]:
  for N in [256, 1024]:
    r=e.smooth(m,N,0,seed=5,precision=prec)
    z=(r['mean']-km)/sd
    print(prec,N,'zrms',np.sqrt(np.mean(z**2)), 'per-dim', np.sqrt(np.mean(z**2,axis=0)), 'lnc', r['log_norm_const'], ll, 'covratio', np.median(np.einsum('tii->ti',r['cov'])/np.einsum('tii->ti',kP),axis=0))
# leaf check FP32 vs FP64: mean of leaves should be prop mean
r=e.smooth(m,1024,0,seed=5,precision=abi.FP64_PARITY,want_leaves=True)
L=r['leaves']; print('leaf mean err', np.abs(L.mean(1)-m.arrays['prop_mean']).max(), 'leaf cov ratio', np.median(np.einsum('tnk,tnk->tk',L-L.mean(1,keepdims=True),L-L.mean(1,keepdims=True))/1024/np.einsum('tii->ti',m.arrays['prop_cov']),axis=0))
