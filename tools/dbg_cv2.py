import numpy as np, sys, os
os.environ['DSMC_DEBUG']='1'
sys.path.insert(0,'.')
from paper_2202_02264_b200 import abi, models
from paper_2202_02264_b200.dsmc import Engine
from oracle.py import Oracle
e=Engine(0); O=Oracle()
m=models.cv_tracking(8)
o=O.smooth(m,8,0,seed=3)
r=e.smooth(m,8,0,seed=3,precision=abi.FP64_PARITY,want_pairs=True)
print(o['pair_left'][0], o['pair_right'][0]); print(r['pair_left'][0], r['pair_right'][0])
print('leaves0', o['leaves'][0]); print('leaves1', o['leaves'][1])
