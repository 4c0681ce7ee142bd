import numpy as np, sys, os
sys.path.insert(0,'.')
from paper_2202_02264_b200 import abi, models
from paper_2202_02264_b200.dsmc import Engine
from oracle.py import Oracle
e=Engine(0); O=Oracle()
m=models.cv_tracking(8)
o=O.smooth(m,8,0,seed=3)
r=e.smooth(m,8,0,seed=3,precision=abi.FP64_PARITY,want_pairs=True)
print(os.environ.get('DSMC_DEBUG'), os.environ.get('DSMC_SYNC'), 'match', np.array_equal(o['pair_right'], r['pair_right']))
