for nb in 1 2 3 7 16 32; do
for tma in 0 1; do
  if [ $tma = 1 ]; then export CD_DISABLE_TMA=1; else unset CD_DISABLE_TMA; fi
  timeout 60 python -c "
import sys; sys.path.insert(0,'.'); sys.path.insert(0,'tests')
import numpy as np, torch, synthetic, oracle, paper_1602_07527_b200 as cd
from gpu_helpers import to_dev, to_host, nerr
L, Lb, Sd = synthetic.draw(300, 77, sdot=True)
try:
    r = cd.chol_rev(to_dev(L), to_dev(Lb), nb=$nb); torch.cuda.synchronize()
    print('nb=$nb notma=$tma rev', nerr(to_host(r), oracle.chol_rev(L, Lb)))
except Exception as e: print('nb=$nb notma=$tma rev FAIL', str(e)[:150])
" 2>&1 | tail -1
done; done
