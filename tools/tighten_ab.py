import os, sys, subprocess, json
import numpy as np
sys.path.insert(0, os.getcwd())
code = r'''
import os, sys, numpy as np
sys.path.insert(0, os.getcwd())
import paper_2411_03289_b200 as G
from paper_2411_03289_b200 import workloads as W
from tests.helpers import build_pair
cfg = sys.argv[1]
w = W.CONFIGS[cfg]
_, pd, _, td, _ = build_pair(w, samples=512)
x = np.array(w.x0)
d = G.StepDiagnostics()
pd.plan_step(x, td, d)
np.savez(sys.argv[2], radii=pd.lane_radii(), cov=pd.horizon_covariances(), inf=int(d.tightening_infeasible))
print('minr', pd.lane_radii().min(), 'T', len(pd.lane_radii()), file=sys.stderr)
'''
open('/tmp/tc_one.py', 'w').write(code)
for cfg in ('config3', 'config2'):
    outs = {}
    for e in ('0', '1'):
        env = dict(os.environ, GPMPPI_TIGHTEN_SEQUENTIAL=e)
        f = f'/tmp/tc_{cfg}_{e}.npz'
        r = subprocess.run([sys.executable, '/tmp/tc_one.py', cfg, f], env=env, capture_output=True, text=True)
        print(cfg, e, r.stderr[-300:].strip())
        outs[e] = np.load(f)
    a, b = outs['0'], outs['1']
    print(cfg, 'inf', a['inf'], b['inf'], 'radii maxdiff', np.abs(a['radii'] - b['radii']).max(), 'cov maxrel', np.abs(a['cov'] - b['cov']).max() / (np.abs(b['cov']).max() + 1e-300))
    dk = np.nonzero(np.abs(a['cov'] - b['cov']).reshape(a['cov'].shape[0], -1).max(1) > 0)[0]
    print('first differing step', dk[:5], 'radii a/b', a['radii'][:3], b['radii'][:3])
