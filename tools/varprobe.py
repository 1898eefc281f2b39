import numpy as np, time
import paper_2411_03289_b200 as G
from paper_2411_03289_b200 import workloads as W
for n in [60, 512, 700, 2048]:
    X, Y, K = W.gp_training_set(n, 1, seed=n)
    m = G.GpModel.fit(X, Y, K)
    rng = np.random.default_rng(7); S = 2000
    q = np.column_stack([rng.uniform(-0.5, 2, S), rng.uniform(-2, 2, S), rng.uniform(-0.5, 2, S), rng.uniform(-2, 2, S)])
    q32 = q.astype(np.float32).astype(np.float64)
    _, v64 = m.predict_batch(q32)
    for path in [0,1,2]:
        v = m.variance_batch(q32, path)[:, 0]
        d = v - v64[:, 0]
        print(n, path, "maxabs %.3g  mean %.3g  median|.| %.3g  rel(max/var) %.3g  var range %.3g..%.3g" % (np.abs(d).max(), d.mean(), np.median(np.abs(d)), np.max(np.abs(d)/np.maximum(v64[:,0],1e-12)), v64.min(), v64.max()))
