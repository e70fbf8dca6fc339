"""Per-sequence parity of the config-3 per-sample all-pole path (fp32) against the oracle."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import oracle
from paper_2511_14390_b200 import inputs
from test_gpu_tv import np_problem, run_tv_gpu
from gpu_util import nrm_err

c = inputs.CONFIGS["c3"]
p = inputs.tv_allpole_problem(1003, batch=c["batch"], length=c["length"], order=c["order"], dtype="f32")
q = np_problem(p, "f32")
g = run_tv_gpu(q, "f32")
o = oracle.tv_allpole(q["a"], q["x"], q["zi"], q["gy"], q["gzf"])
for k in ("y", "gx", "ga"):
    print(k, "global", nrm_err(g[k], o[k]))
    per = [nrm_err(g[k][b], o[k][b]) for b in range(c["batch"])]
    print("  per-seq (own rms):", " ".join(f"{e:.1e}" for e in per))
    rmsg = np.sqrt(np.mean(o[k] ** 2))
    mx = [np.max(np.abs(g[k][b] - o[k][b])) / rmsg for b in range(c["batch"])]
    print("  per-seq max err / global rms:", " ".join(f"{e:.1e}" for e in mx))
    print("  per-seq rms / global rms:", " ".join(f"{np.sqrt(np.mean(o[k][b]**2))/rmsg:.2f}" for b in range(c["batch"])))
# where is the worst ga element
b = int(np.argmax([np.max(np.abs(g["ga"][b] - o["ga"][b])) for b in range(c["batch"])]))
d = np.abs(g["ga"][b] - o["ga"][b])
n, i = np.unravel_index(np.argmax(d), d.shape)
print("worst ga at seq", b, "n", n, "i", i, "err", d[n, i], "ga", o["ga"][b, n, i], "g(n)", o["gx"][b, n], "y(n-i-1)",
      o["y"][b, n - i - 1] if n - i - 1 >= 0 else None, "gpu g(n)", g["gx"][b, n])
