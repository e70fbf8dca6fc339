import sys, os, torch, numpy as np
sys.path.insert(0, os.getcwd())
import bench
from paper_2511_14390_b200 import _binding as B
w = dict(bench.WORKLOADS[sys.argv[1]], key=sys.argv[1])
prob = bench.Problem(w, 0, 1, 2)
prob.desc.flags = 0
ntot = w["batch"] * ((w["length"] + 4095) // 4096)
buf = torch.zeros(ntot * 8, dtype=torch.int64, device="cuda")
B.iir_debug_trace(buf)
s = torch.cuda.Stream()
st = prob.sets[0]
with torch.cuda.stream(s):
    B.iir_forward(prob.desc, prob.b, prob.a, st["x"], prob.zi, st["y"], prob.zf, prob.tape, prob.tb, prob.ws, prob.wb, s)
s.synchronize()
t = buf.view(ntot, 8).cpu().numpy()
t0 = t[t[:, 0] > 0, 0].min()
for k in [0, 1, 2, 12, 15, 16, 100]:
    print(k, [(int(v - t0) // 1000 if v > 0 else -1) for v in t[k]])
print("tiles never started:", np.where(t[:, 0] == 0)[0][:50])
print("tiles without phase1:", np.where(t[:, 1] == 0)[0][:50])
print("tiles without phase2:", np.where(t[:, 2] == 0)[0][:50])
print("tiles without phase3:", np.where(t[:, 3] == 0)[0][:50])
