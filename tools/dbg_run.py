import sys, os, time, torch
sys.path.insert(0, os.getcwd())
import bench
from paper_2511_14390_b200 import _binding as B
w = dict(bench.WORKLOADS[sys.argv[1]], key=sys.argv[1])
ready = sys.argv[2] == "ready"
prob = bench.Problem(w, 0, 1, 2)
if not ready:
    prob.desc.flags = 0
s = torch.cuda.Stream()
for i in range(4):
    t0 = time.time()
    st = prob.sets[0]
    with torch.cuda.stream(s):
        B.iir_forward(prob.desc, prob.b, prob.a, st["x"], prob.zi, st["y"], prob.zf, prob.tape, prob.tb, prob.ws, prob.wb, s)
    s.synchronize(); t1 = time.time()
    with torch.cuda.stream(s):
        B.iir_backward(prob.desc, st["gy"], prob.gzf, prob.b, prob.a, st["x"], st["y"], prob.zi, prob.tape, prob.tb, st["gx"], prob.gb, prob.ga, prob.gzi, prob.ws, prob.wb, s)
    s.synchronize(); t2 = time.time()
    print(i, "fwd %.3f ms  bwd %.3f ms" % ((t1-t0)*1e3, (t2-t1)*1e3), flush=True)
