import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import oracle
from paper_1803_07289_b200 import _ops
from paper_1803_07289_b200.core import synthetic_layer

def layer(n, cin, cout, k, seed):
    loc, feat, th, tb, up = synthetic_layer(seed, 0, n, 3, cin, cout)
    t = {k_: torch.from_numpy(v).cuda().float() for k_, v in dict(loc=loc, feat=feat, th=th, tb=tb, up=up).items()}
    t["nbr"] = _ops.knn(t["loc"], 1, n, k)
    t["csr"] = _ops.csr_build(t["nbr"], 1, n)
    h = dict(loc=loc, feat=feat, th=th, tb=tb, up=up, nbr=t["nbr"].cpu().numpy().astype(np.int64))
    return t, h

for n in (128, 1000):
    t, h = layer(n, 64, 64, 8, seed=25)
    df, dth, dtb, dl = _ops.conv_backward(t["up"], t["feat"], t["loc"], t["nbr"], t["csr"], t["th"], t["tb"], 1, n, mode="split")
    torch.cuda.synchronize()
    rdf, rdth, rdtb, rdl = oracle.conv_backward(h["up"], h["feat"], h["loc"], h["nbr"], h["th"], h["tb"])
    for name, a, b in (("df", df, rdf), ("dth", dth, rdth), ("dtb", dtb, rdtb), ("dl", dl, rdl)):
        a = a.cpu().numpy()
        print(n, name, "maxabs", np.abs(a).max(), "ref", np.abs(b).max(), "relerr", np.linalg.norm(a - b) / np.linalg.norm(b))
    a = dth.cpu().numpy(); print(a.reshape(-1)[:8], rdth.reshape(-1)[:8])
