"""C2-shaped conv forward / backward (with d_locations) / deconv written to an .npz: run once with
and once without FC_NO_CONCURRENT=1 to check that the concurrent channel-block passes of small
clouds give bitwise the sequential results (tests/test_gpu_wide.py).
   python scripts/concurrent_passes_check.py out.npz"""
import sys, torch, numpy as np
sys.path.insert(0,'.')
from paper_1803_07289_b200 import _ops
B,n,k,ci,co=8,1024,16,64,128
T=B*n
g=torch.Generator(device='cuda'); g.manual_seed(2)
pos=(torch.floor(torch.rand(T,3,device='cuda',dtype=torch.float64,generator=g)*2**24)/2**24).float()
nbr=_ops.knn(pos,B,n,k); csr=_ops.csr_build(nbr,B,n)
f=torch.randn(T,ci,device='cuda',generator=g); th=0.1*torch.randn(co,ci,3,device='cuda',generator=g); tb=0.1*torch.randn(co,ci,device='cuda',generator=g)
up=torch.randn(T,co,device='cuda',generator=g)
out=_ops.conv_forward(f,pos,nbr,th,tb,B,n)
res=_ops.conv_backward(up,f,pos,nbr,csr,th,tb,B,n,need=(True,True,True,True))
y=_ops.deconv_forward(up,pos,csr,th,tb,B,n,k)
np.savez(sys.argv[1], out=out.cpu().numpy(), *[r.cpu().numpy() for r in res], y=y.cpu().numpy())
