import sys, os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2603_20009_b200 import device as dev, native
M,N,K=777,1536,1536
rng=np.random.default_rng(1)
a=rng.standard_normal((M,K)).astype(np.float32); b=rng.standard_normal((N,K)).astype(np.float32)
A=dev.to_device_matrix(a); B=dev.to_device_matrix(b)
ah,al=dev.split_hilo(A,K); bh,bl=dev.split_hilo(B,K)
ref=a.astype(np.float64)@b.astype(np.float64).T
scale=np.sqrt((a.astype(np.float64)**2)@(b.astype(np.float64)**2).T)
for kc in (1536,256,64,32):
    acc=torch.zeros((M,N),dtype=torch.float32,device='cuda')
    out=torch.empty((M,N),dtype=torch.float32,device='cuda')
    for k0 in range(0,K,kc):
        dev.gemm(ah[:,k0:],al[:,k0:],bh[:,k0:],bl[:,k0:],M,N,kc,native.GEMM_STORE,out=out)
        acc+=out
    e=np.abs(acc.cpu().numpy()-ref)/scale
    print('chunk',kc,'max',e.max(),'mean',e.mean())
# 1xTF32 (hi only) for reference
out=torch.empty((M,N),dtype=torch.float32,device='cuda'); z=torch.zeros_like(ah); zb=torch.zeros_like(bh)
dev.gemm(A,z,B,zb,M,N,K,native.GEMM_STORE,out=out)
e=np.abs(out.cpu().numpy()-ref)/scale; print('1xtf32 raw max',e.max(),'mean',e.mean())
# numpy fp32 sgemm for comparison
s=(a@b.T); e=np.abs(s-ref)/scale; print('openblas sgemm max',e.max(),'mean',e.mean())
