"""Debug: GEMM certification flags vs float64 truth (thr1 set to the median candidate D64)."""
import sys
import numpy as np
import torch
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
from conftest import make_blobs
from paper_2603_20009_b200 import device as dev, native
n, k, d, dp = 600, 300, 256, 32
rng = np.random.default_rng(2)
x = make_blobs(n, d, 20, seed=2, spread=3.0)
MODE = sys.argv[1] if len(sys.argv) > 1 else "noisy"
if MODE == "self":
    k = 600
    c = np.ascontiguousarray(x[rng.choice(n, k, replace=False)])
else:
    c = np.ascontiguousarray(x[rng.choice(n, k, replace=False)] + rng.standard_normal((k, d)).astype(np.float32) * 0.5)
X = torch.zeros((n, d), device="cuda"); X[:] = torch.tensor(x)
Cm = torch.zeros((k, d), device="cuda"); Cm[:] = torch.tensor(c)
xh, xl = dev.split_hilo(X, d); ch, cl = dev.split_hilo(Cm, d)
dtrue = ((x[:, None, :dp + 64].astype(np.float64) - c[None, :, :dp + 64]) ** 2).sum(-1)
thr = torch.full((n,), 1e30, device="cuda")
thr1_np = np.median(dtrue, axis=1).astype(np.float32)
if MODE == "self":
    thr1_np[:] = 0.0
thr1 = torch.tensor(thr1_np, device="cuda")
cap = 512
rec = torch.empty((n, cap, 2), dtype=torch.int32, device="cuda"); ci = rec[..., 0]; cv = rec[..., 1].view(torch.float32); cc = torch.empty(n, dtype=torch.int32, device="cuda")
dev.gemm(xh, xl, ch, cl, n, k, dp, native.GEMM_GATE, xsq=dev.row_sq_norms(X, dp), ysq=dev.row_sq_norms(Cm, dp), thr=thr,
         cand=rec, cand_cnt=cc, cand_cap=cap, ext_k=64, xsq_ext=dev.row_sq_norms(X, dp + 64),
         ysq_ext=dev.row_sq_norms(Cm, dp + 64), thr1=thr1, cert_eps=3e-5 if MODE == "self" else 0.0)
torch.cuda.synchronize()
idx = ci.cpu().numpy()
print("counts", cc.cpu().numpy()[:4])
flags = idx[:, :k] < 0
js = idx[:, :k] & 0x7fffffff
exp = dtrue[np.arange(n)[:, None], js] > thr1_np[:, None]
clear = np.abs(dtrue[np.arange(n)[:, None], js] - thr1_np[:, None]) > 1e-2
print("flag rate", flags.mean(), "expected rate", exp.mean(), "mismatch (clear margin)", np.mean((flags != exp) & clear))
bad = np.argwhere((flags != exp) & clear)[:5]
for r, e in bad:
    print("row", r, "col", js[r, e], "flag", flags[r, e], "d64 true", dtrue[r, js[r, e]], "thr1", thr1_np[r])

if MODE == "self":
    print("self mode: flag rate on all candidates", flags.mean())
    xe = dev.row_sq_norms(X, dp + 64).cpu().numpy()
    print("xs_e[:3]", xe[:3], "margin", 3e-5 * 2 * xe[:3])
