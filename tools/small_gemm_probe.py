import numpy as np, torch, sys
sys.path.insert(0, "/root/repo")
from paper_2603_20009_b200.engine import chain_gemm
from paper_2603_20009_b200.device import to_device_matrix
rng = np.random.default_rng(0)
for (M, N, K) in [(24, 48, 48), (24, 128, 128), (120, 128, 128), (256, 128, 128), (48, 256, 256), (400, 96, 96), (4096, 64, 64), (1000, 200, 200), (3000, 48, 48)]:
    a = rng.standard_normal((M, K)).astype(np.float32)
    R = rng.standard_normal((N, K)).astype(np.float32)  # x @ R.T
    want = a @ R.T
    out = torch.empty((M, (N + 3) // 4 * 4), device="cuda")
    chain_gemm(to_device_matrix(a), to_device_matrix(R), M, N, K, out, 0, 448)
    got = out[:, :N].cpu().numpy()
    # also x @ R (NN)
    R2 = rng.standard_normal((K, N)).astype(np.float32)
    want2 = a @ R2
    out2 = torch.empty((M, (N + 3) // 4 * 4), device="cuda")
    chain_gemm(to_device_matrix(a), to_device_matrix(np.ascontiguousarray(R2.T)), M, N, K, out2, 0, 448)
    got2 = out2[:, :N].cpu().numpy()
    print((M, N, K), "NT diff", int((got != want).sum()), "NN diff", int((got2 != want2).sum()), "of", M * N, flush=True)
