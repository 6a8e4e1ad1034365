"""The exact-chain layer: device contractions and norms bitwise equal to the reference's
numerics backends (OpenBLAS sgemm / portable_matmul / np.einsum), and the tensor-core full pass
settled to the reference's exact argmin and distance bits.

Golden hashes: tests/golden/make_blas_bits.py (run on the survey container, whose OpenBLAS
produced every reference golden).  The GPU box's own numpy is also compared (diagnostic: its CPU
may select another OpenBLAS kernel)."""

import hashlib
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden", "blas_bits.npz")


def _mk():
    import importlib.util
    spec = importlib.util.spec_from_file_location("mbb", os.path.join(HERE, "golden", "make_blas_bits.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


MB = _mk()


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _pad(x):
    from paper_2603_20009_b200 import device
    return device.to_device_matrix(x)


@pytest.mark.parametrize("kmajor", [False, True])
@pytest.mark.parametrize("case", MB.GEMM_CASES)
def test_chain_gemm_bitwise_openblas(case, kmajor):
    """skm_chain_gemm (fma chain, K blocks of 448) == the survey container's sgemm, bit for bit,
    with b as [N][K] rows and as a k-major [K][N] matrix (the cp.async kernel the rotation uses)."""
    from paper_2603_20009_b200.engine import chain_gemm
    M, N, K, lay = case
    a, b = MB.gemm_inputs(M, N, K, lay, 0)
    bt = b if lay == "nt" else np.ascontiguousarray(b.T)
    out = torch.empty((M, (N + 3) // 4 * 4), dtype=torch.float32, device="cuda")
    if kmajor:
        chain_gemm(_pad(a), _pad(np.ascontiguousarray(bt.T)), M, N, K, out, 0, 448, b_kmajor=True)
    else:
        chain_gemm(_pad(a), _pad(bt), M, N, K, out, 0, 448)
    got = out[:, :N].cpu().numpy()
    g = np.load(GOLD)
    here = a @ b.T if lay == "nt" else a @ b
    print(case, "differs from this box's numpy in", int(np.count_nonzero(got != here)), "of", got.size)
    assert _sha(got) == str(g[f"gemm_{M}_{N}_{K}_{lay}"])


def test_chain_gemm_portable_bitwise():
    """flavour 1 == the reference's portable_matmul (mul + add chain, _kernels.pyx:122-142)."""
    from oracle import kernels_np as O
    from paper_2603_20009_b200.engine import chain_gemm
    rng = np.random.default_rng(11)
    a = rng.standard_normal((130, 700)).astype(np.float32)
    b = rng.standard_normal((70, 700)).astype(np.float32)
    want = np.empty((130, 70), np.float32)
    O.portable_matmul(a, b, 700, want)
    out = torch.empty((130, 72), dtype=torch.float32, device="cuda")
    chain_gemm(_pad(a), _pad(b), 130, 70, 700, out, 1, 0)
    assert np.array_equal(out[:, :70].cpu().numpy(), want)
    out.zero_()
    chain_gemm(_pad(a), _pad(np.ascontiguousarray(b.T)), 130, 70, 700, out, 1, 0, b_kmajor=True)
    assert np.array_equal(out[:, :70].cpu().numpy(), want)


@pytest.mark.parametrize("shape", [(1000, 1536, 1536), (517, 1002, 1002), (300, 77, 1001), (129, 130, 449),
                                   (64, 40, 7), (257, 1024, 897)])
def test_chain_gemm_kmajor_equals_rowmajor(shape):
    """The k-major cp.async kernel and the [N][K] kernel produce the same bits, including ragged
    M / N / K tiles, K blocks that start off a 16-byte boundary (K = 1002: 448 + 277 + 277) and
    signed zeros from the distance clamp."""
    from paper_2603_20009_b200.engine import chain_gemm
    M, N, K = shape
    rng = np.random.default_rng(M + N + K)
    a = rng.standard_normal((M, K)).astype(np.float32)
    b = rng.standard_normal((N, K)).astype(np.float32)
    a[:, ::5] = 0.0
    A, B, BT = _pad(a), _pad(b), _pad(np.ascontiguousarray(b.T))
    ld = (N + 3) // 4 * 4
    for mode in (0, 1):
        kw = {}
        if mode:
            kw = dict(xsq=torch.from_numpy((a.astype(np.float64) ** 2).sum(1).astype(np.float32)).cuda(),
                      ysq=torch.from_numpy((b.astype(np.float64) ** 2).sum(1).astype(np.float32)).cuda())
        for fl, q in ((0, 448), (1, 0)):
            o1 = torch.full((M, ld), 7.0, device="cuda")
            o2 = torch.full((M, ld), 7.0, device="cuda")
            chain_gemm(A, B, M, N, K, o1, fl, q, **kw)
            chain_gemm(A, BT, M, N, K, o2, fl, q, b_kmajor=True, **kw)
            assert torch.equal(o1[:, :N].view(torch.int32), o2[:, :N].view(torch.int32)), (shape, mode, fl)


@pytest.mark.parametrize("case", MB.NORM_CASES)
def test_row_norms_bitwise_einsum(case):
    from paper_2603_20009_b200 import device
    n, d = case
    m = MB.norm_input(n, d, 0)
    g = np.load(GOLD)
    X = _pad(m)
    for dims in (d, max(1, d // 3 + 1)):
        got = device.row_sq_norms(X, dims).cpu().numpy()
        want = np.einsum("ij,ij->i", m[:, :dims], m[:, :dims], dtype=np.float64).astype(np.float32)
        assert np.array_equal(got, want)
        assert _sha(got) == str(g[f"norm_{n}_{d}_{dims}"])


@pytest.mark.parametrize("n,k,d", [(5000, 300, 128), (3000, 700, 1536), (2500, 64, 1000)])
def test_full_assign_pass_exact(n, k, d):
    """Tensor-core ARGMIN + top-2 margin + exact fix-up == argmin of the reference's own distance
    block (chain GEMM + expansion), assignments and tau bitwise, including planted exact ties."""
    from conftest import make_blobs
    from paper_2603_20009_b200.config import KMeansConfig
    from paper_2603_20009_b200.engine import Centroids, DeviceData, Workspace, chain_gemm, full_assign_pass
    x = make_blobs(n, d, 40, seed=d, spread=2.0)
    rng = np.random.default_rng(d)
    c = np.ascontiguousarray(x[rng.choice(n, k, replace=False)])
    c[k // 2: k // 2 + 20] = c[:20]  # duplicated centroids: exact ties, lowest index must win
    X, Cm = _pad(x), _pad(c)
    data = DeviceData(X, d)
    cents = Centroids(Cm, d)
    cents.refresh(d, None)
    ws = Workspace(X.device, n, k, d, KMeansConfig(k=k))
    full_assign_pass(data, cents, ws)
    D = torch.empty((n, (k + 3) // 4 * 4), dtype=torch.float32, device="cuda")
    chain_gemm(X, Cm, n, k, d, D, 0, 448, xsq=data.norms(d), ysq=cents.ysq)
    Dn = D[:, :k].cpu().numpy()
    assert np.array_equal(ws.assign[:n].cpu().numpy(), np.argmin(Dn, axis=1))
    assert np.array_equal(ws.tau[:n].cpu().numpy(), Dn.min(axis=1))
    print("rows re-evaluated exactly:", int(ws.amb_count.item()))
