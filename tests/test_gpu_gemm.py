"""tcgen05 GEMM core vs torch fp32 matmul of the same fp16 operands (exact inputs, fp32
accumulate: only summation order differs), all four operand majors, ragged tails, split-K."""
import pytest
import torch

pytestmark = pytest.mark.gpu


def _ref(A, a_mn, B, b_mn):
    Am = A.float().t() if a_mn else A.float()      # [M][K]
    Bm = B.float().t() if b_mn else B.float()      # [N][K]
    return Am @ Bm.t()


@pytest.mark.parametrize("a_mn,b_mn", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("M,N,K,bn,splits,cg", [
    (128, 128, 64, 128, 1, 1),
    (256, 256, 512, 256, 1, 1),
    (200, 192, 136, 64, 1, 1),      # ragged M and K tails, N tile 64
    (384, 512, 1000, 128, 3, 1),    # split-K with a ragged last split
    (64, 64, 4096, 64, 8, 1),
    (256, 256, 512, 256, 1, 2),     # CTA pair (tcgen05 cta_group::2), one 256x256 tile
    (640, 512, 520, 256, 1, 2),     # CTA pairs, ragged M (2.5 pair tiles) and K
    (512, 384, 2048, 128, 5, 2),    # CTA pairs, BN 128 (64-col halves), split-K
    (100, 256, 64, 256, 1, 2),      # a single partial pair tile (peer rows all out of bounds)
])
def test_gemm_majors(a_mn, b_mn, M, N, K, bn, splits, cg):
    import paper_2306_16688_b200 as P
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N + K)
    A = torch.randn((K, M) if a_mn else (M, K), generator=g, device="cuda").half()
    B = torch.randn((K, N) if b_mn else (N, K), generator=g, device="cuda").half()
    ref = _ref(A, a_mn, B, b_mn)

    def padded(X):       # rows stored with a 16-byte-multiple stride (TMA rule), pad = garbage
        w = (X.shape[1] + 7) // 8 * 8
        Y = torch.full((X.shape[0], w), 3.0, device="cuda").half()
        Y[:, :X.shape[1]] = X
        return Y

    D = P.debug_gemm(padded(A), a_mn, padded(B), b_mn, M, N, K, bn=bn, splits=splits, cg=cg)
    torch.cuda.synchronize()
    err = (D - ref).abs().max().item()
    assert err <= 1e-3 * ref.abs().max().item() + 1e-4, err


def test_gemm_k_not_multiple_of_8_rows_padded():
    """K-major operands whose K (=115) is not a multiple of 8, stored with a padded stride."""
    import paper_2306_16688_b200 as P
    M, N, K = 256, 128, 115
    A = torch.zeros(M, 120, device="cuda").half()
    B = torch.zeros(N, 120, device="cuda").half()
    A[:, :K] = torch.randn(M, K, device="cuda").half()
    B[:, :K] = torch.randn(N, K, device="cuda").half()
    A[:, K:] = 7.0   # garbage in the pad must not leak (TMA bounds = K)
    B[:, K:] = -3.0
    D = P.debug_gemm(A, 0, B, 0, M, N, K, bn=128)
    ref = A[:, :K].float() @ B[:, :K].float().t()
    torch.cuda.synchronize()
    assert (D - ref).abs().max().item() <= 1e-3 * ref.abs().max().item()


@pytest.mark.parametrize("M,N,K,splits", [(512, 512, 4096, 7), (256, 1024, 640, 1), (384, 512, 1000, 3)])
def test_gemm_dw512_pair_tile(M, N, K, splits):
    """The dW tile: 512 columns per CTA pair as two N = 256 MMAs sharing the A tile (MN-major
    A and B, split-K partials), ragged M (384 = 1.5 pair tiles) and K."""
    import paper_2306_16688_b200 as P
    g = torch.Generator(device="cuda").manual_seed(M + N + K)
    A = torch.randn((K, M), generator=g, device="cuda").half()
    B = torch.randn((K, N), generator=g, device="cuda").half()
    D = P.debug_gemm(A, 1, B, 1, M, N, K, bn=512, splits=splits, cg=2)
    ref = _ref(A, 1, B, 1)
    torch.cuda.synchronize()
    assert torch.allclose(D, ref, rtol=1e-3, atol=1e-3 * ref.abs().max().item())
