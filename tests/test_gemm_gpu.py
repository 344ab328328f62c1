"""K5 tcgen05 grouped GEMM vs a plain PyTorch fp32 reference of the same op."""
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2410_17043_b200 import _lib
    return torch, _lib.load(), _lib


_CTR = []


def _ctr(torch):
    """The caller-owned tile-counter pair of the GEMM's dynamic tile order."""
    if not _CTR:
        _CTR.append(torch.zeros(2, dtype=torch.int32, device="cuda"))
    return _CTR[0].data_ptr()


def _run(torch, L, _lib, G, cap, m_rows, N, K, epilogue, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    a = (torch.randn(G * cap, K, device="cuda", generator=g)).to(torch.bfloat16)
    b = (torch.randn(G * N, K, device="cuda", generator=g) / K ** 0.5).to(torch.bfloat16)
    out_cols = N // 2 if epilogue else N
    c = torch.full((G * cap, out_cols), float("nan"), device="cuda", dtype=torch.bfloat16)
    m = torch.tensor(m_rows, dtype=torch.int32, device="cuda")
    rc = L.aurora_grouped_gemm(a.data_ptr(), b.data_ptr(), c.data_ptr(), None, m.data_ptr(), G, cap, N, K, epilogue,
                               _ctr(torch), 0, _lib.stream_ptr())
    assert rc == 0
    torch.cuda.synchronize()
    for gi in range(G):
        if m_rows[gi] == 0:
            continue
        rows = slice(gi * cap, gi * cap + m_rows[gi])
        ref = a[rows].float() @ b[gi * N:(gi + 1) * N].float().T
        if epilogue:
            blocks = ref.view(ref.shape[0], N // 256, 2, 128)
            gate, up = blocks[:, :, 0, :], blocks[:, :, 1, :]
            ref = (torch.nn.functional.silu(gate) * up).reshape(ref.shape[0], N // 2)
        got = c[rows].float()
        assert torch.isfinite(got).all(), f"group {gi}: unwritten rows"
        err = (got - ref).abs().max().item()
        scale = ref.abs().max().item() + 1e-6
        assert err <= 1e-2 * scale + 1e-2, (gi, err, scale)


def test_grouped_gemm_plain(env):
    torch, L, _lib = env
    _run(torch, L, _lib, G=3, cap=300, m_rows=[300, 129, 1], N=512, K=256, epilogue=0)


def test_grouped_gemm_large_k_and_empty_group(env):
    torch, L, _lib = env
    _run(torch, L, _lib, G=4, cap=512, m_rows=[512, 0, 77, 256], N=1024, K=1024, epilogue=0, seed=1)


def test_grouped_gemm_swiglu(env):
    torch, L, _lib = env
    _run(torch, L, _lib, G=2, cap=200, m_rows=[200, 65], N=768, K=512, epilogue=1, seed=2)


def test_expert_ffn_matches_fp32(env):
    torch, L, _lib = env
    G, cap, H, F = 2, 256, 512, 256
    g = torch.Generator(device="cuda").manual_seed(3)
    x = torch.randn(G * cap, H, device="cuda", generator=g).to(torch.bfloat16)
    w1 = (torch.randn(G, F, H, device="cuda", generator=g) / H ** 0.5).to(torch.bfloat16)
    w3 = (torch.randn(G, F, H, device="cuda", generator=g) / H ** 0.5).to(torch.bfloat16)
    w2 = (torch.randn(G, H, F, device="cuda", generator=g) / F ** 0.5).to(torch.bfloat16)
    # interleave gate/up in 128-row blocks: [g0 u0 g1 u1 ...]
    w13 = torch.stack([w1.view(G, F // 128, 128, H), w3.view(G, F // 128, 128, H)], dim=2).reshape(G, 2 * F, H)
    h = torch.empty(G * cap, F, device="cuda", dtype=torch.bfloat16)
    y = torch.empty(G * cap, H, device="cuda", dtype=torch.bfloat16)
    m_rows = [cap, 100]
    m = torch.tensor(m_rows, dtype=torch.int32, device="cuda")
    rc = L.aurora_expert_ffn(x.data_ptr(), w13.contiguous().data_ptr(), w2.data_ptr(), h.data_ptr(), y.data_ptr(),
                             None, m.data_ptr(), G, cap, H, F, None, _ctr(torch), 0, _lib.stream_ptr())
    assert rc == 0
    torch.cuda.synchronize()
    for gi in range(G):
        xs = x[gi * cap: gi * cap + m_rows[gi]].float()
        ref = (torch.nn.functional.silu(xs @ w1[gi].float().T) * (xs @ w3[gi].float().T)) @ w2[gi].float().T
        got = y[gi * cap: gi * cap + m_rows[gi]].float()
        err = (got - ref).abs().max().item()
        assert err <= 2e-2 * ref.abs().max().item() + 1e-2, (gi, err)


@pytest.mark.parametrize("epilogue", [0, 1])
def test_grouped_gemm_half_tile_boundaries(env, epilogue):
    """Group tails of exactly 128 / 129 / 64 / 1 rows next to full tiles (the
    epilogue masks the padding rows of every partial 256-row tile)."""
    torch, L, _lib = env
    _run(torch, L, _lib, G=5, cap=512, m_rows=[128, 384, 385, 64, 257], N=768, K=512, epilogue=epilogue, seed=3)
