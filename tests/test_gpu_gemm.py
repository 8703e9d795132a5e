"""K1 tcgen05 GEMM: every fused epilogue vs a torch fp32 reference, split-K
cluster reduction, batch invariance (row bits independent of M) and shape
edge cases (M=1, ragged M, M > 256 -> several token tiles, N padding)."""
import ctypes as C

import numpy as np
import pytest

from paper_2602_02204_b200 import dev_lib, check

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def gemm(W, X, M, epi, out, ldo, gate=None, ldg=0, goff=0, rpg=16, max_splits=8):
    sp = C.c_int32()
    check(dev_lib().omni_k_gemm(C.c_uint64(W.data_ptr()), W.shape[0], W.shape[1], C.c_uint64(X.data_ptr()), M, epi,
                                C.c_uint64(out.data_ptr()), ldo, C.c_uint64(gate.data_ptr() if gate is not None else 0),
                                ldg, goff, rpg, max_splits, C.byref(sp)))
    torch.cuda.synchronize()
    return sp.value


@pytest.mark.parametrize("N,K,M", [(128, 64, 1), (256, 2048, 5), (3072, 2048, 16), (2048, 8192, 200),
                                   (1024, 1024, 300), (16384, 2048, 33), (128, 128, 257),
                                   (3072, 2048, 48), (2048, 8192, 64), (2048, 2048, 37)])
@pytest.mark.parametrize("max_splits", [1, 8])
def test_f32_matches_torch(N, K, M, max_splits):
    g = torch.Generator(device="cuda").manual_seed(N * 7 + M)
    W = (torch.randn(N, K, device="cuda", generator=g) / K ** 0.5).bfloat16()
    X = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    out = torch.zeros(M, N, device="cuda")
    gemm(W, X, M, 1, out, N, max_splits=max_splits)
    ref = X.float() @ W.float().t()
    assert (out - ref).abs().max().item() < 1e-4 * max(1.0, K / 1024)


@pytest.mark.parametrize("epi", [0, 2, 3, 4, 5])
@pytest.mark.parametrize("N,K,M", [(256, 256, 7), (1024, 2048, 40), (512, 512, 300)])
def test_epilogues(epi, N, K, M):
    g = torch.Generator(device="cuda").manual_seed(epi * 100 + M)
    W = (torch.randn(N, K, device="cuda", generator=g) / K ** 0.5).bfloat16()
    X = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    acc = X.float() @ W.float().t()
    gate = None
    if epi == 4:  # tile-interleaved gate/up rows
        out = torch.zeros(M, N // 2, device="cuda", dtype=torch.bfloat16)
        t = acc.view(M, N // 128, 2, 64)
        ref = (torch.nn.functional.silu(t[:, :, 0]) * t[:, :, 1]).reshape(M, N // 2)
        ldo, tol = N // 2, 3e-2
    elif epi == 5:
        out = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
        ref, ldo, tol = torch.nn.functional.gelu(acc, approximate="tanh"), N, 3e-2
    elif epi == 2:
        base = torch.randn(M, N, device="cuda", generator=g)
        out, ref, ldo, tol = base.clone(), base + acc, N, 1e-4
    elif epi == 3:
        base = torch.randn(M, N, device="cuda", generator=g)
        gate = torch.randn((M + 15) // 16, 3 * N, device="cuda", generator=g)
        out = base.clone()
        ref = base + gate[torch.arange(M, device="cuda") // 16][:, N:2 * N] * acc
        ldo, tol = N, 1e-4
    else:
        out = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
        ref, ldo, tol = acc, N, 3e-2
    gemm(W, X, M, epi, out, ldo, gate, 3 * N if gate is not None else 0, N if gate is not None else 0)
    err = (out.float() - ref.float()).abs()
    assert err.max().item() <= tol * max(1.0, ref.abs().max().item() / 4)


def test_batch_invariance_row_bits():
    g = torch.Generator(device="cuda").manual_seed(3)
    W = (torch.randn(2048, 2048, device="cuda", generator=g) / 45).bfloat16()
    X = torch.randn(256, 2048, device="cuda", generator=g).bfloat16()
    ref = None
    for M in (1, 2, 15, 16, 17, 64, 100, 256):
        out = torch.zeros(M, 2048, device="cuda")
        gemm(W, X, M, 1, out, 2048)
        ref = out[0].clone() if ref is None else ref
        assert torch.equal(out[0], ref), f"row 0 bits changed at M={M}"


def test_n_padding_and_valid_rows():
    # N=64 (DiT out-projection) is padded to one 128-row tile; only 64 columns stored
    g = torch.Generator(device="cuda").manual_seed(5)
    W = torch.zeros(128, 1024, device="cuda", dtype=torch.bfloat16)
    W[:64] = (torch.randn(64, 1024, device="cuda", generator=g) / 32).bfloat16()
    X = torch.randn(48, 1024, device="cuda", generator=g).bfloat16()
    out = torch.full((48, 64), 7.0, device="cuda")
    sp = C.c_int32()
    check(dev_lib().omni_k_gemm(C.c_uint64(W.data_ptr()), 64, 1024, C.c_uint64(X.data_ptr()), 48, 1,
                                C.c_uint64(out.data_ptr()), 64, C.c_uint64(0), 0, 0, 1, 1, C.byref(sp)))
    torch.cuda.synchronize()
    assert (out - X.float() @ W[:64].float().t()).abs().max().item() < 1e-4
