import ctypes as C, sys, torch, time
sys.path.insert(0, '.')
from paper_2602_02204_b200 import dev_lib, check
L = dev_lib()
torch.manual_seed(0)
def run(N, K, M, epi=1):
    W = (torch.randn(N, K, device='cuda') / K**0.5).bfloat16()
    X = torch.randn(M, K, device='cuda').bfloat16()
    ref = X.float() @ W.float().t()
    out = torch.zeros(M, N, device='cuda', dtype=torch.float32)
    sp = C.c_int32(0)
    check(L.omni_k_gemm(C.c_uint64(W.data_ptr()), N, K, C.c_uint64(X.data_ptr()), M, epi, C.c_uint64(out.data_ptr()), N, C.c_uint64(0), 0, 0, 1, 8, C.byref(sp)))
    torch.cuda.synchronize()
    err = (out - ref).abs().max().item()
    print(f"N={N} K={K} M={M} splits={sp.value} maxerr={err:.3e} refmax={ref.abs().max().item():.2f}", flush=True)
    return out, W, X
for (N,K,M) in [(128,64,300),(128,64,1),(128,128,16),(256,2048,5),(3072,2048,16),(2048,2048,64),(16384,2048,33),(2048,8192,200),(1024,1024,2048)]:
    run(N,K,M)
# epilogue variants vs torch
def epi_test(N,K,M,epi):
    W = (torch.randn(N, K, device='cuda') / K**0.5).bfloat16(); X = torch.randn(M, K, device='cuda').bfloat16()
    acc = X.float() @ W.float().t()
    if epi == 4:
        out = torch.zeros(M, N//2, device='cuda', dtype=torch.bfloat16)
        t = acc.view(M, N//128, 2, 64); ref = (torch.nn.functional.silu(t[:,:,0]) * t[:,:,1]).reshape(M, N//2)
        ldo = N//2
    elif epi == 5:
        out = torch.zeros(M, N, device='cuda', dtype=torch.bfloat16); ref = torch.nn.functional.gelu(acc, approximate='tanh'); ldo=N
    elif epi == 2:
        base = torch.randn(M, N, device='cuda'); out = base.clone(); ref = base + acc; ldo=N
    elif epi == 3:
        base = torch.randn(M, N, device='cuda'); out = base.clone(); G = 16; gate = torch.randn((M+G-1)//G, 3*N, device='cuda')
        ref = base + gate[torch.arange(M, device='cuda')//G][:, N:2*N] * acc; ldo=N
    else:
        out = torch.zeros(M, N, device='cuda', dtype=torch.bfloat16); ref = acc; ldo=N
    g = gate if epi == 3 else None
    check(L.omni_k_gemm(C.c_uint64(W.data_ptr()), N, K, C.c_uint64(X.data_ptr()), M, epi, C.c_uint64(out.data_ptr()), ldo,
        C.c_uint64(g.data_ptr() if g is not None else 0), 3*N if g is not None else 0, N if g is not None else 0, 16, 8, None))
    torch.cuda.synchronize()
    print(f"epi={epi} N={N} K={K} M={M} maxerr={(out.float()-ref.float()).abs().max().item():.3e}", flush=True)
for epi in [0,2,3,4,5]:
    for (N,K,M) in [(256,256,7),(1024,2048,40),(512,512,300)]:
        epi_test(N,K,M,epi)
# batch invariance
out1, W, X = run(2048, 2048, 1)
Xb = torch.cat([X, torch.randn(255, 2048, device='cuda').bfloat16()])
outb = torch.zeros(256, 2048, device='cuda')
check(L.omni_k_gemm(C.c_uint64(W.data_ptr()), 2048, 2048, C.c_uint64(Xb.data_ptr()), 256, 1, C.c_uint64(outb.data_ptr()), 2048, C.c_uint64(0), 0, 0, 1, 8, None))
torch.cuda.synchronize()
print("batch-invariant row0:", torch.equal(out1[0], outb[0]))
# timing
for (N,K,M,ms_) in [(3072,2048,1,8),(3072,2048,16,8),(2048,2048,16,8),(16384,2048,1,8),(16384,2048,16,8),(16384,2048,64,8),(2048,8192,16,8),(2048,8192,64,8),(3072,1024,2048,1),(4096,1024,8192,1),(1024,4096,8192,1)]:
    W = torch.randn(N, K, device='cuda').bfloat16(); X = torch.randn(M, K, device='cuda').bfloat16(); out = torch.zeros(M, N, device='cuda')
    ms = C.c_float(0)
    check(L.omni_k_gemm_time(C.c_uint64(W.data_ptr()), N, K, C.c_uint64(X.data_ptr()), M, 1, C.c_uint64(out.data_ptr()), N, 50, C.byref(ms)))
    us = ms.value*1e3
    gbs = (N*K*2 + M*K*2 + M*N*4)/us/1e3
    tf = 2*M*N*K/us/1e6
    print(f"time N={N} K={K} M={M}: {us:.1f} us  {gbs:.0f} GB/s  {tf:.1f} TF/s", flush=True)
