"""Scratch GPU probe: tcgen05 GEMM vs torch fp32 matmul at decode shapes + timing."""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2603_23414_b200 import _lib

lib = _lib.load()
torch.manual_seed(0)
dev = "cuda"
for (M, N, K) in [(16, 256, 128), (200, 384, 256), (256, 6144, 4096), (64, 4096, 14336), (1, 128, 64),
                  (600, 512, 128), (256, 128256, 4096)]:
    X = (torch.randn(M, K, device=dev) * 0.5).to(torch.bfloat16)
    W = (torch.randn(N, K, device=dev) * 0.02).to(torch.bfloat16)
    splits = lib.srl_op_gemm_splits(M, N, K, 148)
    out = torch.full((splits, M, N), float("nan"), device=dev)
    s = torch.cuda.current_stream().cuda_stream
    rc = lib.srl_op_gemm_bf16(X.data_ptr(), M, W.data_ptr(), N, K, out.data_ptr(), splits, s)
    torch.cuda.synchronize()
    ref = X.float() @ W.float().t()
    got = out.sum(0)
    err = (got - ref).abs().max().item()
    rel = ((got - ref).norm() / ref.norm()).item()
    # timing
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        lib.srl_op_gemm_bf16(X.data_ptr(), M, W.data_ptr(), N, K, out.data_ptr(), splits, s)
    ev0.record()
    it = 20
    for _ in range(it):
        lib.srl_op_gemm_bf16(X.data_ptr(), M, W.data_ptr(), N, K, out.data_ptr(), splits, s)
    ev1.record()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / it
    gbs = (N * K * 2) / (ms * 1e-3) / 1e9
    tfl = 2 * M * N * K / (ms * 1e-3) / 1e12
    print(f"M={M} N={N} K={K} splits={splits} rc={rc} maxabs={err:.3e} rel={rel:.3e} "
          f"t={ms*1e3:.1f}us W-GB/s={gbs:.0f} TF/s={tfl:.1f}", flush=True)
